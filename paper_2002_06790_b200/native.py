"""ctypes binding of libdfsim_b200.so (include/dfsim_b200.h).

There is no fallback: if the library is missing, cannot be loaded, or no CUDA
device is present, every entry point raises :class:`NativeError`.  ctypes drops
the GIL for the duration of each foreign call; a per-device :class:`Context` is
shared by every thread and serialises its calls with a lock (see ``Context``), so
the reference's ``--jobs`` threads (cli.py:133-137) may call the drop-in concurrently.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import (
    STATUS_BAD_ARGUMENT,
    STATUS_CHECK_FAILED,
    STATUS_CUDA,
    STATUS_OK,
    NativeError,
)

# DFSIM_LIB=checked loads the bounds-checked build (tests / profiles/sanitize_run.py only)
LIB_PATH = Path(__file__).resolve().parent / (
    "libdfsim_b200_checked.so" if os.environ.get("DFSIM_LIB") == "checked" else "libdfsim_b200.so")

P = ctypes.c_void_p
I32, I64, U8 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8


class Graph(ctypes.Structure):
    _fields_ = [("n_nodes", I32), ("n_devices", I32), ("n_edges", I64), ("succ_off", P), ("succ_idx", P),
                ("indeg", P), ("device", P), ("sources", P), ("n_sources", I32), ("queue_off", P), ("topo", P),
                ("max_indeg", I32)]


class BaseGraph(ctypes.Structure):
    _fields_ = [("n_base", I32), ("in_off", P), ("in_src", P), ("base_dev", P), ("remap", P), ("marked", P),
                ("n_refs", I32)]


class ExpandPlan(ctypes.Structure):
    _fields_ = [("replicas", I32), ("n_collectives", I32), ("clone_rank", P), ("coll_rank", P), ("map_dev", P),
                ("fabric_dev", I32), ("ps", I32), ("push_rank", P), ("pull_rank", P), ("up_dev", P), ("down_dev", P),
                ("ps_dev", I32)]


class ProfileTables(ctypes.Structure):
    _fields_ = [("op", P), ("kind", P), ("sig", P), ("comm_bytes", P), ("comm_ok", P), ("group_size", P),
                ("link_thr", P), ("link_lat", P),
                ("n_sigs", I32), ("sig_off", P), ("sig_name", P), ("sig_val", P),
                ("n_exact", I32), ("exact_key", P), ("exact_mean", P),
                ("n_models", I32), ("model_key", P), ("model_off", P), ("model_name", P), ("model_coef", P),
                ("model_icpt", P),
                ("n_nccl", I32), ("nccl_key", P), ("nccl_thr", P),
                ("n_paths", I32), ("uni_ok", P), ("uni_thr", P), ("uni_lat", P),
                ("n_override_sets", I32), ("ov_off", P), ("ov_node", P), ("ov_val", P)]


class Strategies(ctypes.Structure):
    _fields_ = [("n_sims", I64), ("hw", P), ("op_gap", P), ("algo", P), ("path", P), ("override_set", P),
                ("gvariant", P)]


class SimTables(ctypes.Structure):
    _fields_ = [("n_nodes", I32), ("n_devices", I32), ("n_edges", I64), ("meta", P), ("succ_off", P), ("succ", P),
                ("cidx", P), ("cnt_init", P), ("n_counter_words", I32), ("counter_bits", I32), ("rank", P),
                ("sources", P), ("n_sources", I32), ("qcap", I32), ("device", P), ("succ_packed", I32)]


class FusedStrategies(ctypes.Structure):
    _fields_ = [("n_sims", I64), ("n_variants", I32), ("base", P), ("n_chunks", I32), ("order", P),
                ("chunk_first", P), ("chunk_count", P), ("chunk_variant", P), ("op_gap", P), ("override_set", P),
                ("ov_off", P), ("ov_node", P), ("ov_val", P), ("max_chunk", I32), ("ov_any", P),
                ("sched_tiled", I32)]


class CpTables(ctypes.Structure):
    _fields_ = [("n_nodes", I32), ("n_slots", I32), ("n_edges", I32), ("rank_of_pos", P), ("cp_meta", P),
                ("cp_slot", P), ("cp_succ_slot", P), ("n_groups", I32), ("group_off", P), ("n_chunks", I32),
                ("chunk_off", P), ("chunk_positions", I32), ("n_long", I32), ("cp_spill", P), ("spill_off", P),
                ("spill_list", P), ("max_spill_reads", I32), ("pinfo", P), ("slot_region", I32), ("stage_doubles", I32)]


class CpLaneTables(ctypes.Structure):
    _fields_ = [("n_nodes", I32), ("n_chunks", I32), ("chunk_positions", I32), ("n_slots", I32), ("rmax", I32),
                ("n_long", I32), ("n_spill_list", I32), ("block_max", I32), ("blocks", P), ("block_off", P),
                ("bounds", P), ("spill_off", P), ("spill_list", P), ("rank_of_pos", P)]


class SummaryTables(ctypes.Structure):
    _fields_ = [("n_nodes", I32), ("n_keys", I32), ("base_order", P), ("key", P), ("comm", P)]


class TraceTables(ctypes.Structure):
    _fields_ = [("n_nodes", I32), ("n_tracks", I32), ("id_blob", P), ("id_off", P), ("name_blob", P),
                ("name_off", P), ("tag", P), ("tag_name", P), ("track", P), ("track_name", P)]


class Document(ctypes.Structure):
    _fields_ = [(n, I32) for n in ("n_nodes", "n_devices", "n_ops", "n_sigs", "n_fnames", "n_declared", "max_indeg",
                                    "n_sources")] + [("n_edges", I64)] + [
        (n, P) for n in ("id_blob", "id_off", "op_blob", "op_off", "dev_blob", "dev_off", "fname_blob", "fname_off",
                         "op_of", "kind_of", "dev_of", "indeg", "succ_off", "succ_idx", "sources", "queue_off",
                         "sig_of", "sig_off", "sig_fname", "sig_fval", "comm_ok", "comm_bytes", "group_size",
                         "link_thr", "link_lat", "node_lo", "node_hi")] + [
        (n, I64) for n in ("meta_lo", "meta_hi", "decl_lo", "decl_hi")]


_SIGNATURES = {
    "dfsim_abi_version": (I32, []),
    "dfsim_ctx_create": (ctypes.c_int, [I32, P, ctypes.POINTER(P)]),
    "dfsim_ctx_destroy": (ctypes.c_int, [P]),
    "dfsim_ctx_set_stream": (ctypes.c_int, [P, P]),
    "dfsim_ctx_launch_count": (I64, [P]),
    "dfsim_ctx_last_error": (ctypes.c_char_p, [P]),
    "dfsim_topo_order": (ctypes.c_int, [P, ctypes.POINTER(Graph), P, ctypes.POINTER(I32)]),
    "dfsim_expand_dp": (ctypes.c_int, [P, ctypes.POINTER(BaseGraph), ctypes.POINTER(ExpandPlan), P, P, I64, P, P, P,
                                       P, P, I32, ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I32)]),
    "dfsim_estimate_batch": (ctypes.c_int, [P, I32, ctypes.POINTER(ProfileTables), ctypes.POINTER(Strategies), P, P,
                                            P]),
    "dfsim_simulate_batch": (ctypes.c_int, [P, ctypes.POINTER(Graph), I64, P, I64, P, P, P, P, P]),
    "dfsim_critical_path_batch": (ctypes.c_int, [P, ctypes.POINTER(Graph), I64, P, P, P, P, P]),
    "dfsim_critical_path_wide": (ctypes.c_int, [P, ctypes.POINTER(Graph), P, P, I32, I64, P, P, P, P]),
    "dfsim_simulate_batch_ex": (ctypes.c_int, [P, ctypes.POINTER(Graph), I64, P, I64, P, P, P, P, P, P, P, I32]),
    "dfsim_resolve_variants": (ctypes.c_int, [P, I32, ctypes.POINTER(ProfileTables), I32, P, P, P, P, P, P]),
    "dfsim_override_rows": (ctypes.c_int, [P, I32, I32, P, P, P, P, P, P, P]),
    "dfsim_simulate_fused": (ctypes.c_int, [P, ctypes.POINTER(SimTables), ctypes.POINTER(FusedStrategies), P, P, P,
                                            P, P]),
    "dfsim_critical_path_levels": (ctypes.c_int, [P, ctypes.POINTER(CpTables), I64, P, P, P, P]),
    "dfsim_critical_path_levels_capacity": (I32, [ctypes.POINTER(CpTables)]),
    "dfsim_critical_path_lanes": (ctypes.c_int, [P, ctypes.POINTER(CpLaneTables), I32, I64, P, P, P, P]),
    "dfsim_critical_path_lanes_ex": (ctypes.c_int, [P, ctypes.POINTER(CpLaneTables), I32, I64, P, P, I32, P, P, P]),
    "dfsim_critical_path_lanes_capacity": (I32, [ctypes.POINTER(CpLaneTables), I32]),
    "dfsim_cp_lanes_plan": (ctypes.c_int, [I32, P, P, P, I32, I32, I32, I32, P, P, P, P, P, P]),
    "dfsim_predict_batch": (ctypes.c_int, [P, I32, P, ctypes.c_double, I64, P, P]),
    "dfsim_comm_batch": (ctypes.c_int, [P, I64, P, P, P, P, P, P]),
    "dfsim_topological_order": (I32, [I32, P, P, P, P]),
    "dfsim_level_order": (I32, [I32, P, P, P, P, P, P]),
    "dfsim_cp_levels_plan": (I32, [I32, P, P, P, P, P, I32, I32, I32] + [P] * 11),
    "dfsim_fused_capacity": (I32, [ctypes.POINTER(SimTables)]),
    "dfsim_fused_chunk": (I32, [ctypes.POINTER(SimTables), I64, I32]),
    "dfsim_argmin": (ctypes.c_int, [P, I64, P, I64, P]),
    "dfsim_argmin_records": (ctypes.c_int, [P, I64, P, P]),
    "dfsim_summarize": (ctypes.c_int, [P, ctypes.POINTER(SummaryTables), I64, P, P, I64, P, I32, P, P, P]),
    "dfsim_trace_write": (I64, [ctypes.POINTER(TraceTables), I64, P, P, P, P, I64]),
    "dfsim_document_parse": (ctypes.c_int, [ctypes.c_char_p, I64, ctypes.POINTER(P), ctypes.c_char_p, I64]),
    "dfsim_document_view": (ctypes.POINTER(Document), [P]),
    "dfsim_document_free": (None, [P]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def load_library(path: Path | None = None):
    """Load (once) and type the shared library; raises NativeError if unavailable."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeError(f"{p} is missing: build it with `python -m paper_2002_06790_b200.build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        if path is None:
            _lib = lib
        return lib


class Context:
    """One dfsim_ctx per CUDA device; calls run on the caller's current torch stream.

    Thread safety (the reference allows concurrent simulations, and its CLI
    sweeps on a thread pool, cli.py:133-137): ctypes releases the GIL during every call, so
    ``call`` holds this context's lock across binding the caller's stream, the C call and
    reading its error text.  Launches from several threads are thereby serialised per device
    (they are asynchronous, so the GPU work itself still overlaps on the callers' streams);
    device scratch belongs to (context, stream) inside the library."""

    _by_device: dict[int, "Context"] = {}
    _create_lock = threading.Lock()

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise NativeError("no CUDA device: the B200 path has no CPU fallback")
        self.lib = load_library()
        self.device = device
        handle = P()
        with torch.cuda.device(device):
            torch.cuda.init()
            self._check(self.lib.dfsim_ctx_create(device, None, ctypes.byref(handle)), "ctx_create", ctx=False)
        self.handle = handle
        self.lock = threading.RLock()

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        import torch

        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        ctx = cls._by_device.get(device)
        if ctx is None:
            with cls._create_lock:
                ctx = cls._by_device.get(device)
                if ctx is None:
                    ctx = cls._by_device[device] = Context(device)
        return ctx

    def bind_stream(self):
        import torch

        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.lib.dfsim_ctx_set_stream(self.handle, P(stream))

    def launches(self) -> int:
        return int(self.lib.dfsim_ctx_launch_count(self.handle))

    def _check(self, rc: int, what: str, ctx: bool = True):
        if rc == STATUS_OK:
            return
        msg = self.lib.dfsim_ctx_last_error(self.handle).decode() if ctx else ""
        if rc == STATUS_BAD_ARGUMENT:
            raise ValueError(f"{what}: {msg}")
        if rc == STATUS_CUDA:
            raise NativeError(f"{what}: CUDA failure: {msg}")
        if rc == STATUS_CHECK_FAILED:
            raise NativeError(f"{what}: {msg}")
        raise NativeError(f"{what}: status {rc}: {msg}")

    def call(self, name: str, *args):
        with self.lock:
            self.bind_stream()
            self._check(getattr(self.lib, name)(self.handle, *args), name)


def ptr(t) -> P:
    """Device (or host) address of a torch tensor / None."""
    return P(0) if t is None else P(t.data_ptr())
