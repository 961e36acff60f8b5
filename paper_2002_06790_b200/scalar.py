"""The reference's remaining hot-path functions, one call at a time (drop-in names of
pkg/src/dfsim/__init__.py:6-43 for SURVEY.md §8a rows P, C, X2, X5, T).

* ``predict`` (costmodel.py:158-165), ``comm_time_us`` / ``transfer_time`` /
  ``allreduce_time`` (costmodel.py:168-223): evaluated by the sm_100a formula kernels
  (csrc/formulas.cu, the same arithmetic as the batched estimate kernel K2).
  ``predict_batch`` / ``comm_batch`` take many rows per launch.
* ``topological_order`` (graph.py:424-443): host C++ Kahn with a rank heap
  (csrc/topo.cpp), the reference's exact order and CycleError.
* ``query_exact`` / ``query_grid`` / ``query_link`` (profiledb.py:107-125) and
  ``apply_overrides`` (strategy.py:285-297): dictionary lookups and copies on the host
  objects -- no arithmetic, nothing to put on a device.
Argument checks and exceptions follow the reference line by line.
"""

from __future__ import annotations

import numpy as np

from . import native
from .errors import CycleError, MissingDurationError, UnknownCollectiveError
from .lowering import find_cycle, host_csr, resolve_overrides
from .model import ALGO_MEASURED, ALGO_RING, DEVICE_LINK, SCENARIO_NCCL_ALLREDUCE, DurationEntry, DurationTable

COLLECTIVE_ALGOS = (ALGO_MEASURED, ALGO_RING)
SOURCE_OVERRIDE = "Override"


def _dev(a, dtype, device):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=dtype), device=f"cuda:{device}")


def predict_batch(model, feature_rows, device: int | None = None) -> np.ndarray:
    """``predict(model, row)`` for every row of ``feature_rows`` ([n, k]) in one launch."""
    ctx = native.Context.get(device)
    k = len(model.feature_names)
    rows = np.asarray(feature_rows, dtype=np.float64).reshape(-1, k) if k else np.zeros((len(feature_rows), 0))
    n = rows.shape[0]
    if n == 0:
        return np.zeros(0)
    import torch

    coef = _dev(np.asarray(model.coefficients, np.float64) if k else np.zeros(1), np.float64, ctx.device)
    feats = _dev(rows if k else np.zeros(1), np.float64, ctx.device)
    out = torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}")
    ctx.call("dfsim_predict_batch", k, native.ptr(coef), float(model.intercept), n, native.ptr(feats), native.ptr(out))
    return out.cpu().numpy()


def predict(model, features) -> float:
    """Model value at a feature vector, clamped to nonnegative (costmodel.py:158-165)."""
    if len(features) != len(model.feature_names):
        raise ValueError(f"expected {len(model.feature_names)} features, got {len(features)}")
    return float(predict_batch(model, [list(features)])[0])


def comm_batch(kind, num_bytes, participants, throughput_mbps, latency_us, device: int | None = None) -> np.ndarray:
    """Formula rows in one launch: kind 0 = comm_time_us, 1 = ring allreduce (see csrc/formulas.cu)."""
    ctx = native.Context.get(device)
    n = len(kind)
    if n == 0:
        return np.zeros(0)
    import torch

    t = [_dev(kind, np.uint8, ctx.device), _dev(num_bytes, np.int64, ctx.device),
         _dev(participants, np.int32, ctx.device), _dev(throughput_mbps, np.float64, ctx.device),
         _dev(latency_us, np.float64, ctx.device)]
    out = torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}")
    ctx.call("dfsim_comm_batch", n, *(native.ptr(x) for x in t), native.ptr(out))
    return out.cpu().numpy()


def comm_time_us(num_bytes: int, throughput_mbps: float, latency_us: float = 0.0) -> float:
    """latency + (bytes / MiB) / throughput * 1e6 (costmodel.py:168-173)."""
    return float(comm_batch([0], [num_bytes], [0], [throughput_mbps], [latency_us])[0])


def transfer_time(num_bytes: int, link) -> float:
    """Point-to-point transfer over a Link device, microseconds (costmodel.py:176-182)."""
    if link.kind != DEVICE_LINK:
        raise ValueError(f"transfer_time needs a Link device, got {link.kind}")
    if num_bytes <= 0:
        raise ValueError(f"bytes must be > 0, got {num_bytes}")
    return comm_time_us(num_bytes, link.throughput_mbps, link.latency_us)


def allreduce_time(num_bytes: int, participants: int, db, algo: str = ALGO_MEASURED, path: str = "PCIeSwitch",
                   fallback_link=None) -> float:
    """Allreduce across ``participants`` devices, microseconds (costmodel.py:185-223)."""
    if num_bytes <= 0:
        raise ValueError(f"bytes must be > 0, got {num_bytes}")
    if participants < 2:
        raise ValueError(f"participants must be >= 2, got {participants}")
    if algo not in COLLECTIVE_ALGOS:
        raise ValueError(f"unknown collective algorithm {algo!r}")
    if algo == ALGO_MEASURED:
        rec = query_link(db, SCENARIO_NCCL_ALLREDUCE, path, participants)
        if rec is not None:
            return comm_time_us(num_bytes, rec.throughput_mbps)
        if fallback_link is None:
            raise UnknownCollectiveError(
                f"no {SCENARIO_NCCL_ALLREDUCE} record for path={path!r} "
                f"participants={participants} and no fallback link")
    if fallback_link is None:
        raise UnknownCollectiveError("ring formula requires a fallback link")
    return float(comm_batch([1], [num_bytes], [participants], [fallback_link.throughput_mbps],
                            [fallback_link.latency_us])[0])


def query_exact(db, sig):
    """Record whose signature equals ``sig`` exactly, else None (profiledb.py:107-112)."""
    grid = db.op_records.get((sig.op_type, sig.hardware))
    if grid is None:
        return None
    return grid.get(sig.arg_features)


def query_grid(db, op_type: str, hardware: str) -> list:
    """All records for (op_type, hardware), sorted by argument features (profiledb.py:115-118)."""
    grid = db.op_records.get((op_type, hardware), {})
    return [grid[k] for k in sorted(grid)]


def query_link(db, scenario: str, path: str, participants: int):
    """Exact-key link lookup; unrecorded combinations return None (profiledb.py:121-125)."""
    if participants < 1:
        raise ValueError(f"participants must be >= 1, got {participants}")
    return db.link_records.get((scenario, path, participants))


def topological_order(g) -> list[str]:
    """Kahn's algorithm with a heap, ties by lexicographic node id (graph.py:424-443)."""
    csr = host_csr(g)
    ids, n = csr["ids"], len(csr["ids"])
    order = np.empty(max(n, 1), np.int32)
    lib = native.load_library()
    p = lambda a: np.ascontiguousarray(a, np.int32).ctypes.data_as(native.P)  # noqa: E731
    off, idx, indeg = (np.ascontiguousarray(csr[k], np.int32) for k in ("succ_off", "succ_idx", "indeg"))
    k = lib.dfsim_topological_order(n, p(off), p(idx) if len(idx) else None, p(indeg), order.ctypes.data_as(native.P))
    if k < 0:
        raise ValueError("topological_order: bad graph arrays")
    if k != n:
        done = {ids[i] for i in order[:k].tolist()}
        cycle = find_cycle(g)
        raise CycleError(cycle or [nid for nid in g.nodes if nid not in done])
    return [ids[i] for i in order[:n].tolist()]


def apply_overrides(table, cfg, g):
    """Stamp manual override durations onto a copy of the table (strategy.py:285-297)."""
    missing = sorted(nid for nid in g.nodes if nid not in table.entries)
    if missing:
        raise MissingDurationError(missing)
    entries = dict(table.entries)
    for nid, value in resolve_overrides(cfg.overrides, sorted(g.nodes)).items():
        entries[nid] = DurationEntry(value, SOURCE_OVERRIDE)
    return DurationTable(entries=entries)
