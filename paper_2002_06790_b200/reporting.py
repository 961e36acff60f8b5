"""Schedule reports on the device: ``summarize`` and ``to_trace``.

Drop-ins for reporting.py:117-162 (``summarize``) and reporting.py:43-74
(``to_trace``), plus batched forms over the schedules a sweep left in HBM
(:meth:`SweepResult.summaries <paper_2002_06790_b200.batch.SweepResult.summaries>`).

Division of work:

* K6 ``dfsim_summarize`` (csrc/summarize.cu) rebuilds each schedule's entry order
  (engine.py:88) on the device and folds, in that order, the per-op-key totals
  (reporting.py:131-133), compute/comm busy (142-148) and the interval overlap sweep
  (92-114, 149); the critical path (154) is K4 (``simulator.critical_path``).
* The host keeps the few steps whose cost does not grow with the graph: the
  first-appearance order of the key totals, the reference's own ``sum`` (Neumaier in
  CPython 3.12) over them, the ``sorted(..., key=(-total, name))`` ranking and the
  utilisation ratios (engine.py:218-222).
* ``to_trace`` runs the byte-identical C++ writer ``dfsim_trace_write`` (csrc/trace.cpp).

Parity: tests/test_gpu_reporting.py against the reference's own summaries and trace
hashes in tests/golden/ (make_golden.py runs reporting.summarize / to_trace).
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import DfsimError
from .model import DEVICE_COMPUTE, SOURCE_TAGS, Schedule, utilization


@dataclass
class SummaryReport:
    """reporting.py:19-31 (same fields, same meaning)."""

    makespan_us: float
    per_device_busy_us: dict
    utilization: dict
    device_kinds: dict
    top_k_ops: list          # (op key, total us, share of all op time)
    compute_us: float
    comm_us: float
    overlap_us: float
    critical_path_nodes: list = field(default_factory=list)
    critical_path_us: float = 0.0


# ----------------------------------------------------------------------------- device folds


class SummaryTables:
    """Class-wide K6 tables (node-rank indexed) on one device.

    ``keys[k]`` is the k-th distinct op key (``op_type or node_id``) in code-point order;
    ``key_of[v]`` its index for node rank v; ``comm[v]`` = the node's device is not Compute
    in ``kinds`` (absent devices count as Compute, reporting.py:140)."""

    def __init__(self, key_strings, comm, dev_rank, device: int, base_order=None):
        import torch

        n = len(key_strings)
        self.n = n
        self.keys = sorted(set(key_strings)) or [""]
        kidx = {k: i for i, k in enumerate(self.keys)}
        self.key_of = np.fromiter((kidx[k] for k in key_strings), dtype=np.int32, count=n)
        d = f"cuda:{device}"
        self.t_key = torch.from_numpy(self.key_of if n else np.zeros(1, np.int32)).to(d)
        self.t_comm = torch.from_numpy(np.asarray(comm, np.uint8) if n else np.zeros(1, np.uint8)).to(d)
        if base_order is None and dev_rank is not None:
            base_order = np.lexsort((np.arange(n), np.asarray(dev_rank))).astype(np.int32) if n else None
        self.t_base = None if base_order is None or not n else torch.from_numpy(np.asarray(base_order, np.int32)).to(d)
        self.struct = native.SummaryTables(n, len(self.keys), native.ptr(self.t_base), native.ptr(self.t_key),
                                           native.ptr(self.t_comm))


def run_summary(ctx, tables: SummaryTables, start, finish, entry_order=None):
    """K6 over rows start/finish [R][>=N] (device, by node index).  Returns device tensors
    (entry_order [R][N], key_total [R][K], key_first [R][K], sums [R][3])."""
    import torch

    R, N, K = start.shape[0], tables.n, len(tables.keys)
    dev = start.device
    given = entry_order is not None
    if entry_order is None:
        entry_order = torch.empty((R, max(N, 1)), dtype=torch.int32, device=dev)
    key_total = torch.empty((R, K), dtype=torch.float64, device=dev)
    key_first = torch.empty((R, K), dtype=torch.int32, device=dev)
    sums = torch.empty((R, 3), dtype=torch.float64, device=dev)
    ctx.call("dfsim_summarize", ctypes.byref(tables.struct), R, native.ptr(start), native.ptr(finish),
             start.stride(0) if R else max(N, 1), native.ptr(entry_order), 1 if given else 0,
             native.ptr(key_total), native.ptr(key_first), native.ptr(sums))
    return entry_order, key_total, key_first, sums


def rank_ops(keys, key_total_row, key_first_row, top_k: int):
    """reporting.py:131-138 on one row of K6 output: totals in first-appearance order,
    the reference's own sum and (-total, name) ranking."""
    present = np.nonzero(key_first_row >= 0)[0]
    present = present[np.argsort(key_first_row[present], kind="stable")]
    totals = {keys[k]: float(key_total_row[k]) for k in present.tolist()}
    grand_total = sum(totals.values())
    ranked = sorted(totals.items(), key=lambda kv: (-kv[1], kv[0]))[: max(0, top_k)]
    return [(name, total, total / grand_total if grand_total > 0 else 0.0) for name, total in ranked]


# ----------------------------------------------------------------------------- drop-ins


def summarize(s: Schedule, g, top_k: int = 10, device: int | None = None) -> SummaryReport:
    """reporting.summarize (reporting.py:117-162) with the folds on the GPU."""
    import torch

    from .simulator import critical_path

    schedule_ids = {e.node_id for e in s.entries}
    if schedule_ids != set(g.nodes):
        raise DfsimError("schedule does not correspond to the graph (node sets differ)")
    ctx = native.Context.get(device)
    kinds = {dev: spec.kind for dev, spec in g.devices.items()}
    entries = s.entries
    n = len(entries)
    # node index = entry index; the Schedule's own entry order is the fold order
    keys = [e.op_type or e.node_id for e in entries]
    comm = [kinds.get(e.device, DEVICE_COMPUTE) != DEVICE_COMPUTE for e in entries]
    tables = SummaryTables(keys, comm, None, ctx.device)
    d = f"cuda:{ctx.device}"
    st = torch.tensor([[e.start_us for e in entries]], dtype=torch.float64).reshape(1, n).to(d)
    fi = torch.tensor([[e.finish_us for e in entries]], dtype=torch.float64).reshape(1, n).to(d)
    order = torch.arange(max(n, 1), dtype=torch.int32, device=d).reshape(1, -1)
    _, key_total, key_first, sums = run_summary(ctx, tables, st, fi, entry_order=order)
    durations = {e.node_id: e.finish_us - e.start_us for e in entries}
    cp_len, cp_nodes = critical_path(g, durations, ctx.device)
    kt, kf, sm = key_total.cpu().numpy()[0], key_first.cpu().numpy()[0], sums.cpu().numpy()[0]
    return SummaryReport(
        makespan_us=s.makespan_us,
        per_device_busy_us=dict(s.per_device_busy_us),
        utilization=utilization(s),
        device_kinds=kinds,
        top_k_ops=rank_ops(tables.keys, kt, kf, top_k) if n else [],
        compute_us=float(sm[0]),
        comm_us=float(sm[1]),
        overlap_us=float(sm[2]),
        critical_path_nodes=cp_nodes,
        critical_path_us=cp_len,
    )


class TraceTables:
    """Host string tables of dfsim_trace_write for n nodes (kept alive with the struct)."""

    def __init__(self, ids, names, tags, tracks, track_names, tag_names=SOURCE_TAGS):
        n = len(ids)
        self.n = n
        self._id_blob, self._id_off = _blob(ids)
        self._name_blob, self._name_off = _blob(names)
        self._tag = np.ascontiguousarray(tags, dtype=np.uint8) if n else np.zeros(1, np.uint8)
        self._track = np.ascontiguousarray(tracks, dtype=np.int32) if n else np.zeros(1, np.int32)
        tn = [t.encode("utf-8", "surrogatepass") for t in tag_names] + [b""]
        self._tag_names = (ctypes.c_char_p * len(tn))(*tn)
        enc = [t.encode("utf-8", "surrogatepass") for t in track_names]
        self._track_names = (ctypes.c_char_p * max(len(enc), 1))(*enc) if enc else None
        self.struct = native.TraceTables(
            n, len(track_names), self._id_blob.ctypes.data, self._id_off.ctypes.data, self._name_blob.ctypes.data,
            self._name_off.ctypes.data, self._tag.ctypes.data, ctypes.cast(self._tag_names, native.P),
            self._track.ctypes.data, ctypes.cast(self._track_names, native.P) if enc else None)

    def write(self, entry_node, start, finish, tags=None) -> str:
        """The document for entries ``entry_node`` (node indices in entry order); ``tags``
        optionally replaces the per-node source tags for this call."""
        lib = native.load_library()
        if tags is not None:
            self._tag = np.ascontiguousarray(tags, dtype=np.uint8) if self.n else np.zeros(1, np.uint8)
            self.struct.tag = self._tag.ctypes.data
        en = np.ascontiguousarray(entry_node, dtype=np.int32)
        st = np.ascontiguousarray(start, dtype=np.float64)
        fi = np.ascontiguousarray(finish, dtype=np.float64)
        args = (ctypes.byref(self.struct), len(en), en.ctypes.data, st.ctypes.data, fi.ctypes.data)
        cap = 256 + 200 * len(en) + 96 * self.struct.n_tracks + len(self._id_blob) * 6 + len(self._name_blob) * 6
        buf = getattr(self, "_buf", None)  # reused between calls (no zero-fill, no fresh pages)
        if buf is None or len(buf) < cap:
            buf = self._buf = np.empty(cap, np.uint8)
        size = lib.dfsim_trace_write(*args, buf.ctypes.data, len(buf))
        if size < 0:
            raise ValueError("dfsim_trace_write: bad arguments")
        if size > len(buf):
            buf = self._buf = np.empty(size, np.uint8)
            lib.dfsim_trace_write(*args, buf.ctypes.data, size)
        return buf[:size].tobytes().decode("ascii")


def _blob(strings):
    enc = [x.encode("utf-8", "surrogatepass") for x in strings]
    off = np.zeros(len(enc) + 1, np.int64)
    if enc:
        np.cumsum([len(b) for b in enc], out=off[1:])
    blob = np.frombuffer(b"".join(enc) + b"\0", dtype=np.uint8).copy()
    return blob, off


def to_trace(s: Schedule) -> str:
    """reporting.to_trace (reporting.py:43-74), byte-identical, from the C++ writer."""
    devices = sorted(s.per_device_busy_us)
    tid = {dev: i for i, dev in enumerate(devices)}
    entries = s.entries
    tag_of = {t: i for i, t in enumerate(SOURCE_TAGS)}
    for e in entries:  # any source string beyond the four reference tags gets its own slot
        if e.source not in tag_of:
            tag_of[e.source] = len(tag_of)
    if len(tag_of) > 255:
        raise ValueError("more than 255 distinct duration sources")
    t = TraceTables([e.node_id for e in entries], [e.op_type or e.node_id for e in entries],
                    [tag_of[e.source] for e in entries], [tid.get(e.device, len(devices)) for e in entries], devices,
                    tag_names=list(tag_of))
    return t.write(np.arange(len(entries)), [e.start_us for e in entries], [e.finish_us for e in entries])


def trace_intervals(trace_text: str) -> list:
    """reporting.py:77-86: (device, start, finish, op name) tuples of a trace document."""
    events = json.loads(trace_text)
    names = {ev["tid"]: ev["args"]["name"] for ev in events if ev["ph"] == "M"}
    return [(names.get(ev["tid"], str(ev["tid"])), ev["ts"], ev["ts"] + ev["dur"], ev["name"])
            for ev in events if ev["ph"] == "X"]


def render_summary_text(report: SummaryReport) -> str:
    """reporting.py:165-191 (plain formatting of a SummaryReport)."""
    lines = [
        f"makespan: {report.makespan_us / 1000.0:.2f} ms ({report.makespan_us:.3f} us)",
        f"compute busy: {report.compute_us:.3f} us",
        f"communication busy: {report.comm_us:.3f} us",
        f"compute/comm overlap: {report.overlap_us:.3f} us",
        "",
        "device utilization:",
    ]
    for dev in sorted(report.per_device_busy_us):
        lines.append(f"  {dev} [{report.device_kinds.get(dev, '?')}]: busy {report.per_device_busy_us[dev]:.3f} us, "
                     f"utilization {report.utilization.get(dev, 0.0):6.2%}")
    lines += ["", "top ops by total time:"]
    lines += [f"  {name}: {total:.3f} us ({share:.2%})" for name, total, share in report.top_k_ops]
    lines += ["", f"critical path: {report.critical_path_us:.3f} us over {len(report.critical_path_nodes)} nodes"]
    if report.critical_path_nodes:
        lines.append("  " + " -> ".join(report.critical_path_nodes))
    return "\n".join(lines) + "\n"
