"""Drop-in ``simulate`` / ``critical_path`` and their batched array forms.

``simulate(g, durations)`` keeps the reference signature and result type
(engine.py:96 -> Schedule); ``critical_path(g, durations)`` keeps graph.py:446.
Both lower the graph once (cached on the graph object), then run the sm_100a
kernels of libdfsim_b200.so: K3 ``dfsim_simulate_batch`` and K4
``dfsim_critical_path_batch``.  ``simulate_arrays`` / ``critical_path_arrays``
are the batched forms over [S, N] device tensors used by the sweep.
"""

from __future__ import annotations

import numpy as np

from . import native
from .errors import CycleError, MissingDurationError
from .lowering import LoweredGraph, lowered, raise_topo_cycle
from .model import Schedule, ScheduledNode


def _torch():
    import torch

    return torch


def simulate_arrays(lg: LoweredGraph, dur, *, schedule: bool = True, busy: bool = True, out=None) -> dict:
    """K3 over every row of ``dur`` ([S, N] float64 CUDA tensor, or [N] broadcast).

    Returns device tensors: makespan[S], n_placed[S], and when requested
    start/finish [S, N] (NaN where a node was never placed) and busy [S, D].
    """
    torch = _torch()
    dev = f"cuda:{lg.ctx.device}"
    if dur.dim() == 1:
        S, stride = 1, 0
    else:
        S, stride = dur.shape[0], dur.stride(0)
    assert dur.dtype == torch.float64 and dur.is_cuda and (dur.dim() == 1 or dur.stride(1) == 1)
    N, D = lg.n, lg.n_devices
    o = out if out is not None else {}
    if schedule:
        if "start" not in o:
            o["start"] = torch.full((S, max(N, 1)), float("nan"), dtype=torch.float64, device=dev)
            o["finish"] = torch.full((S, max(N, 1)), float("nan"), dtype=torch.float64, device=dev)
    o.setdefault("makespan", torch.empty(S, dtype=torch.float64, device=dev))
    o.setdefault("n_placed", torch.empty(S, dtype=torch.int32, device=dev))
    if busy:
        o.setdefault("busy", torch.zeros((S, max(D, 1)), dtype=torch.float64, device=dev))
    lg.ctx.call("dfsim_simulate_batch", native.ctypes.byref(lg.struct), S, native.ptr(dur), stride,
                native.ptr(o.get("start") if schedule else None), native.ptr(o.get("finish") if schedule else None),
                native.ptr(o["makespan"]), native.ptr(o.get("busy") if busy else None), native.ptr(o["n_placed"]))
    return o


WIDE_CP_NODES = 65536  # from here on one CTA per candidate beats one thread per candidate


def critical_path_arrays(lg: LoweredGraph, start, finish, *, paths: bool = False, out=None) -> dict:
    """K4 over [S, N] schedules (``start`` None: ``finish`` holds plain durations)."""
    torch = _torch()
    if not lg.acyclic:
        raise ValueError("critical path needs an acyclic graph")
    S = finish.shape[0] if finish.dim() == 2 else 1
    dev = finish.device
    o = out if out is not None else {}
    o.setdefault("cp_len", torch.empty(S, dtype=torch.float64, device=dev))
    if not paths and lg.n >= WIDE_CP_NODES and lg.levels() is not None:
        order, loff, n_levels = lg.levels()  # K4 wide: level-parallel inside each candidate
        lg.ctx.call("dfsim_critical_path_wide", native.ctypes.byref(lg.struct), native.ptr(order), native.ptr(loff),
                    n_levels, S, native.ptr(start), native.ptr(finish), native.ptr(o["cp_len"]), native.P(0))
        return o
    if paths:
        o.setdefault("cp_path", torch.empty((S, max(lg.n, 1)), dtype=torch.int32, device=dev))
        o.setdefault("cp_path_len", torch.empty(S, dtype=torch.int32, device=dev))
    lg.ctx.call("dfsim_critical_path_batch", native.ctypes.byref(lg.struct), S, native.ptr(start),
                native.ptr(finish), native.ptr(o["cp_len"]), native.ptr(o.get("cp_path") if paths else None),
                native.ptr(o.get("cp_path_len") if paths else None))
    return o


def _durations_of(table) -> tuple[dict, dict]:
    entries = table.entries
    return {nid: e.duration_us for nid, e in entries.items()}, entries


def simulate(g, durations, device: int | None = None) -> Schedule:
    """engine.py:96-146 on the GPU; same Schedule (entries in (start, device, id) order)."""
    torch = _torch()
    values, entries = _durations_of(durations)
    missing = sorted(nid for nid in g.nodes if nid not in values)
    if missing:
        raise MissingDurationError(missing)
    lg = lowered(g, device)
    N = lg.n
    dur = torch.from_numpy(np.fromiter((values[nid] for nid in lg.ids), dtype=np.float64, count=N))
    dur = dur.to(f"cuda:{lg.ctx.device}") if N else torch.zeros(1, dtype=torch.float64, device=f"cuda:{lg.ctx.device}")
    o = simulate_arrays(lg, dur)
    placed = int(o["n_placed"][0].item())
    start = o["start"][0, :N].cpu().numpy()
    finish = o["finish"][0, :N].cpu().numpy()
    if placed != N:
        raise CycleError(sorted(lg.ids[i] for i in np.nonzero(np.isnan(start))[0]))
    return build_schedule(g, lg, start, finish, float(o["makespan"][0].item()),
                          o["busy"][0, : lg.n_devices].cpu().numpy(), entries)


def build_schedule(g, lg: LoweredGraph, start, finish, makespan, busy_by_rank, entries=None,
                   devices=None) -> Schedule:
    """Schedule object from kernel outputs; entries ordered (start, device, id) (engine.py:88).
    ``devices``: names by device rank when they differ from lg's (another collective path)."""
    dev = lg.device_of_rank()
    order = np.lexsort((np.arange(lg.n), dev, start)) if lg.n else np.zeros(0, np.int64)
    ids, devices = lg.ids, (lg.devices if devices is None else devices)
    out = []
    for i in order.tolist():
        nid = ids[i]
        out.append(ScheduledNode(nid, devices[dev[i]], float(start[i]), float(finish[i]),
                                 entries[nid].source if entries is not None else "",
                                 g.nodes[nid].op_type))
    busy = {d: 0.0 for d in g.devices}
    dev_busy = {devices[k]: float(busy_by_rank[k]) for k in range(lg.n_devices)}
    for d in g.devices:
        if d in dev_busy:
            busy[d] = dev_busy[d]
    for e in out:  # devices outside g.devices appear in entry order (engine.py:90-92)
        if e.device not in busy:
            busy[e.device] = dev_busy[e.device]
    return Schedule(entries=out, makespan_us=makespan, per_device_busy_us=busy)


def critical_path(g, durations: dict, device: int | None = None) -> tuple[float, list[str]]:
    """graph.py:446-485 on the GPU: (length, lexicographically smallest longest path)."""
    torch = _torch()
    missing = sorted(nid for nid in g.nodes if nid not in durations)
    if missing:
        raise MissingDurationError(missing)
    if not g.nodes:
        return 0.0, []
    lg = lowered(g, device)
    if not lg.acyclic:
        raise_topo_cycle(g, lg)
    d = torch.from_numpy(np.fromiter((durations[nid] for nid in lg.ids), dtype=np.float64, count=lg.n))
    d = d.to(f"cuda:{lg.ctx.device}").reshape(1, -1)
    o = critical_path_arrays(lg, None, d, paths=True)
    k = int(o["cp_path_len"][0].item())
    path = o["cp_path"][0, :k].cpu().numpy()
    return float(o["cp_len"][0].item()), [lg.ids[i] for i in path.tolist()]
