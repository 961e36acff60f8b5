"""Candidate sweeps sharded over several GPUs.

The reference's only many-strategy fan-out is ``dfsim simulate --config ... --jobs J``
(cli.py:123-149: one ``_run_one_simulation`` per config on a thread pool).  Candidates
are independent, so each GPU takes a contiguous slice of the config list and runs the
whole hot path on it (expand -> estimate -> simulate -> critical path, batch.sweep_local)
with no data-path traffic between GPUs.  The single exchange is K5's: every GPU reduces its
slice to one 16-byte winner ``(makespan, global index)``; the winners are gathered and
reduced again on the device (``dfsim_argmin_records``) -- the first minimum over the whole
list, ties across shards included, exactly ``min(range(S), key=makespan.__getitem__)``.

Two ways to run it, same results as ``sweep_variants`` on one GPU:
* one process per GPU under ``torch.distributed`` (NCCL over NVLink; ``torchrun``): every
  rank calls ``sweep_sharded`` with the full config list, simulates its own slice, and the
  winners travel by ``all_gather_into_tensor``.  With ``gather_all`` (default) the per-rank
  makespans and critical-path lengths are all-gathered too, so every rank returns the full
  arrays (16 bytes per candidate).
* one process driving several devices (``devices=[0, 1, ...]``, no process group): one host
  thread per device issues that device's launches (ctypes releases the GIL, so the devices
  run concurrently), and the winners are copied peer-to-peer to ``devices[0]``.
"""

from __future__ import annotations

import threading

import numpy as np

from . import native
from .batch import SweepResult, shard, sweep_local


def _dist_world(group):
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return None
    if not (dist.is_available() and dist.is_initialized()):
        return None
    return dist.get_rank(group), dist.get_world_size(group)


def sweep_sharded(graphs, db, configs, graph_of=None, devices=None, keep_schedules: bool = False,
                  fused: bool = True, streams: int = 32, group=None, gather_all: bool = True) -> SweepResult:
    """``sweep_variants`` over several GPUs; identical results (makespans, critical paths,
    best index and makespan, the first failing config's exception).

    ``graphs``: one graph or a list; ``graph_of[i]``: the graph of ``configs[i]`` (default 0).
    Under an initialised process group the candidates are split over its ranks (``devices``
    may name this rank's device; default the current CUDA device), otherwise over
    ``devices`` (default: every visible GPU) from this process.

    The returned ``SweepResult`` keeps the schedules (``keep_schedules``) of the candidates
    simulated in this process; ``schedule(i)`` / ``summary(i)`` / ``trace(i)`` work for those.
    """
    if not isinstance(graphs, (list, tuple)):
        graphs = [graphs]
    graph_of = list(graph_of) if graph_of is not None else [0] * len(configs)
    if len(graph_of) != len(configs):
        raise ValueError("graph_of must name one graph per config")
    dist_rw = _dist_world(group)
    if dist_rw is not None and dist_rw[1] > 1:
        return _sweep_distributed(graphs, db, configs, graph_of, devices, keep_schedules, fused, streams, group,
                                  gather_all, *dist_rw)
    return _sweep_devices(graphs, db, configs, graph_of, devices, keep_schedules, fused, streams)


def _merge(results, shards, S) -> SweepResult:
    """One SweepResult from per-shard results (candidate indices made global)."""
    out = SweepResult(np.zeros(S), np.zeros(S), -1, float("nan"))
    for (lo, hi), res in zip(shards, results):
        if res is None:
            continue
        out.makespan[lo:hi] = res.makespan
        out.cp_len[lo:hi] = res.cp_len
        base = len(out.classes)
        for tc, idx, o in res.classes:
            out.classes.append((tc, [lo + i for i in idx], o))
        for i, (c, row) in res._where.items():
            out._where[lo + i] = (base + c, row)
    return out


def _sweep_devices(graphs, db, configs, graph_of, devices, keep_schedules, fused, streams) -> SweepResult:
    import torch

    devs = list(devices) if devices is not None else list(range(torch.cuda.device_count()))
    if not devs:
        raise native.NativeError("no CUDA device: the B200 path has no CPU fallback")
    S, W = len(configs), len(devs)
    shards = [shard(S, k, W) for k in range(W)]
    results, records, failures, errors = [None] * W, [None] * W, [None] * W, [None] * W

    def run(k):
        lo, hi = shards[k]
        try:
            with torch.cuda.device(devs[k]):
                results[k], records[k], failures[k] = sweep_local(
                    graphs, db, configs[lo:hi], graph_of[lo:hi], devs[k], keep_schedules, fused, streams,
                    index_base=lo)
                torch.cuda.current_stream(devs[k]).synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised on the caller's thread
            errors[k] = e

    threads = [threading.Thread(target=run, args=(k,), name=f"dfsim-shard-{devs[k]}") for k in range(W)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    fails = [(shards[k][0] + f[0], f[1]) for k, f in enumerate(failures) if f is not None]
    if fails:
        raise min(fails, key=lambda f: f[0])[1]
    out = _merge(results, shards, S)
    # K5 across devices: the winners (16 bytes each) peer-to-peer to devs[0], reduced there
    d0 = devs[0]
    recs = torch.stack([r.to(f"cuda:{d0}") for r in records])
    best = torch.empty(2, dtype=torch.float64, device=f"cuda:{d0}")
    with torch.cuda.device(d0):
        native.Context.get(d0).call("dfsim_argmin_records", W, native.ptr(recs), native.ptr(best))
    b = best.cpu()
    out.best_makespan = float(b[0].item())
    out.best_index = int(b[1:2].view(torch.int64).item()) if S else -1
    return out


def _sweep_distributed(graphs, db, configs, graph_of, devices, keep_schedules, fused, streams, group, gather_all,
                       rank, world, _local=None, _best=None) -> SweepResult:
    """One rank's part.  ``_local`` / ``_best`` replace the device steps (sweep_local and the
    NCCL winner reduction) in the CPU protocol tests (tests/test_distributed.py, gloo)."""
    import torch

    from .batch import gather_best

    if _local is None:
        device = (devices[0] if isinstance(devices, (list, tuple)) else devices) if devices is not None \
            else torch.cuda.current_device()
        with torch.cuda.device(device):
            return _sweep_distributed(graphs, db, configs, graph_of, devices, keep_schedules, fused, streams,
                                      group, gather_all, rank, world,
                                      _local=lambda c, gof, base: sweep_local(graphs, db, c, gof, device,
                                                                              keep_schedules, fused, streams,
                                                                              index_base=base),
                                      _best=gather_best)
    import torch.distributed as dist

    S = len(configs)
    shards = [shard(S, r, world) for r in range(world)]
    lo, hi = shards[rank]
    res, rec, failure = _local(configs[lo:hi], graph_of[lo:hi], lo)
    # every rank raises the same exception: the first failing config over all shards
    fails = [None] * world
    dist.all_gather_object(fails, (lo + failure[0], failure[1]) if failure is not None else None, group=group)
    fails = [f for f in fails if f is not None]
    if fails:
        raise min(fails, key=lambda f: f[0])[1]
    best = _best(rec, group).cpu()  # all-gather of 16-byte winners + k_argmin_records
    if gather_all:
        m = max(hi_ - lo_ for lo_, hi_ in shards)
        mine = torch.full((2, max(m, 1)), float("nan"), dtype=torch.float64, device=rec.device)
        mine[0, : hi - lo] = torch.from_numpy(res.makespan)
        mine[1, : hi - lo] = torch.from_numpy(res.cp_len)
        allv = torch.empty((world * 2, max(m, 1)), dtype=torch.float64, device=rec.device)
        dist.all_gather_into_tensor(allv, mine, group=group)
        allv = allv.reshape(world, 2, -1).cpu().numpy()
        full = [None] * world
        for r, (a, b) in enumerate(shards):
            part = SweepResult(allv[r, 0, : b - a], allv[r, 1, : b - a], -1, float("nan"))
            full[r] = part if r != rank else res
        out = _merge(full, shards, S)
    else:
        out = _merge([res if r == rank else None for r in range(world)], shards, S)
    out.best_makespan = float(best[0].item())
    out.best_index = int(best[1:2].view(torch.int64).item()) if S else -1
    return out
