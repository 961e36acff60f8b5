"""Batched strategy sweep: many candidate StrategyConfigs for one graph.

This replaces the reference's only many-strategies driver, ``dfsim simulate
--config A --config B ... --jobs J`` (cli.py:123-149), which runs
``_run_one_simulation`` (cli.py:71-116) once per config.  Here candidates are
grouped into topology classes (same expanded graph: replicas, device_map,
gradient markers, collective path -- strategy.py:202-252); each class is
expanded once on the GPU (K1), then all of its candidates go through
K2 estimate -> K3 simulate -> K4 critical path in single launches, and the best
candidate is the first minimum makespan (K5).  Multi-GPU: ``sweep_sharded``
splits the candidate list over ranks and all-gathers one 16-byte winner record
per rank over NCCL.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import CycleError
from .estimate import estimate_batch, raise_for_row
from .expansion import ExpansionPlan
from .lowering import LoweredGraph, LoweredProfiles, lowered
from .model import SOURCE_TAGS, DurationEntry
from .simulator import build_schedule, critical_path_arrays, simulate_arrays


def class_key(cfg) -> tuple:
    """Candidates with equal keys share one expanded graph (cli.py:83 decides expansion)."""
    if not (cfg.replicas > 1 or cfg.device_map):
        return ("plain",)
    return ("dp", cfg.replicas, tuple(cfg.device_map), tuple(cfg.gradient_markers), cfg.collective.path)


class TopologyClass:
    """One expanded graph resident on a device + profile tables for a candidate list."""

    def __init__(self, g, db, configs, device: int | None = None):
        ctx = native.Context.get(device)
        self.ctx = ctx
        cfg0 = configs[0]
        self.plan = None
        if class_key(cfg0) == ("plain",):
            self.graph = g
            self.lg: LoweredGraph = lowered(g, ctx.device)
        else:
            self.plan = ExpansionPlan(g, cfg0, ctx.device)
            self.graph, self.lg = self.plan.graph, self.plan.lowered
        self.ids = self.lg.ids
        self.configs = list(configs)
        self.lp = LoweredProfiles(self.graph, self.ids, db, self.configs, ctx.device)

    def expand(self):
        """Re-run K1 from the resident base arrays (the per-class device step)."""
        if self.plan is not None:
            self.plan.reexpand()

    def run(self, *, schedules: bool = True, paths: bool = False, out: dict | None = None,
            events: dict | None = None) -> dict:
        """K2 -> K3 -> K4 for every candidate; asynchronous on the current stream.

        ``events`` (optional): dict of stage name -> (start, end) torch.cuda.Event
        pairs recorded around "estimate", "simulate" and "critical_path".
        """
        o = out if out is not None else {}
        ev = events or {}

        def rec(name, i):
            if name in ev:
                ev[name][i].record()

        rec("estimate", 0)
        estimate_batch(self.lp, self.lg.n, out=o)
        rec("estimate", 1)
        rec("simulate", 0)
        simulate_arrays(self.lg, o["dur"], schedule=True, busy=True, out=o)
        rec("simulate", 1)
        rec("critical_path", 0)
        if self.lg.acyclic and self.lg.n:
            critical_path_arrays(self.lg, o["start"], o["finish"], paths=paths, out=o)
        rec("critical_path", 1)
        if not schedules:
            for k in ("start", "finish", "dur"):
                o.pop(k, None)
        return o

    def best(self, o: dict, index_base: int = 0, record=None):
        """K5 on this device: first minimum (makespan, index_base + row) -> 16-byte record."""
        import torch

        rec = record if record is not None else torch.empty(2, dtype=torch.float64, device=o["makespan"].device)
        self.ctx.call("dfsim_argmin", self.lp.n_sims, native.ptr(o["makespan"]), index_base, native.ptr(rec))
        return rec


@dataclass
class SweepResult:
    makespan: np.ndarray
    cp_len: np.ndarray
    best_index: int
    best_makespan: float
    classes: list = field(default_factory=list)   # (TopologyClass, config indices, outputs)
    _where: dict = field(default_factory=dict)    # config index -> (class position, row)

    def _row(self, i):
        c, row = self._where[i]
        tc, _, o = self.classes[c]
        if "start" not in o:
            raise ValueError("run sweep(..., keep_schedules=True) to rebuild schedules")
        return tc, o, row

    def schedule(self, i: int):
        """The reference Schedule object of candidate i."""
        tc, o, row = self._row(i)
        n = tc.lg.n
        src = o["src"][row, :n].cpu().numpy()
        dur = o["dur"][row, :n].cpu().numpy()
        entries = {nid: DurationEntry(float(dur[k]), SOURCE_TAGS[src[k]]) for k, nid in enumerate(tc.ids)}
        return build_schedule(tc.graph, tc.lg, o["start"][row, :n].cpu().numpy(), o["finish"][row, :n].cpu().numpy(),
                              float(o["makespan"][row].item()), o["busy"][row, : tc.lg.n_devices].cpu().numpy(),
                              entries)

    def critical_path(self, i: int):
        tc, o, row = self._row(i)
        p = critical_path_arrays(tc.lg, o["start"][row:row + 1], o["finish"][row:row + 1], paths=True)
        k = int(p["cp_path_len"][0].item())
        return float(p["cp_len"][0].item()), [tc.ids[j] for j in p["cp_path"][0, :k].cpu().tolist()]


def sweep(g, db, configs, device: int | None = None, keep_schedules: bool = False) -> SweepResult:
    """Evaluate every config like ``_run_one_simulation`` and pick the best.

    Errors follow the reference sweep: the first failing config (in list order)
    raises its UnknownOpError / ValueError / CycleError (cli.py:132-145).
    """
    import torch

    groups: dict = {}
    for i, cfg in enumerate(configs):
        groups.setdefault(class_key(cfg), []).append(i)
    S = len(configs)
    ctx = native.Context.get(device)
    dev = f"cuda:{ctx.device}"
    makespan = torch.full((max(S, 1),), float("inf"), dtype=torch.float64, device=dev)
    cp_len = torch.zeros(max(S, 1), dtype=torch.float64, device=dev)
    result = SweepResult(np.zeros(0), np.zeros(0), -1, float("nan"))
    failures = []
    for pos, (key, idx) in enumerate(groups.items()):
        tc = TopologyClass(g, db, [configs[i] for i in idx], ctx.device)
        o = tc.run(schedules=True)
        t_idx = torch.as_tensor(idx, dtype=torch.int64, device=dev)
        makespan.index_copy_(0, t_idx, o["makespan"])
        if "cp_len" in o:
            cp_len.index_copy_(0, t_idx, o["cp_len"])
        bad = o["bad"].cpu().numpy()
        placed = o["n_placed"].cpu().numpy()
        for row in np.nonzero((bad > 0) | (placed != tc.lg.n))[0].tolist():
            failures.append((idx[row], tc, o, row))
        if not keep_schedules:
            for k in ("start", "finish"):
                o.pop(k, None)
        result.classes.append((tc, idx, o))
        for row, i in enumerate(idx):
            result._where[i] = (pos, row)
    if failures:
        i, tc, o, row = min(failures, key=lambda f: f[0])
        n = tc.lg.n
        if int(o["bad"][row].item()):
            raise_for_row(tc.graph, tc.ids, o["dur"][row, :n].cpu().numpy(), o["src"][row, :n].cpu().numpy())
        st = o["start"][row, :n].cpu().numpy() if "start" in o else None
        raise CycleError(sorted(tc.ids[k] for k in np.nonzero(np.isnan(st))[0]) if st is not None else [])
    rec = torch.empty(2, dtype=torch.float64, device=dev)
    ctx.call("dfsim_argmin", S, native.ptr(makespan), 0, native.ptr(rec))
    r = rec.cpu()
    result.makespan = makespan[:S].cpu().numpy()
    result.cp_len = cp_len[:S].cpu().numpy()
    result.best_makespan = float(r[0].item())
    result.best_index = int(r[1:2].view(torch.int64).item()) if S else -1
    return result


def gather_best(record, group=None):
    """All-gather each rank's 16-byte (makespan, global index) winner over NCCL and
    reduce lexicographically on the device (K5's cross-GPU step)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    allrec = torch.empty(world * 2, dtype=torch.float64, device=record.device)
    dist.all_gather_into_tensor(allrec, record, group=group)
    out = torch.empty(2, dtype=torch.float64, device=record.device)
    ctx = native.Context.get(record.device.index)
    ctx.call("dfsim_argmin_records", world, native.ptr(allrec), native.ptr(out))
    return out
