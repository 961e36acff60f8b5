"""Batched strategy sweep: many candidate StrategyConfigs for one graph.

This replaces the reference's only many-strategies driver, ``dfsim simulate
--config A --config B ... --jobs J`` (cli.py:123-149), which runs
``_run_one_simulation`` (cli.py:71-116) once per config.  Here candidates are
grouped into topology classes (same expanded graph: replicas, device_map,
gradient markers, collective path -- strategy.py:202-252); each class is
expanded once on the GPU (K1), then all of its candidates go through
K2 estimate -> K3 simulate -> K4 critical path in single launches, and the best
candidate is the first minimum makespan (K5).  Multi-GPU: ``sharded.sweep_sharded``
splits the candidate list over GPUs (ranks of a process group, or devices of one
process) and reduces one 16-byte winner record per GPU (NCCL all-gather / P2P).
"""

from __future__ import annotations

import itertools
import operator
import os
import threading
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import CycleError, DfsimError, NativeError
from .estimate import estimate_batch, raise_for_row
from .expansion import ExpansionPlan
from .lowering import LoweredGraph, LoweredProfiles, lowered, resolve_overrides
from .model import SOURCE_TAGS, DurationEntry
from .prepare import ClassTables
from .simulator import build_schedule, critical_path_arrays, simulate_arrays


def class_key(cfg) -> tuple:
    """Candidates with equal keys share one expanded graph structure (cli.py:83 decides
    expansion).  The collective path is not part of the key: it names the devices an expansion
    adds and sets the PS links' attributes, but not the ids, the CSR or the device ranks --
    group_classes checks that per path (expansion.path_roles)."""
    if getattr(cfg, "sync", "allreduce") == "parameter_server":
        return ("ps", cfg.replicas, tuple(cfg.device_map), tuple(cfg.gradient_markers), cfg.ps_device)
    if not (cfg.replicas > 1 or cfg.device_map):
        return ("plain",)
    return ("dp", cfg.replicas, tuple(cfg.device_map), tuple(cfg.gradient_markers))


# class fields: (attribute, by value, default when absent -- the reference's own StrategyConfig
# has no PS extension fields; None: required)
_FIELDS = (("replicas", False, None), ("device_map", True, None), ("gradient_markers", True, None),
           ("collective.path", False, None), ("sync", False, "allreduce"), ("ps_device", False, "ps0"))


_COLLECTIVE = operator.attrgetter("collective")
# the fast path's fields (the whole collective: comparing one object is cheaper than a dotted get)
_CLASS_FIELDS = operator.attrgetter("replicas", "device_map", "gradient_markers", "collective", "sync", "ps_device")


def _column(configs, name, default) -> list:
    try:
        return list(map(operator.attrgetter(name), configs))
    except AttributeError:
        if default is None:
            raise
        return [getattr(c, name, default) for c in configs]


def _all_same(col) -> bool:
    """Every entry is the first one (identity; a C-level pass)."""
    return all(map(operator.is_, col, itertools.repeat(col[0]))) if col else True


def _value_codes(objs, key) -> list:
    """Small int per object, equal for equal ``key(obj)``: objects are deduplicated by identity
    first (sweeps usually share them), so each distinct object is keyed only once."""
    objs = list(objs)
    by_id = dict(zip(map(id, objs), objs))
    codes: dict = {}
    code_of = {i: codes.setdefault(key(o), len(codes)) for i, o in by_id.items()}
    return list(map(code_of.__getitem__, map(id, objs)))


def group_classes(graphs, configs, graph_of, db=None) -> list:
    """Config indices of each topology class, classes in order of first appearance.  A class
    is (class_key, structure of the candidate's graph, device roles of the expansion); keys
    are derived once per distinct field combination, not per candidate (sweeps hold 10^4-10^5
    configs)."""
    from .expansion import path_roles
    from .variants import structure_key

    # structures interned to small ints: equal structures compare in full once here, not at
    # every class-key lookup below
    canon: dict = {}
    skeys = {gi: canon.setdefault(structure_key(graphs[gi]), len(canon)) for gi in dict.fromkeys(graph_of)}
    if not configs:
        return []
    # field columns; a column whose objects are all one object (the common case: sweeps share
    # them) drops out after one identity pass, without hashing any value
    cols = []
    try:  # one pass when every class field is shared (equal tuples compare by identity first)
        t0 = _CLASS_FIELDS(configs[0])
        uniform = all(map(operator.eq, map(_CLASS_FIELDS, configs), itertools.repeat(t0)))
    except (AttributeError, TypeError, ValueError):  # missing PS fields; array-valued fields
        uniform = False
    for name, by_value, default in () if uniform else _FIELDS:
        col = _column(configs, name, default)
        if _all_same(col):
            continue
        if by_value:  # tuples by value (sweeps often build per-candidate objects), coded per object
            col = _value_codes(col, tuple)
        if len(dict.fromkeys(col)) > 1:
            cols.append(col)
    if not _all_same(graph_of) and len(dict.fromkeys(graph_of)) > 1:
        cols.append(list(graph_of))
    if not cols:
        return [list(range(len(configs)))]
    raw = list(zip(*cols))
    # first config of each distinct field combination (reversed: the smallest index is written last)
    first = dict(zip(reversed(raw), range(len(raw) - 1, -1, -1)))
    cls_of_key: dict = {}
    roles: dict = {}

    def key_of(i):
        cfg, gi = configs[i], graph_of[i]
        k = class_key(cfg)
        if k == ("plain",):
            return k, skeys[gi], None
        rk = (k, skeys[gi], cfg.collective.path)  # graph variants of one structure share their roles
        if rk not in roles:  # None (expansion would fail): a class of its own per path
            roles[rk] = path_roles(graphs[gi], cfg, db) or ("\x00fails", cfg.collective.path)
        return k, skeys[gi], roles[rk]

    cls_of_raw = {r: cls_of_key.setdefault(key_of(i), len(cls_of_key)) for r, i in first.items()}
    cls = np.fromiter(map(cls_of_raw.__getitem__, raw), np.int64, len(raw))
    order = np.argsort(cls, kind="stable")  # config order inside each class
    cuts = np.flatnonzero(np.diff(cls[order])) + 1
    groups = np.split(order, cuts) if len(order) else []
    groups.sort(key=lambda g: int(g[0]))  # classes in order of first appearance
    return [g.tolist() for g in groups]


class TopologyClass:
    """One expanded graph resident on a device + profile tables for a candidate list.

    ``fused=True`` (default) runs the fused hot path -- K2a variant resolve,
    K3 v2 engine with on-the-fly durations, K4 v2 level-order critical path --
    whenever the class fits it (prepare.ClassTables.fused_ok) and every variant
    resolves without errors; otherwise the unfused K2 -> K3 -> K4 path runs,
    which also produces the reference's exact error for failing candidates.
    """

    def __init__(self, g, db, configs, device: int | None = None, fused: bool = True, graphs=None,
                 graph_of=None, fit_cache=None):
        ctx = native.Context.get(device)
        self.ctx = ctx
        cfg0 = configs[0]
        self.plan = None
        key = class_key(cfg0)
        if graphs is not None:
            g = graphs[graph_of[0]]
        self._graph = None
        if key == ("plain",):
            kind, self._graph = "plain", g
            self.lg: LoweredGraph = lowered(g, ctx.device)
            structure = None
        else:  # K1 on the device: data-parallel allreduce, or the parameter-server expansion (ps.py)
            kind = "ps" if key[0] == "ps" else "dp"
            self.plan = structure = ExpansionPlan(g, cfg0, ctx.device, build_objects=False, db=db)
            self.lg = self.plan.lowered
        self.ids = self.lg.ids
        self.configs = list(configs)
        variant_rows, strat_gv = None, None
        one_graph = graphs is None or _all_same(graph_of) or len(dict.fromkeys(graph_of)) == 1
        multi = not one_graph
        self._db = db
        self._path_objects = {}  # path -> (graph objects, device names) of the other paths in the class
        if multi or kind != "plain":
            # estimate inputs from the base graph(s): a clone's row is its base node's, so features
            # are computed once per base node and collective / PS node, not per expanded node
            from .variants import variant_arrays_many

            if graphs is None:
                graphs, graph_of = [g], [0] * len(configs)
            if one_graph and (kind != "ps" or _all_same(list(map(_COLLECTIVE, configs)))):
                vkeys = None  # one variant (the common case): no per-candidate keys
            elif kind == "ps":  # the PS links' attributes depend on the path: a variant per (graph, path)
                paths = [c.collective.path for c in configs]
                vkeys = list(zip(graph_of, paths))
            else:
                vkeys = list(graph_of)
            if vkeys is None:
                vk0 = (graph_of[0], cfg0.collective.path) if kind == "ps" else graph_of[0]
                gv_of, first_cfg = {vk0: 0}, {vk0: cfg0}
                strat_gv = np.zeros(len(configs), np.int32)
            else:
                gv_of = {vk: k for k, vk in enumerate(dict.fromkeys(vkeys))}
                first_i = dict(zip(reversed(vkeys), range(len(vkeys) - 1, -1, -1)))  # first config of each key
                first_cfg = {vk: configs[i] for vk, i in first_i.items()}
                strat_gv = np.fromiter(map(gv_of.__getitem__, vkeys), np.int32, len(vkeys))
            variant_rows = variant_arrays_many(kind, self.ids, [graphs[vk[0] if kind == "ps" else vk] for vk in gv_of],
                                               structure, cfg0, db, cfgs=[first_cfg[vk] for vk in gv_of])
        self.lp = LoweredProfiles(g if self.plan is not None else self.graph, self.ids, db, self.configs,
                                  ctx.device, None, strat_gv, fit_cache=fit_cache, variant_arrays=variant_rows,
                                  op_kind=self.plan.op_kind() if self.plan is not None else None)
        self.tables = None
        self.fused = False
        if fused and self.lg.acyclic and 0 < self.lg.n <= 65535 and self.lp.fused_values_ok:
            self.tables = ClassTables(self.lg, n_sims=len(configs))
            if self.tables.fused_ok:
                self._prepare_variants()

    @property
    def graph(self):
        """The class's expanded graph objects (built on first use for expanded classes)."""
        return self._graph if self.plan is None else self.plan.graph

    def objects_for(self, row: int):
        """(graph objects, device names by rank) of candidate ``row``: the class's own for its
        first config's collective path; for another path of the class (group_classes), the
        host objects of that path's expansion (same ids and ranks, its own device names)."""
        path = self.configs[row].collective.path if self.plan is not None else None
        if self.plan is None or path == self.plan.cfg.collective.path:
            return self.graph, self.lg.devices
        got = self._path_objects.get(path)
        if got is None:
            cfg = self.configs[row]
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                plan = ExpansionPlan(self.plan._g, cfg, run_k1=False, build_objects=False, db=self._db)
            if plan.ids != self.ids or len(plan.devices) != len(self.lg.devices):
                raise DfsimError("internal: paths of one topology class expand differently")
            got = self._path_objects[path] = (plan.graph, plan.devices)
        return got

    # ------------------------------------------------------------------ fused path
    def _prepare_variants(self):
        import torch

        lp, N = self.lp, self.lg.n
        # variant = (graph variant, hardware, algorithm, path): one int64 key per candidate
        cols = [np.asarray(c, np.int64) for c in (lp.strat_gv, lp.strat_hw, lp.strat_algo, lp.strat_path)]
        span = [int(c.max(initial=0)) + 1 for c in cols]
        key = ((cols[0] * span[1] + cols[1]) * span[2] + cols[2]) * span[3] + cols[3]
        uniq, var_of = np.unique(key, return_inverse=True)
        var_of = var_of.astype(np.int64)
        V = len(uniq)
        dev = f"cuda:{self.ctx.device}"
        u_path, rest = uniq % span[3], uniq // span[3]
        u_algo, rest = rest % span[2], rest // span[2]
        u_hw, u_gv = rest % span[1], rest // span[1]
        self.v_gv = torch.as_tensor(u_gv, dtype=torch.int32, device=dev)
        self.v_hw = torch.as_tensor(u_hw, dtype=torch.int32, device=dev)
        self.v_algo = torch.as_tensor(u_algo, dtype=torch.uint8, device=dev)
        self.v_path = torch.as_tensor(u_path, dtype=torch.int32, device=dev)
        self.n_variants = V
        self.var_of = var_of
        self.base = torch.empty((V, N), dtype=torch.float64, device=dev)
        self.status = torch.empty((V, N), dtype=torch.uint8, device=dev)
        self.resolve()
        st = self.status.cpu().numpy()
        if (st >= 253).any():
            return  # some candidate fails estimation: keep the unfused path (exact error semantics)
        cap = int(self.ctx.lib.dfsim_fused_capacity(native.ctypes.byref(self.tables.sim_struct)))
        cp_ok = (self.tables.lane is not None
                 or (self.tables.cp_struct is not None and self.ctx.lib.dfsim_critical_path_levels_capacity(
                     native.ctypes.byref(self.tables.cp_struct)) > 0))
        if cap <= 0 or not cp_ok:
            return  # engine or critical-path tables exceed shared memory: rank-layout kernels
        self.chunk_capacity = cap
        # a small class is cut into smaller chunks so that its CTAs cover the SMs (the
        # launcher sizes CTAs to the largest chunk)
        sms = torch.cuda.get_device_properties(self.ctx.device).multi_processor_count
        cap = int(self.ctx.lib.dfsim_fused_chunk(native.ctypes.byref(self.tables.sim_struct), lp.n_sims, sms))
        if os.environ.get("DFSIM_FUSED_CHUNK"):  # measurement knob: fixed chunk (clamped to the capacity)
            cap = max(1, min(self.chunk_capacity, int(os.environ["DFSIM_FUSED_CHUNK"])))
        # candidates with manual overrides: when the (variant, override set) combinations are few
        # enough to fill warps (>= 32 candidates each on average), each gets its own duration row
        # (dfsim_override_rows) and the engine never searches an override table; otherwise
        # the engine looks overrides up per popped node (skipping nodes in no set)
        row_of, self.combo = var_of, None
        ovs = np.asarray(lp.strat_ov, np.int64)
        if ovs.size and ovs.max() >= 0:
            n_sets = int(ovs.max()) + 1
            ck = var_of * (n_sets + 1) + (ovs + 1)
            cuniq, combo_of = np.unique(ck, return_inverse=True)
            C = len(cuniq)
            if C * 32 <= lp.n_sims and C * N * 8 <= (1 << 30) and not os.environ.get("DFSIM_OV_SEARCH_ALL"):
                self.combo = (torch.as_tensor(cuniq // (n_sets + 1), dtype=torch.int32, device=dev),
                              torch.as_tensor(cuniq % (n_sets + 1) - 1, dtype=torch.int32, device=dev),
                              torch.empty((C, N), dtype=torch.float64, device=dev))
                row_of = combo_of.astype(np.int64)
                self.resolve()
        order = np.argsort(row_of, kind="stable")
        firsts, counts, variants = [], [], []
        sorted_var = row_of[order]
        bounds = np.flatnonzero(np.diff(sorted_var)) + 1
        for a, b in zip(np.r_[0, bounds], np.r_[bounds, len(order)]):
            for c in range(a, b, cap):  # full chunks (whole warps), then the variant's remainder
                firsts.append(int(c))
                counts.append(int(min(cap, b - c)))
                variants.append(int(sorted_var[a]))
        T = lambda x, dt: torch.as_tensor(np.asarray(x), dtype=dt, device=dev)  # noqa: E731
        self.f_order = T(order, torch.int64)  # slot k of the tiled schedules holds candidate order[k]
        # K4 v3 (lane = candidate) reads tiles of 32 candidates, one coalesced run per position;
        # K4 v2 (a half-warp per candidate, consecutive positions) reads rows
        self.tiled = self.tables.lane is not None
        self.slot_of = np.empty(len(order), np.int64)
        self.slot_of[order] = np.arange(len(order))
        self.f_first, self.f_count, self.f_var = T(firsts, torch.int32), T(counts, torch.int32), T(variants, torch.int32)
        t, s = lp.tensors, lp.t_strat
        rows = self.combo[2] if self.combo is not None else self.base
        self.fused_strat = native.FusedStrategies(
            lp.n_sims, rows.shape[0], native.ptr(rows), len(firsts), native.ptr(self.f_order), native.ptr(self.f_first),
            native.ptr(self.f_count), native.ptr(self.f_var), native.ptr(s["gap"]),
            native.ptr(s["ov"]) if self.combo is None and lp.strat_ov.size and lp.strat_ov.max() >= 0 else native.P(0),
            native.ptr(t["ooff"]), native.ptr(t["onode"]), native.ptr(t["oval"]), max(counts, default=0),
            native.P(0) if os.environ.get("DFSIM_OV_SEARCH_ALL") else native.ptr(t["oany"]), int(self.tiled))
        self.fused = True

    def resolve(self):
        """K2a: estimate every node once per (hardware, algorithm, path) variant (and stamp the
        override sets into the (variant, set) rows when the class uses them)."""
        self.ctx.call("dfsim_resolve_variants", self.lg.n, native.ctypes.byref(self.lp.struct), self.n_variants,
                      native.ptr(self.v_hw), native.ptr(self.v_algo), native.ptr(self.v_path),
                      native.ptr(self.v_gv), native.ptr(self.base), native.ptr(self.status))
        if getattr(self, "combo", None) is not None:
            c_var, c_set, rows = self.combo
            t = self.lp.tensors
            self.ctx.call("dfsim_override_rows", self.lg.n, rows.shape[0], native.ptr(self.base), native.ptr(c_var),
                          native.ptr(c_set), native.ptr(t["ooff"]), native.ptr(t["onode"]), native.ptr(t["oval"]),
                          native.ptr(rows))

    def fallback_if_needed(self, o) -> bool:
        """Re-run ring-overflow candidates on the exact engine (host sync on the flags).
        Returns True when some candidate was re-run (its critical path must then be redone)."""
        import torch

        if not self.fused:
            return False
        flagged = torch.nonzero(o["flags"]).flatten()
        if flagged.numel():
            self._fallback(o, flagged.cpu().tolist())
            return True
        return False

    def _fallback(self, o, rows):
        """Exact engine for candidates whose FIFO ring overflowed (never changes results)."""
        import torch

        dev = o["makespan"].device
        idx = torch.as_tensor(rows, dtype=torch.int64, device=dev)
        s = self.lp.t_strat
        sub = {k: v.index_select(0, idx).contiguous() for k, v in s.items()}
        strat = native.Strategies(len(rows), native.ptr(sub["hw"]), native.ptr(sub["gap"]), native.ptr(sub["algo"]),
                                  native.ptr(sub["path"]), native.ptr(sub["ov"]), native.ptr(sub["gv"]))
        N = self.lg.n
        dur = torch.empty((len(rows), N), dtype=torch.float64, device=dev)
        src = torch.empty((len(rows), N), dtype=torch.uint8, device=dev)
        bad = torch.empty(len(rows), dtype=torch.int32, device=dev)
        self.ctx.call("dfsim_estimate_batch", N, native.ctypes.byref(self.lp.struct), native.ctypes.byref(strat),
                      native.ptr(dur), native.ptr(src), native.ptr(bad))
        # the exact engine writes the re-run rows' pairs by position into a scratch block, then
        # they go to the candidates' slots of the tiled schedule (a rare path)
        R = len(rows)
        pairs = torch.empty((R, N, 2), dtype=torch.float64, device=dev)
        D = o["busy"].shape[1]
        ms, busy, placed = (torch.empty(R, dtype=torch.float64, device=dev),
                            torch.empty((R, D), dtype=torch.float64, device=dev),
                            torch.empty(R, dtype=torch.int32, device=dev))
        self.ctx.call("dfsim_simulate_batch_ex", native.ctypes.byref(self.lg.struct), R, native.ptr(dur), N,
                      native.ptr(pairs), native.P(0), native.ptr(ms), native.ptr(busy), native.ptr(placed),
                      native.ptr(self.tables.t["pos32"]), native.P(0), 1)
        if self.tiled:
            slots = torch.as_tensor(self.slot_of[np.asarray(rows, np.int64)], dtype=torch.int64, device=dev)
            o["sched"][slots // 32, :N, slots % 32, :] = pairs
        else:
            o["sched"][idx] = pairs
        o["makespan"][idx] = ms
        o["busy"][idx] = busy
        o["n_placed"][idx] = placed
        o.setdefault("fallback_rows", []).extend(int(r) for r in rows)

    def run_fused(self, o: dict, ev: dict, paths: bool = False, defer_fallback: bool = False):
        import torch

        lg, S, N, D = self.lg, self.lp.n_sims, self.lg.n, self.lg.n_devices
        dev = f"cuda:{self.ctx.device}"
        if "sched" not in o:  # callers may pre-place any output (e.g. flags as a view of a shared buffer)
            # (start, finish) pairs by position: 32-candidate tiles (K4 v3) or rows (dfsim_simulate_fused)
            o["sched"] = (torch.empty(((S + 31) // 32, N, 32, 2), dtype=torch.float64, device=dev) if self.tiled
                          else torch.empty((S, N, 2), dtype=torch.float64, device=dev))
            o.setdefault("makespan", torch.empty(S, dtype=torch.float64, device=dev))
            o.setdefault("busy", torch.empty((S, max(D, 1)), dtype=torch.float64, device=dev))
            o.setdefault("n_placed", torch.empty(S, dtype=torch.int32, device=dev))
            o.setdefault("flags", torch.empty(S, dtype=torch.int32, device=dev))
            o.setdefault("cp_len", torch.empty(S, dtype=torch.float64, device=dev))
            o.setdefault("cp_src", torch.empty(S, dtype=torch.int32, device=dev))
            o.setdefault("bad", torch.zeros(S, dtype=torch.int32, device=dev))
        o["layout"] = "position"
        rec = lambda name, i: ev[name][i].record() if name in ev else None  # noqa: E731
        rec("estimate", 0)
        self.resolve()
        rec("estimate", 1)
        rec("simulate", 0)
        self.ctx.call("dfsim_simulate_fused", native.ctypes.byref(self.tables.sim_struct),
                      native.ctypes.byref(self.fused_strat), native.ptr(o["sched"]),
                      native.ptr(o["makespan"]), native.ptr(o["busy"]), native.ptr(o["n_placed"]),
                      native.ptr(o["flags"]))
        rec("simulate", 1)
        if not defer_fallback:
            self.fallback_if_needed(o)
        rec("critical_path", 0)
        self.tables.critical_path(S, o["sched"], o["cp_len"], o["cp_src"], self.f_order if self.tiled else None)
        rec("critical_path", 1)
        return o

    def expand(self):
        """Re-run K1 from the resident base arrays (the per-class device step)."""
        if self.plan is not None:
            self.plan.reexpand(topo=not self.fused)

    def run(self, *, schedules: bool = True, paths: bool = False, out: dict | None = None,
            events: dict | None = None, defer_fallback: bool = False) -> dict:
        """K2 -> K3 -> K4 for every candidate; asynchronous on the current stream.

        ``events`` (optional): dict of stage name -> (start, end) torch.cuda.Event
        pairs recorded around "estimate", "simulate" and "critical_path".
        """
        o = out if out is not None else {}
        ev = events or {}
        if self.fused:
            self.run_fused(o, ev, defer_fallback=defer_fallback)
        else:
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
            o["layout"] = "rank"
        if not schedules:
            for k in ("start", "finish", "sched", "dur"):
                o.pop(k, None)
        return o

    def rows_by_position(self, o: dict, rows):
        """(start, finish) of candidates ``rows`` as [R, N] device tensors by level position
        (fused layouts: gathered from the 32-candidate tiles) or by rank (unfused)."""
        import torch

        n = self.lg.n
        r = torch.as_tensor(list(rows), dtype=torch.int64, device=o["makespan"].device)
        if o.get("layout") == "position" and self.tiled:  # the candidates' slots in the engine's tiles
            k = torch.as_tensor(self.slot_of[np.asarray(list(rows), np.int64)], device=r.device)
            pairs = o["sched"][k // 32, :, k % 32, :]  # [R, N, 2]
            return pairs[:, :n, 0], pairs[:, :n, 1]
        if o.get("layout") == "position":
            pairs = o["sched"].index_select(0, r)
            return pairs[:, :n, 0], pairs[:, :n, 1]
        return o["start"].index_select(0, r)[:, :n], o["finish"].index_select(0, r)[:, :n]

    def rows_by_rank_batch(self, o: dict, rows):
        """(start, finish) of several candidates as contiguous [R][N] device tensors by node rank."""
        import torch

        st, fi = self.rows_by_position(o, rows)
        if o.get("layout") == "position":
            pos = torch.as_tensor(self.tables.pos, device=st.device)
            st, fi = st.index_select(1, pos), fi.index_select(1, pos)
        return st.contiguous(), fi.contiguous()

    def rows_by_rank(self, o: dict, row: int):
        """(start, finish) of one candidate as device tensors in node-rank order."""
        st, fi = self.rows_by_rank_batch(o, [row])
        return st[0], fi[0]

    def summary_tables(self):
        """K6 tables of this class (cached): op key, comm flag and (device, id) order per node rank."""
        if getattr(self, "_summary", None) is None:
            from .model import DEVICE_COMPUTE
            from .reporting import SummaryTables

            g = self.graph
            kinds = {d: spec.kind for d, spec in g.devices.items()}
            keys = [g.nodes[nid].op_type or nid for nid in self.ids]
            comm = [kinds.get(g.nodes[nid].device, DEVICE_COMPUTE) != DEVICE_COMPUTE for nid in self.ids]
            self._summary = SummaryTables(keys, comm, self.lg.device_of_rank(), self.ctx.device)
        return self._summary

    def critical_path_only(self, o: dict):
        """Re-run K4 on the current schedules (after a deferred fallback): only the re-run
        candidates when K4 v3 can take a candidate list."""
        if self.fused:
            rows = o.get("fallback_rows")
            self.tables.critical_path(self.lp.n_sims, o["sched"], o["cp_len"], o["cp_src"],
                                      self.f_order if self.tiled else None,
                                      slots=(self.slot_of if self.tiled else np.arange(self.lp.n_sims))[
                                          np.asarray(rows, np.int64)] if rows else None)
        elif self.lg.acyclic and self.lg.n:
            critical_path_arrays(self.lg, o["start"], o["finish"], out=o)

    def best(self, o: dict, index_base: int = 0, record=None):
        """K5 on this device: first minimum (makespan, index_base + row) -> 16-byte record."""
        import torch

        rec = record if record is not None else torch.empty(2, dtype=torch.float64, device=o["makespan"].device)
        self.ctx.call("dfsim_argmin", self.lp.n_sims, native.ptr(o["makespan"]), index_base, native.ptr(rec))
        return rec


class _Where:
    """config index -> (class position, row) over two arrays (sweeps hold 10^4-10^5 configs)."""

    def __init__(self, cls, row):
        self.cls, self.row = cls, row

    def __getitem__(self, i):
        c = int(self.cls[i])
        if c < 0:
            raise KeyError(i)
        return c, int(self.row[i])

    def items(self):
        for i in np.flatnonzero(self.cls >= 0).tolist():
            yield i, (int(self.cls[i]), int(self.row[i]))


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
        if "sched" not in o and "start" not in o:
            raise ValueError("run sweep(..., keep_schedules=True) to rebuild schedules")
        return tc, o, row

    def schedule(self, i: int):
        """The reference Schedule object of candidate i."""
        tc, o, row = self._row(i)
        st, fi = tc.rows_by_rank(o, row)
        entries = self._entries(tc, o, row)
        g, devices = tc.objects_for(row)
        return build_schedule(g, tc.lg, st.cpu().numpy(), fi.cpu().numpy(),
                              float(o["makespan"][row].item()), o["busy"][row, : tc.lg.n_devices].cpu().numpy(),
                              entries, devices=devices)

    def _entries(self, tc, o, row):
        """Duration source tags of one candidate (the fused path keeps per-variant tags)."""
        n = tc.lg.n
        if "src" in o:
            src = o["src"][row, :n].cpu().numpy()
        else:
            src = tc.status[int(tc.var_of[row])].cpu().numpy().copy()
            cfg = tc.configs[row]
            if cfg.overrides:
                rank = tc.lg.rank_of()
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    for nid in resolve_overrides(cfg.overrides, tc.ids):
                        src[rank[nid]] = 0
        return {nid: DurationEntry(0.0, SOURCE_TAGS[src[k]]) for k, nid in enumerate(tc.ids)}

    def summaries(self, indices, top_k: int = 10) -> list:
        """reporting.summarize (reporting.py:117-162) of several candidates' schedules, computed
        from the schedules still in HBM: K6 folds + K4 paths on the device, one launch
        sequence per topology class.  Returns SummaryReport objects in ``indices`` order."""
        from .reporting import SummaryReport, rank_ops, run_summary

        indices = list(indices)
        out = [None] * len(indices)
        by_class: dict = {}
        for k, i in enumerate(indices):
            c, row = self._where[i]
            by_class.setdefault(c, []).append((k, row))
        for c, items in by_class.items():
            tc, _, o = self.classes[c]
            if "sched" not in o and "start" not in o:
                raise ValueError("run sweep(..., keep_schedules=True) to summarise schedules")
            rows = [row for _, row in items]
            st, fi = tc.rows_by_rank_batch(o, rows)
            tables = tc.summary_tables()
            order, key_total, key_first, sums = run_summary(tc.ctx, tables, st, fi)
            p = critical_path_arrays(tc.lg, st, fi, paths=True) if tc.lg.n else None
            lg = tc.lg
            kt, kf, sm = key_total.cpu().numpy(), key_first.cpu().numpy(), sums.cpu().numpy()
            ms = o["makespan"].cpu().numpy()
            busy_rows = o["busy"].cpu().numpy()
            order_h = order.cpu().numpy()
            cp_len = p["cp_len"].cpu().numpy() if p else None
            cp_path = p["cp_path"].cpu().numpy() if p else None
            cp_plen = p["cp_path_len"].cpu().numpy() if p else None
            dev_of = lg.device_of_rank()
            for j, (k, row) in enumerate(items):
                g, devices = tc.objects_for(row)
                kinds = {d: spec.kind for d, spec in g.devices.items()}
                extra = [d for d in devices if d not in g.devices]
                busy = {d: 0.0 for d in g.devices}
                rank_busy = {devices[r]: float(busy_rows[row, r]) for r in range(lg.n_devices)}
                for d in g.devices:
                    if d in rank_busy:
                        busy[d] = rank_busy[d]
                if extra:  # devices outside g.devices join in entry order (engine.py:90-92)
                    for v in order_h[j, : lg.n].tolist():
                        d = devices[dev_of[v]]
                        if d not in busy:
                            busy[d] = rank_busy[d]
                makespan = float(ms[row])
                util = {d: (b / makespan if makespan > 0 else 0.0) for d, b in busy.items()}
                path = [tc.ids[v] for v in cp_path[j, : int(cp_plen[j])].tolist()] if p else []
                out[k] = SummaryReport(
                    makespan_us=makespan, per_device_busy_us=busy, utilization=util, device_kinds=dict(kinds),
                    top_k_ops=rank_ops(tables.keys, kt[j], kf[j], top_k) if lg.n else [],
                    compute_us=float(sm[j, 0]), comm_us=float(sm[j, 1]), overlap_us=float(sm[j, 2]),
                    critical_path_nodes=path, critical_path_us=float(cp_len[j]) if p else 0.0)
        return out

    def summary(self, i: int, top_k: int = 10):
        return self.summaries([i], top_k)[0]

    def trace(self, i: int) -> str:
        """reporting.to_trace of candidate i's schedule (byte-identical; C++ writer)."""
        from .reporting import TraceTables, run_summary

        tc, o, row = self._row(i)
        st, fi = tc.rows_by_rank_batch(o, [row])
        order, _, _, _ = run_summary(tc.ctx, tc.summary_tables(), st, fi)
        lg = tc.lg
        g, devices = tc.objects_for(row)
        cache = tc.__dict__.setdefault("_trace_tables", {})  # per collective path (device names)
        tt = cache.get(id(devices))
        if tt is None:
            tracks = sorted(set(g.devices) | set(devices))
            tid = {d: k for k, d in enumerate(tracks)}
            tt = cache[id(devices)] = TraceTables(tc.ids, [g.nodes[nid].op_type or nid for nid in tc.ids],
                                                  np.zeros(lg.n, np.uint8),
                                                  [tid[devices[d]] for d in lg.device_of_rank()], tracks)
        src = self._entries(tc, o, row)
        tags = np.fromiter((SOURCE_TAGS.index(src[nid].source) for nid in tc.ids), dtype=np.uint8, count=lg.n)
        return tt.write(order.cpu().numpy()[0, : lg.n], st.cpu().numpy()[0], fi.cpu().numpy()[0], tags=tags)

    def critical_path(self, i: int):
        tc, o, row = self._row(i)
        st, fi = tc.rows_by_rank(o, row)
        p = critical_path_arrays(tc.lg, st.reshape(1, -1).contiguous(), fi.reshape(1, -1).contiguous(), paths=True)
        k = int(p["cp_path_len"][0].item())
        return float(p["cp_len"][0].item()), [tc.ids[j] for j in p["cp_path"][0, :k].cpu().tolist()]


def sweep(g, db, configs, device: int | None = None, keep_schedules: bool = False,
          fused: bool = True) -> SweepResult:
    """Evaluate every config like ``_run_one_simulation`` and pick the best.

    Errors follow the reference sweep: the first failing config (in list order)
    raises its UnknownOpError / ValueError / CycleError (cli.py:132-145).
    """
    return sweep_variants([g], db, configs, [0] * len(configs), device, keep_schedules, fused)


def sweep_variants(graphs, db, configs, graph_of, device: int | None = None, keep_schedules: bool = False,
                   fused: bool = True, streams: int = 32) -> SweepResult:
    """``sweep`` where candidate i runs ``configs[i]`` on ``graphs[graph_of[i]]`` (e.g. one graph per
    batch size).  Graphs of identical structure share a topology class (variants.py).

    Classes are launched round-robin on up to ``streams`` CUDA streams (each stream has its
    own device scratch in the context), so many small classes share the GPU."""
    result, _, failure = sweep_local(graphs, db, configs, graph_of, device, keep_schedules, fused, streams)
    if failure is not None:
        raise failure[1]
    return result


def _row_error(tc, o, row) -> Exception:
    """The reference's exception for a failed candidate row (estimation error or cycle)."""
    n = tc.lg.n
    if int(o["bad"][row].item()):
        try:
            raise_for_row(tc.graph, tc.ids, o["dur"][row, :n].cpu().numpy(), o["src"][row, :n].cpu().numpy())
        except Exception as e:  # noqa: BLE001 -- returned, raised by the caller
            return e
    if "sched" not in o and "start" not in o:
        return CycleError([])
    st = tc.rows_by_rank(o, row)[0].cpu().numpy() if tc.fused else o["start"][row, :n].cpu().numpy()
    return CycleError(sorted(tc.ids[k] for k in np.nonzero(np.isnan(st))[0]))


_STREAMS: dict = {}
_STREAMS_LOCK = threading.Lock()


def _side_streams(device: int, n: int) -> list:
    """n class streams of ``device``, the same ones on every call: PyTorch caches freed device
    blocks per stream and the library keeps device scratch per (context, stream), so fresh
    streams per sweep would allocate afresh every time (and grow the scratch list)."""
    import torch

    with _STREAMS_LOCK:
        have = _STREAMS.setdefault(device, [])
        while len(have) < n:
            have.append(torch.cuda.Stream(device))
        return have[:n]


def sweep_local(graphs, db, configs, graph_of, device: int | None = None, keep_schedules: bool = False,
                fused: bool = True, streams: int = 32, index_base: int = 0):
    """The per-device body of every sweep: returns ``(result, record, failure)`` without raising.

    ``record`` is K5's 16-byte winner ``(makespan, index_base + first minimum row)`` on the
    device (for a cross-GPU reduction); ``failure`` is ``(local index, exception)`` of the first
    failing config in list order (cli.py:132-145) or None.  ``result.best_*`` are this shard's."""
    import torch

    groups = group_classes(graphs, configs, graph_of, db)
    S = len(configs)
    ctx = native.Context.get(device)
    dev = f"cuda:{ctx.device}"
    makespan = torch.full((max(S, 1),), float("inf"), dtype=torch.float64, device=dev)
    cp_len = torch.zeros(max(S, 1), dtype=torch.float64, device=dev)
    result = SweepResult(np.zeros(0), np.zeros(0), -1, float("nan"))
    failures = []  # (config index, exception)
    where_cls, where_row = np.full(S, -1, np.int32), np.zeros(S, np.int32)
    result._where = _Where(where_cls, where_row)
    built = []
    fits: dict = {}  # fitted models shared by the classes of this sweep (costmodel.py:313-316 fits per call)
    for idx in groups:
        whole = len(idx) == S  # one class (idx == range(S)): no per-candidate gathers
        try:
            built.append((idx, TopologyClass(graphs[graph_of[idx[0]]], db, configs if whole else [configs[i] for i in idx],
                                             ctx.device, fused=fused, graphs=graphs,
                                             graph_of=graph_of if whole else [graph_of[i] for i in idx],
                                             fit_cache=fits)))
        except NativeError:
            raise
        except Exception as e:  # noqa: BLE001 -- expansion / lowering error: the class's first config fails
            failures.append((idx[0], e))
    built.sort(key=lambda b: -b[1].lg.n * len(b[0]))  # most work first: the longest CTAs must not form the tail
    outs = [{} for _ in built]
    side = _side_streams(ctx.device, min(max(streams, 1), len(built))) if len(built) > 1 else []
    cur = torch.cuda.current_stream(ctx.device)
    for st in side:
        st.wait_stream(cur)
    for k, ((idx, tc), o) in enumerate(zip(built, outs)):
        if side:
            with torch.cuda.stream(side[k % len(side)]):
                tc.run(schedules=True, out=o, defer_fallback=True)
        else:
            tc.run(schedules=True, out=o, defer_fallback=True)
    for st in side:
        cur.wait_stream(st)
    fused_flags = [o["flags"].any() for (_, tc), o in zip(built, outs) if tc.fused]
    if fused_flags and bool(torch.stack(fused_flags).any()):  # one host check for every class
        for (idx, tc), o in zip(built, outs):  # exact re-run of ring overflows, then their critical paths
            if tc.fallback_if_needed(o):
                tc.critical_path_only(o)
    for pos, ((idx, tc), o) in enumerate(zip(built, outs)):
        lo = idx[0]
        if idx[-1] - lo + 1 == len(idx):  # a contiguous run of candidates (indices ascend in a class)
            makespan[lo:lo + len(idx)].copy_(o["makespan"])
            if "cp_len" in o:
                cp_len[lo:lo + len(idx)].copy_(o["cp_len"])
        else:
            t_idx = torch.as_tensor(idx, dtype=torch.int64, device=dev)
            makespan.index_copy_(0, t_idx, o["makespan"])
            if "cp_len" in o:
                cp_len.index_copy_(0, t_idx, o["cp_len"])
        bad = o["bad"].cpu().numpy()
        placed = o["n_placed"].cpu().numpy()
        rows = np.nonzero((bad > 0) | (placed != tc.lg.n))[0]
        if rows.size:  # this class's first failing row, while its schedules are still here
            row = int(rows[0])
            failures.append((idx[row], _row_error(tc, o, row)))
        if not keep_schedules:
            for k in ("start", "finish", "sched"):
                o.pop(k, None)
        result.classes.append((tc, idx, o))
        ia = slice(lo, lo + len(idx)) if idx[-1] - lo + 1 == len(idx) else np.asarray(idx, np.int64)
        where_cls[ia] = pos
        where_row[ia] = np.arange(len(idx), dtype=np.int32)
    failure = min(failures, key=lambda f: f[0]) if failures else None
    rec = torch.empty(2, dtype=torch.float64, device=dev)
    ctx.call("dfsim_argmin", S, native.ptr(makespan), index_base, native.ptr(rec))
    result.makespan = makespan[:S].cpu().numpy()
    result.cp_len = cp_len[:S].cpu().numpy()
    r = rec.cpu()
    result.best_makespan = float(r[0].item())
    result.best_index = int(r[1:2].view(torch.int64).item()) if S else -1
    return result, rec, failure


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous candidate slice [lo, hi) of one rank (no data-path collective)."""
    lo = total * rank // world
    return lo, total * (rank + 1) // world


def exchange_winners(record, group=None):
    """All-gather every rank's 16-byte winner (makespan f64, global index i64 bits) ->
    [world, 2] f64.  NCCL over NVLink for CUDA tensors, gloo for CPU tensors."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty(world * 2, dtype=torch.float64, device=record.device)
    dist.all_gather_into_tensor(out, record.reshape(2), group=group)
    return out.reshape(world, 2)


def gather_best(record, group=None):
    """K5 across GPUs: exchange winners over NCCL, reduce (makespan, index) on the device."""
    import torch

    allrec = exchange_winners(record, group)
    out = torch.empty(2, dtype=torch.float64, device=record.device)
    ctx = native.Context.get(record.device.index)
    ctx.call("dfsim_argmin_records", allrec.shape[0], native.ptr(allrec), native.ptr(out))
    return out
