"""Host lowering: reference objects -> flat device arrays.

Runs once per graph / topology class; everything per-strategy runs on the GPU.

* :class:`LoweredGraph` -- node index = rank of the id string in code-point
  order (the reference's every tie-break: engine.py:112,136; graph.py:430,474,483),
  device index = rank of the device string (engine.py:88 entry order), CSR of
  ``DataflowGraph.successors()`` with multiplicity (graph.py:122-131),
  ``in_degree()`` counting dangling refs (graph.py:133-135), sources, per-device
  FIFO capacities, and a device-computed topological order.
* :class:`LoweredProfiles` -- the estimate tables of costmodel.py:282-376:
  per-node op / kind / feature-vector ids (node_features, costmodel.py:226-246),
  exact records keyed (hw, op, features) (profiledb.py:107-112), host-fitted
  linear models (fit_for_grid, costmodel.py:253-279, the same numpy lstsq call),
  link records (profiledb.py:122-125) and resolved override sets
  (strategy.py:75-87).
"""

from __future__ import annotations

import itertools
import math
import operator
import threading
import warnings

import numpy as np

from . import native
from .errors import CycleError, FitError, FitQualityWarning, PatternWarning
from .model import (
    ALGO_MEASURED,
    ALGO_RING,
    COLLECTIVE,
    COMPUTE,
    DEVICE_LINK,
    SCENARIO_GPU_GPU_UNI,
    SCENARIO_NCCL_ALLREDUCE,
    TRANSFER,
    FitStats,
    LinearCostModel,
)

R_SQUARED_WARN = 0.95


def _dev_tensor(a, device, dtype=None):
    import torch

    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if arr.dtype == np.uint64:  # same bits; torch's uint64 support is partial
        arr = arr.view(np.int64)
    t = torch.from_numpy(arr)
    return t.to(device=f"cuda:{device}", non_blocking=False)


_VIEW_AS = {np.dtype(np.uint64): np.int64, np.dtype(np.uint32): np.int32, np.dtype(np.uint16): np.int16}


def upload(arrays: dict, device) -> dict:
    """Many small host tables -> device tensors with ONE host-to-device copy: ``arrays`` maps a
    name to (array, dtype); each lands 16-byte aligned in one device buffer and comes back as
    a typed view (unsigned 16/32/64-bit as the signed type of the same bits).  Empty arrays
    become one zero element (the C-ABI never sees a null table)."""
    import torch

    layout, pos = [], 0
    for name, (a, dt) in arrays.items():
        arr = np.asarray(a, dt).ravel() if np.size(a) else np.zeros(1, dt)
        arr = np.ascontiguousarray(arr)
        arr = arr.view(_VIEW_AS.get(arr.dtype, arr.dtype))
        pos = (pos + 15) // 16 * 16
        layout.append((name, pos, arr))
        pos += arr.nbytes
    host = torch.empty(max(pos, 16), dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    for _, o, arr in layout:
        hv[o:o + arr.nbytes] = arr.view(np.uint8)
    dev = host.to(f"cuda:{device}", non_blocking=True)
    return {name: dev[o:o + arr.nbytes].view(getattr(torch, arr.dtype.name)) for name, o, arr in layout}


# ----------------------------------------------------------------------------- graph


def host_csr(g, ids=None) -> dict:
    """Rank-ordered CSR arrays of ``g`` (host numpy; graph.py:122-135 semantics)."""
    csr = getattr(g, "csr", None)  # document.DocumentGraph: built by the C++ loader
    if csr is not None and (ids is None or ids is g.ids):
        return csr
    ids = list(ids) if ids is not None else sorted(g.nodes)
    rank = {nid: i for i, nid in enumerate(ids)}
    nodes = g.nodes
    devices = sorted({nodes[nid].device for nid in ids})
    drank = {d: i for i, d in enumerate(devices)}
    N, D = len(ids), len(devices)
    indeg = np.empty(N, dtype=np.int32)
    dev = np.empty(N, dtype=np.int32)
    prods, cons = [], []
    for c, nid in enumerate(ids):
        node = nodes[nid]
        indeg[c] = len(node.inputs)
        dev[c] = drank[node.device]
        for pid, _slot in node.inputs:
            r = rank.get(pid)
            if r is not None:
                prods.append(r)
                cons.append(c)
    prods = np.asarray(prods, dtype=np.int64)
    cons = np.asarray(cons, dtype=np.int32)
    succ_idx = cons[np.argsort(prods, kind="stable")]  # consumers already ascending per producer
    succ_off = np.zeros(N + 1, dtype=np.int32)
    if len(prods):
        np.cumsum(np.bincount(prods, minlength=N), out=succ_off[1:])
    queue_off = np.zeros(D + 1, dtype=np.int32)
    if N:
        np.cumsum(np.bincount(dev, minlength=D), out=queue_off[1:])
    return dict(ids=ids, rank=rank, devices=devices, indeg=indeg, device=dev, succ_off=succ_off,
                succ_idx=succ_idx, sources=np.nonzero(indeg == 0)[0].astype(np.int32), queue_off=queue_off,
                max_indeg=int(indeg.max()) if N else 0)



class LoweredGraph:
    """Rank-ordered CSR of one graph, resident on one CUDA device."""

    def __init__(self, g, device: int | None = None, ids=None, topo: bool = True):
        self.ctx = native.Context.get(device)
        h = host_csr(g, ids)
        self.ids, self.rank, self.devices = h["ids"], h["rank"], h["devices"]
        self.n, self.n_devices = len(self.ids), len(self.devices)
        self.host_dev, self.host_indeg = h["device"], h["indeg"]
        self.host_succ_off, self.host_succ_idx = h["succ_off"], h["succ_idx"]
        self._set_device_arrays(h["succ_off"], h["succ_idx"], h["indeg"], h["device"], h["sources"],
                                h["queue_off"], h["max_indeg"], topo)

    def _set_device_arrays(self, succ_off, succ_idx, indeg, dev, sources, queue_off, max_indeg, topo):
        import torch

        d = self.ctx.device
        self.t_succ_off = _dev_tensor(succ_off, d, np.int32)
        self.t_succ_idx = _dev_tensor(succ_idx if len(succ_idx) else np.zeros(1, np.int32), d, np.int32)
        self.t_indeg = _dev_tensor(indeg if len(indeg) else np.zeros(1, np.int32), d, np.int32)
        self.t_dev = _dev_tensor(dev if len(dev) else np.zeros(1, np.int32), d, np.int32)
        self.t_sources = _dev_tensor(sources if len(sources) else np.zeros(1, np.int32), d, np.int32)
        self.t_queue_off = _dev_tensor(queue_off, d, np.int32)
        self.n_sources = int(len(sources))
        self.n_edges = int(len(succ_idx))
        self.max_indeg = max_indeg
        self.t_topo = torch.empty(max(self.n, 1), dtype=torch.int32, device=f"cuda:{d}")
        self.struct = native.Graph(self.n, self.n_devices, self.n_edges, native.ptr(self.t_succ_off),
                                   native.ptr(self.t_succ_idx), native.ptr(self.t_indeg), native.ptr(self.t_dev),
                                   native.ptr(self.t_sources), self.n_sources, native.ptr(self.t_queue_off),
                                   native.P(0), self.max_indeg)
        self.n_ordered = None
        if topo:
            self.compute_topo()

    def compute_topo(self) -> bool:
        """Device Kahn order; returns False when the graph has a cycle."""
        got = native.I32(0)
        self.ctx.call("dfsim_topo_order", native.ctypes.byref(self.struct), native.ptr(self.t_topo),
                      native.ctypes.byref(got))
        self.n_ordered = int(got.value)
        if self.n_ordered == self.n:
            self.struct.topo = native.ptr(self.t_topo)
        return self.n_ordered == self.n

    @property
    def acyclic(self) -> bool:
        return self.n_ordered == self.n

    @classmethod
    def from_arrays(cls, ids, devices, succ_off_t, succ_idx_t, indeg_t, dev_t, sources_t, queue_off_t, topo_t,
                    n_edges, n_sources, max_indeg, ctx, n_ordered):
        """Wrap arrays already resident on the device (the expansion kernel's output)."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.ids = ids
        self.rank = None
        self.devices = devices
        self.n, self.n_devices = len(ids), len(devices)
        self.t_succ_off, self.t_succ_idx, self.t_indeg, self.t_dev = succ_off_t, succ_idx_t, indeg_t, dev_t
        self.t_sources, self.t_queue_off, self.t_topo = sources_t, queue_off_t, topo_t
        self.n_edges, self.n_sources, self.max_indeg, self.n_ordered = n_edges, n_sources, max_indeg, n_ordered
        self.host_dev = None
        self.struct = native.Graph(self.n, self.n_devices, n_edges, native.ptr(succ_off_t), native.ptr(succ_idx_t),
                                   native.ptr(indeg_t), native.ptr(dev_t), native.ptr(sources_t), n_sources,
                                   native.ptr(queue_off_t), native.ptr(topo_t) if n_ordered == self.n else native.P(0),
                                   max_indeg)
        return self

    def levels(self):
        """(order, level_off, n_levels) of the Kahn waves as device int32 tensors (cached);
        K4 wide walks them in reverse.  None for a cyclic graph."""
        if getattr(self, "_levels", None) is None:
            from .prepare import level_order

            off = self.t_succ_off[: self.n + 1].cpu().numpy().astype(np.int64)
            idx = self.t_succ_idx[: self.n_edges].cpu().numpy().astype(np.int64)
            indeg = self.t_indeg[: self.n].cpu().numpy().astype(np.int64)
            lo = level_order(self.n, off, idx, indeg)
            if lo is None:
                return None
            order, _, loff = lo
            d = self.ctx.device
            self._levels = (_dev_tensor(order if len(order) else np.zeros(1, np.int32), d, np.int32),
                            _dev_tensor(loff, d, np.int32), len(loff) - 1)
        return self._levels

    def rank_of(self):
        if self.rank is None:
            self.rank = {nid: i for i, nid in enumerate(self.ids)}
        return self.rank

    def device_of_rank(self):
        if self.host_dev is None:
            self.host_dev = self.t_dev[: self.n].cpu().numpy()
        return self.host_dev


def lowered(g, device: int | None = None) -> LoweredGraph:
    """Per-graph cache (graphs are immutable by contract, graph.py:110-116)."""
    key = (len(g.nodes), len(g.devices), device)
    cached = getattr(g, "_dfsim_b200_lowered", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    lg = LoweredGraph(g, device)
    try:
        object.__setattr__(g, "_dfsim_b200_lowered", (key, lg))
    except (AttributeError, TypeError):
        pass
    return lg


def find_cycle(g) -> list[str] | None:
    """One cycle's ids, DFS from sorted ids (graph.py:392-418); error path only."""
    succ = {nid: [] for nid in g.nodes}
    for n in g.nodes.values():
        for pid, _ in n.inputs:
            if pid in succ:
                succ[pid].append(n.id)
    for v in succ.values():
        v.sort()
    color = dict.fromkeys(g.nodes, 0)
    for root in sorted(g.nodes):
        if color[root]:
            continue
        stack, path = [[root, 0]], [root]
        color[root] = 1
        while stack:
            top = stack[-1]
            nid, i = top
            if i < len(succ[nid]):
                top[1] += 1
                nxt = succ[nid][i]
                if color[nxt] == 1:
                    return path[path.index(nxt):]
                if color[nxt] == 0:
                    color[nxt] = 1
                    stack.append([nxt, 0])
                    path.append(nxt)
            else:
                color[nid] = 2
                stack.pop()
                path.pop()
    return None


def raise_topo_cycle(g, lg: LoweredGraph):
    """topological_order's error (graph.py:440-442)."""
    cyc = find_cycle(g)
    if cyc:
        raise CycleError(cyc)
    left = {nid: len(n.inputs) for nid, n in g.nodes.items()}
    raise CycleError([nid for nid, d in left.items() if d > 0])


# ----------------------------------------------------------------------------- profiles


_IN_KEY: dict = {}  # (input, dim) -> "in{i}_dim{j}", built once


def _in_key(i: int, j: int) -> str:
    k = _IN_KEY.get((i, j))
    if k is None:
        k = _IN_KEY[(i, j)] = f"in{i}_dim{j}"
    return k


def node_features(g, node) -> tuple:
    """costmodel.py:226-246: numeric non-bool attrs + producer dims, sorted by name."""
    feats = {name: float(value) for name, value in node.attrs.items()
             if type(value) in (int, float) or (not isinstance(value, bool) and isinstance(value, (int, float)))}
    nodes = g.nodes
    for i, (pid, slot) in enumerate(node.inputs):
        producer = nodes.get(pid)
        if producer is None or slot >= len(producer.output_shapes):
            continue
        for j, dim in enumerate(producer.output_shapes[slot].dims):
            key = _in_key(i, j)
            if key in feats:
                raise ValueError(f"node {node.id!r}: attr name collides with {key!r}")
            feats[key] = float(dim)
    out = tuple(sorted(feats.items()))
    if not all(math.isfinite(v) for _, v in out):  # OpSignature's finiteness check (profiledb.py:45-47)
        raise ValueError(f"non-finite feature value in {out}")
    return out


def fit_linear(records) -> LinearCostModel:
    """OLS of mean duration on the features (costmodel.py:93-141), same numpy calls."""
    if not records:
        raise FitError("no records to fit")
    op_type, hardware = records[0].signature.op_type, records[0].signature.hardware
    names = tuple(n for n, _ in records[0].signature.arg_features)
    for rec in records:
        if rec.signature.op_type != op_type or rec.signature.hardware != hardware:
            raise FitError("records mix op types or hardware tags")
        if tuple(n for n, _ in rec.signature.arg_features) != names:
            raise FitError("records mix feature names")
    n, k = len(records), len(names)
    if n < k + 1:
        raise FitError(f"underdetermined: {n} records for {k} features (+ intercept)")
    x = np.array([[v for _, v in rec.signature.arg_features] for rec in records], dtype=float)
    y = np.array([rec.mean_duration_us for rec in records], dtype=float)
    design = np.hstack([x, np.ones((n, 1))])
    if np.linalg.matrix_rank(design) < k + 1:
        bad = _collinear(x, names)
        raise FitError("degenerate design matrix; collinear features: " + ", ".join(bad), collinear_features=bad)
    coef, *_ = np.linalg.lstsq(design, y, rcond=None)
    pred = design @ coef
    ss_res = float(np.sum((y - pred) ** 2))
    ss_tot = float(np.sum((y - np.mean(y)) ** 2))
    if ss_tot == 0.0:
        r2 = 1.0 if ss_res < 1e-18 else 0.0
    else:
        r2 = min(1.0, max(0.0, 1.0 - ss_res / ss_tot))
    max_rel = float(np.max(np.abs(pred - y) / np.abs(y)))
    return LinearCostModel(op_type, hardware, names, tuple(float(c) for c in coef[:k]), float(coef[k]),
                           FitStats(r2, max_rel, n))


def fit_linear_many(record_lists, uniform: bool = False) -> list:
    """``fit_linear`` of many record lists: element i is ``fit_linear(record_lists[i])`` or the
    FitError it raises, bit for bit.  Lists of one (records, features) shape share the stacked
    numpy calls that have a per-matrix loop inside (matrix_rank's SVD, the residual sums along
    the last axis: the same LAPACK call and the same pairwise summation per row); the least
    squares and the prediction stay one call per list, on the same C-contiguous design.  Lists
    that would raise, warn (a zero duration divides by zero) or need the collinearity
    diagnosis run through fit_linear itself.  ``uniform``: every list is known to share one op
    type, hardware tag and feature-name tuple (fit_for_grid's groups).  tests/test_fits.py pins
    the equality."""
    out: list = [None] * len(record_lists)
    shapes: dict = {}
    for i, recs in enumerate(record_lists):
        if recs:
            sig0 = recs[0].signature
            names = tuple(n for n, _ in sig0.arg_features)
            if len(recs) >= len(names) + 1 and (uniform or all(
                    r.signature.op_type == sig0.op_type and r.signature.hardware == sig0.hardware
                    and tuple(n for n, _ in r.signature.arg_features) == names for r in recs)):
                shapes.setdefault((len(recs), len(names)), []).append(i)
                continue
        out[i] = _fit_or_error(recs)
    for (n, k), items in shapes.items():
        x = np.array([[[v for _, v in r.signature.arg_features] for r in record_lists[i]] for i in items],
                     dtype=float).reshape(len(items), n, k)
        y = np.array([[r.mean_duration_us for r in record_lists[i]] for i in items], dtype=float)
        design = np.concatenate([x, np.ones((len(items), n, 1))], axis=2)
        rank = np.linalg.matrix_rank(design)
        fine = (rank == k + 1) & np.all(y != 0.0, axis=1) & np.all(np.isfinite(y), axis=1)
        ok = np.flatnonzero(fine)
        for j in np.flatnonzero(~fine).tolist():
            out[items[j]] = _fit_or_error(record_lists[items[j]])
        if not len(ok):
            continue
        d, yy = design[ok], y[ok]
        coef = _lstsq_stacked(d, yy)
        pred = np.empty_like(yy)
        for t in range(len(ok)):
            pred[t] = d[t] @ coef[t]
        ss_res = np.sum((yy - pred) ** 2, axis=-1)
        ss_tot = np.sum((yy - np.mean(yy, axis=-1, keepdims=True)) ** 2, axis=-1)
        max_rel = np.max(np.abs(pred - yy) / np.abs(yy), axis=-1)
        for t, j in enumerate(ok.tolist()):
            recs = record_lists[items[j]]
            sig0 = recs[0].signature
            res, tot = float(ss_res[t]), float(ss_tot[t])
            if tot == 0.0:
                r2 = 1.0 if res < 1e-18 else 0.0
            else:
                r2 = min(1.0, max(0.0, 1.0 - res / tot))
            out[items[j]] = LinearCostModel(sig0.op_type, sig0.hardware, tuple(nm for nm, _ in sig0.arg_features),
                                            tuple(float(c) for c in coef[t, :k]), float(coef[t, k]),
                                            FitStats(r2, float(max_rel[t]), n))
    return out


def _lstsq_stacked(d, y):
    """``np.linalg.lstsq(d[t], y[t], rcond=None)[0]`` for every t: one call of the gufunc that
    lstsq wraps (numpy/linalg/_linalg.py: dgelsd per matrix, on the same copies), with lstsq's
    rcond and error state; one lstsq call per matrix where that gufunc is not available."""
    m, n = d.shape[-2:]
    gufunc = getattr(getattr(np.linalg, "_umath_linalg", None), "lstsq", None)
    if gufunc is not None:
        try:
            with np.errstate(call=_lstsq_error, invalid="call", over="ignore", divide="ignore", under="ignore"):
                x = gufunc(d, y[..., None], np.finfo(np.float64).eps * max(n, m), signature="ddd->ddid")[0]
            return x[..., 0]
        except TypeError:  # a numpy whose private gufunc has another signature
            pass
    return np.stack([np.linalg.lstsq(d[t], y[t], rcond=None)[0] for t in range(len(d))])


def _lstsq_error(err, flag):
    raise np.linalg.LinAlgError("SVD did not converge in Linear Least Squares")


def _fit_or_error(recs):
    try:
        return fit_linear(recs)
    except FitError as e:
        return e


def _collinear(x, names):
    kept = np.ones((x.shape[0], 1))
    bad = []
    for j, name in enumerate(names):
        cand = np.hstack([kept, x[:, j:j + 1]])
        if np.linalg.matrix_rank(cand) == np.linalg.matrix_rank(kept):
            bad.append(name)
        else:
            kept = cand
    return bad


def fit_for_grid(db, op_type: str, hardware: str):
    """costmodel.py:253-279: largest same-name group (ties: smallest name tuple)."""
    grid_map = db.op_records.get((op_type, hardware), {})
    grid = [grid_map[k] for k in sorted(grid_map)]
    if not grid:
        return None
    groups = {}
    for rec in grid:
        groups.setdefault(tuple(n for n, _ in rec.signature.arg_features), []).append(rec)
    best = max(len(r) for r in groups.values())
    chosen = min(k for k in groups if len(groups[k]) == best)
    try:
        model = fit_linear(groups[chosen])
    except FitError:
        return None
    if model.fit_stats.r_squared < R_SQUARED_WARN:
        warnings.warn(f"linear model for {op_type}/{hardware} has r_squared={model.fit_stats.r_squared:.4f}; "
                      "estimates may be unreliable", FitQualityWarning, stacklevel=3)
    return model


def fit_for_grid_many(db, pairs) -> dict:
    """``fit_for_grid`` of every (op type, hardware) pair, the fits batched (fit_linear_many);
    warnings in the order of ``pairs``."""
    chosen = {}
    for op_type, hardware in pairs:
        grid_map = db.op_records.get((op_type, hardware), {})
        if not grid_map:
            continue
        groups = {}
        for key in sorted(grid_map):  # grid keys are the records' feature tuples
            groups.setdefault(tuple(map(_FIRST, key)), []).append(grid_map[key])
        best = max(len(r) for r in groups.values())
        chosen[(op_type, hardware)] = groups[min(k for k in groups if len(groups[k]) == best)]
    fits = dict(zip(chosen, fit_linear_many(list(chosen.values()), uniform=True)))
    out = {}
    for pair in pairs:
        m = fits.get(pair)
        if m is None or isinstance(m, FitError):
            out[pair] = None
            continue
        if m.fit_stats.r_squared < R_SQUARED_WARN:
            warnings.warn(f"linear model for {pair[0]}/{pair[1]} has r_squared={m.fit_stats.r_squared:.4f}; "
                          "estimates may be unreliable", FitQualityWarning, stacklevel=3)
        out[pair] = m
    return out


def match_pattern(pattern: str, nid: str) -> bool:
    return nid.startswith(pattern[:-1]) if pattern.endswith("*") else nid == pattern


def resolve_overrides(overrides: dict, ids: list) -> dict:
    """strategy.py:75-87 -- later-listed patterns win; unmatched patterns warn."""
    out = {}
    for pattern, value in overrides.items():
        hit = [nid for nid in ids if match_pattern(pattern, nid)]
        if not hit:
            warnings.warn(f"override pattern {pattern!r} matched no node", PatternWarning, stacklevel=3)
        for nid in hit:
            out[nid] = float(value)
    return out


def node_rows(g, ids) -> list:
    """Per node (rank order): (features, comm_ok, bytes, group size, link thr, link lat) -- the
    graph-dependent inputs of estimate_all (costmodel.py:226-246, 347-376)."""
    rows = []
    nodes = g.nodes
    for nid in ids:
        n = nodes[nid]
        feats = node_features(g, n)
        b = n.attrs.get("bytes")
        row = (feats, 0, 0, 0, 1.0, 0.0)
        if n.kind == TRANSFER:
            dev = g.devices.get(n.device)
            if dev is not None and dev.kind == DEVICE_LINK and isinstance(b, int):
                row = (feats, 1, _i64(b), 0, dev.throughput_mbps, dev.latency_us)
        elif n.kind == COLLECTIVE:
            grp = n.attrs.get("group")
            if isinstance(grp, (list, tuple)) and isinstance(b, int):
                row = (feats, 1, _i64(b), len(grp), 1.0, 0.0)
        rows.append(row)
    return rows


class _FeatureRegistry:
    """Process-wide interning of feature vectors (node_features tuples) -> int ids, so that the
    rows of graph variants, clones and classes are combined with numpy instead of per node."""

    def __init__(self):
        self.ids: dict = {}
        self.rows: list = []
        # flat copy: vector k = names[f_name[f_off[k]:f_off[k+1]]], values f_val[...]
        self.names: dict = {}
        self.name_list: list = []
        self.f_off, self.f_name, self.f_val = [0], [], []
        self._flat = None
        self.lock = threading.Lock()

    def intern(self, feats_list) -> np.ndarray:
        with self.lock:
            ids, rows, names = self.ids, self.rows, self.names
            out = np.empty(len(feats_list), np.int64)
            for i, f in enumerate(feats_list):
                k = ids.get(f)
                if k is None:
                    k = ids[f] = len(rows)
                    rows.append(f)
                    for nm, v in f:
                        gid = names.get(nm)
                        if gid is None:
                            gid = names[nm] = len(self.name_list)
                            self.name_list.append(nm)
                        self.f_name.append(gid)
                        self.f_val.append(v)
                    self.f_off.append(len(self.f_name))
                out[i] = k
            return out

    def flat(self):
        """(f_off, f_name, f_val) as numpy arrays; when the registry has grown, only the new
        entries are converted and appended (sweeps intern class after class)."""
        with self.lock:
            if self._flat is None:
                self._flat = (np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float64))
            off, name, val = self._flat
            if len(off) != len(self.f_off):
                k, m = len(off), len(name)
                self._flat = (np.concatenate([off, np.asarray(self.f_off[k:], np.int64)]),
                              np.concatenate([name, np.asarray(self.f_name[m:], np.int64)]),
                              np.concatenate([val, np.asarray(self.f_val[m:], np.float64)]))
            return self._flat


FEATURES = _FeatureRegistry()
ROW_FIELDS = ("fid", "ok", "bytes", "gsize", "thr", "lat")


def row_arrays(rows) -> dict:
    """node_rows tuples -> arrays (features as FEATURES ids)."""
    n = len(rows)
    return dict(fid=FEATURES.intern([r[0] for r in rows]),
                ok=np.fromiter((r[1] for r in rows), np.uint8, n), bytes=np.fromiter((r[2] for r in rows), np.int64, n),
                gsize=np.fromiter((r[3] for r in rows), np.int32, n), thr=np.fromiter((r[4] for r in rows), np.float64, n),
                lat=np.fromiter((r[5] for r in rows), np.float64, n))


def base_arrays(g):
    """Row arrays of every node of g in insertion order + {node id: index}; cached on the graph
    (graphs are immutable by contract, graph.py:110-116)."""
    cached = getattr(g, "_dfsim_base_arr", None)
    if cached is not None and cached[0] == len(g.nodes):
        return cached[1], cached[2]
    order = list(g.nodes)
    arr = row_arrays(node_rows(g, order))
    index = {nid: i for i, nid in enumerate(order)}
    try:
        object.__setattr__(g, "_dfsim_base_arr", (len(order), arr, index))
    except (AttributeError, TypeError):
        pass
    return arr, index


_FIRST = operator.itemgetter(0)
_HARDWARE, _GAP = operator.attrgetter("hardware"), operator.attrgetter("op_gap_us")
_COLLECTIVE, _OVERRIDES = operator.attrgetter("collective"), operator.attrgetter("overrides")
_ALGO, _PATH = operator.attrgetter("collective.algo"), operator.attrgetter("collective.path")


class LoweredProfiles:
    """Device tables for dfsim_estimate_batch over one graph and a list of configs.

    ``variant_rows`` (optional): one ``node_rows`` list per graph variant -- graphs with
    g's structure whose attributes / shapes differ (e.g. one per batch size); candidate i
    then reads variant ``strat_gv[i]``.  Without it there is one variant, g itself.
    """

    def __init__(self, g, ids, db, configs, device: int, variant_rows=None, strat_gv=None, fit_cache=None,
                 variant_arrays=None, op_kind=None):
        self.device = device
        N = len(ids)
        nodes = g.nodes
        rank = {nid: i for i, nid in enumerate(ids)}
        # hardware tags, paths, override sets of the strategies: each distinct value is handled
        # once, the per-candidate columns are built with C-level maps (sweeps hold 10^4-10^5 configs)
        self.hw_ids, self.path_ids = {}, {}
        ov_sets, ov_key_to_id = [], {}
        n = len(configs)
        hws = list(map(_HARDWARE, configs))
        for h in dict.fromkeys(hws):
            self.hw_ids[h] = len(self.hw_ids)
        self.strat_hw = np.fromiter(map(self.hw_ids.__getitem__, hws), np.int32, n)
        self.strat_gap = np.fromiter(map(float, map(_GAP, configs)), np.float64, n)
        # collective algorithm and path by value (sweeps often build a config object per candidate);
        # one identity pass when every candidate shares one collective object
        c0 = configs[0].collective if n else None
        shared = n > 0 and all(map(operator.is_, map(_COLLECTIVE, configs), itertools.repeat(c0)))
        algos, paths = ([c0.algo], [c0.path]) if shared else (list(map(_ALGO, configs)), list(map(_PATH, configs)))
        algo_code = {}
        for al in dict.fromkeys(algos):
            if al not in (ALGO_MEASURED, ALGO_RING):
                raise ValueError(f"unknown collective algorithm {al!r}")
            algo_code[al] = 0 if al == ALGO_MEASURED else 1
        for pth in dict.fromkeys(paths):
            self.path_ids[pth] = len(self.path_ids)
        if shared:
            self.strat_algo = np.full(n, algo_code[algos[0]], np.uint8)
            self.strat_path = np.full(n, self.path_ids[paths[0]], np.int32)
        else:
            self.strat_algo = np.fromiter(map(algo_code.__getitem__, algos), np.uint8, n)
            self.strat_path = np.fromiter(map(self.path_ids.__getitem__, paths), np.int32, n)
        self.strat_ov = np.full(n, -1, np.int32)
        ovs = list(map(_OVERRIDES, configs))
        for i in itertools.compress(range(n), ovs):  # candidates with overrides
            ov_key = tuple(ovs[i].items())
            if ov_key not in ov_key_to_id:
                ov_key_to_id[ov_key] = len(ov_sets)
                ov_sets.append(resolve_overrides(ovs[i], ids))
            self.strat_ov[i] = ov_key_to_id[ov_key]
        # document.DocumentGraph: the C++ loader already interned ops, signatures and comm rows
        doc = (getattr(g, "signatures", None) is not None and variant_rows is None and variant_arrays is None
               and ids is g.ids)
        if variant_arrays is None:
            if variant_rows is None:
                variant_rows = [] if doc else [node_rows(g, ids)]
            variant_arrays = [row_arrays(rows) for rows in variant_rows]
        GV = 1 if doc else (variant_arrays["fid"].shape[0] if isinstance(variant_arrays, dict) else len(variant_arrays))
        self.n_gvariants = GV
        self.strat_gv = (np.asarray(strat_gv, np.int32) if strat_gv is not None
                         else np.zeros(len(configs), np.int32))
        # per node: op, kind (structural); per (variant, node): features and comm attributes
        op_ids, sig_ids = {}, {}
        flat_uniq = None  # registry ids of this class's feature vectors (sig id = index)
        op = np.empty(N, np.int32)
        kind = np.empty(N, np.uint8)
        self.op_nodes = {}
        if doc:
            op_ids = {name: k for k, name in enumerate(g.op_names)}
            op[:], kind[:] = g.op_of, g.kind_of
            order = np.argsort(op, kind="stable")
            bounds = np.searchsorted(op[order], np.arange(len(op_ids) + 1))
            self.op_nodes = {name: order[bounds[k]:bounds[k + 1]].tolist() for name, k in op_ids.items()}
        else:  # op ids in order of first appearance, node lists ascending (one stable sort)
            if op_kind is not None:  # an expansion's ids: op type and kind code by origin (no objects)
                ops, kinds = op_kind
            else:
                objs = [nodes[nid] for nid in ids]
                ops = [n.op_type for n in objs]
                kinds = [0 if n.kind == COMPUTE else (1 if n.kind == TRANSFER else 2) for n in objs]
            op_ids = {name: k for k, name in enumerate(dict.fromkeys(ops))}
            op[:] = np.fromiter(map(op_ids.__getitem__, ops), np.int32, N)
            kind[:] = kinds
            order = np.argsort(op, kind="stable")
            bounds = np.searchsorted(op[order], np.arange(len(op_ids) + 1))
            self.op_nodes = {name: order[bounds[k]:bounds[k + 1]] for name, k in op_ids.items()}
        sig = np.empty((GV, N), np.int32)
        cbytes = np.zeros((GV, N), np.int64)
        cok = np.zeros((GV, N), np.uint8)
        gsize = np.zeros((GV, N), np.int32)
        lthr = np.ones((GV, N), np.float64)
        llat = np.zeros((GV, N), np.float64)
        if doc:
            sig_ids = {feats: k for k, feats in enumerate(g.signatures)}
            sig[0], cok[0], cbytes[0], gsize[0] = g.sig_of, g.comm["ok"], g.comm["bytes"], g.comm["group"]
            lthr[0], llat[0] = g.comm["thr"], g.comm["lat"]
        if variant_arrays:
            # a list of per-variant row dicts, or one dict of stacked [GV, N] fields
            va = variant_arrays if isinstance(variant_arrays, dict) else \
                {k: np.stack([v[k] for v in variant_arrays]) for k in ROW_FIELDS}
            if va["fid"].shape != (GV, N):
                raise ValueError("graph variants must share the class structure")
            fid = va["fid"]
            present = np.zeros(int(fid.max(initial=-1)) + 1, np.int64)  # class-local signature ids:
            present[fid.ravel()] = 1                                    # registry ids in ascending order
            flat_uniq = np.flatnonzero(present)
            sig[:] = (np.cumsum(present) - 1)[fid]
            for name, dst in (("ok", cok), ("bytes", cbytes), ("gsize", gsize), ("thr", lthr), ("lat", llat)):
                dst[:] = va[name]
        self.op_ids = op_ids
        # the fused engine forms durations on the fly (base + gap | override) and relies on every
        # one being a finite non-negative double; anything else (NaN included: DurationEntry's
        # `not x >= 0.0`, costmodel.py:78-80) must take the exact K2 path and its error
        gaps = np.asarray(self.strat_gap, np.float64)
        self.fused_values_ok = (bool(np.all(np.isfinite(gaps) & (gaps >= 0.0)))
                                and all(math.isfinite(v) and v >= 0.0 for res in ov_sets for v in res.values()))
        # exact records for (hw, op, sig) triples present in the graph
        ekeys, emeans = [], []
        for hw, h in self.hw_ids.items():
            for opname, o in op_ids.items():
                grid = db.op_records.get((opname, hw))
                if not grid:
                    continue
                if flat_uniq is not None:  # records whose vectors occur in this class
                    fids = np.fromiter((FEATURES.ids.get(f, -1) for f in grid), np.int64, len(grid))
                    loc = np.searchsorted(flat_uniq, fids)
                    hit = (fids >= 0) & (loc < len(flat_uniq)) & (flat_uniq[np.minimum(loc, len(flat_uniq) - 1)] == fids)
                    recs = list(grid.values())
                    for j in np.flatnonzero(hit).tolist():
                        ekeys.append((h << 42) | (o << 21) | int(loc[j]))
                        emeans.append(recs[j].mean_duration_us)
                    continue
                for feats, rec in grid.items():
                    s = sig_ids.get(feats)
                    if s is not None:
                        ekeys.append((h << 42) | (o << 21) | s)
                        emeans.append(rec.mean_duration_us)
        # fitted models where some node could need one (the reference fits lazily, costmodel.py:313-316)
        mkeys, moff, mnames, mcoef, micpt = [], [0], [], [], []
        exact_keys = np.unique(np.asarray(ekeys, np.uint64))
        self.models = {}
        if flat_uniq is not None:  # the class's feature entries, gathered from the registry
            f_off, f_name, f_val = FEATURES.flat()
            starts, lens = f_off[flat_uniq], f_off[flat_uniq + 1] - f_off[flat_uniq]
            seg = np.zeros(len(flat_uniq) + 1, np.int64)
            np.cumsum(lens, out=seg[1:])
            take = np.repeat(starts - seg[:-1], lens) + np.arange(int(seg[-1]), dtype=np.int64)
            g_names, g_vals = f_name[take], f_val[take]
            name_pool = {FEATURES.name_list[k] for k in np.unique(g_names).tolist()}
        else:
            name_pool = {nm for feats in sig_ids for nm, _ in feats}
        fitted, wanted = [], []
        for hw, h in self.hw_ids.items():
            need = self._ops_needing_models(h, op, sig, exact_keys, ids, ov_sets)
            wanted += [(opname, hw, (h << 21) | o) for opname, o in op_ids.items()
                       if o in need and db.op_records.get((opname, hw))]
        fit_cache = {} if fit_cache is None else fit_cache  # one fit per (op, hw) per sweep
        fit_cache.update(fit_for_grid_many(db, [(op_, hw) for op_, hw, _ in wanted if (op_, hw) not in fit_cache]))
        for opname, hw, key in wanted:
            m = self.models[(opname, hw)] = fit_cache[(opname, hw)]
            if m is not None:
                name_pool.update(m.feature_names)
                fitted.append((key, m))
        names_sorted = sorted(name_pool)
        name_id = {nm: i for i, nm in enumerate(names_sorted)}
        fitted.sort(key=lambda kv: kv[0])
        for key, m in fitted:
            mkeys.append(key)
            mnames.extend(name_id[nm] for nm in m.feature_names)
            mcoef.extend(m.coefficients)
            moff.append(len(mnames))
            micpt.append(m.intercept)
        # feature vectors
        if flat_uniq is not None:  # names ascend within a vector in both orders (ids follow the sorted names)
            local = np.full(len(FEATURES.name_list), -1, np.int64)
            for nm, i in name_id.items():
                k = FEATURES.names.get(nm)
                if k is not None:
                    local[k] = i
            soff, sname, sval = seg, local[g_names], g_vals
        else:
            soff, sname, sval = [0], [], []
            for feats in sig_ids:  # insertion order == id order
                for nm, v in feats:
                    sname.append(name_id[nm])
                    sval.append(v)
                soff.append(len(sname))
        # links
        n_paths = len(self.path_ids)
        uni_ok = np.zeros(max(n_paths, 1), np.uint8)
        uni_thr = np.ones(max(n_paths, 1), np.float64)
        uni_lat = np.zeros(max(n_paths, 1), np.float64)
        nkeys, nthr = [], []
        for path, p in self.path_ids.items():
            rec = db.link_records.get((SCENARIO_GPU_GPU_UNI, path, 2))
            if rec is not None:
                uni_ok[p], uni_thr[p], uni_lat[p] = 1, rec.throughput_mbps, rec.latency_us
        for (scen, path, parts), rec in db.link_records.items():
            if scen == SCENARIO_NCCL_ALLREDUCE and path in self.path_ids:
                nkeys.append((self.path_ids[path] << 32) | int(parts))
                nthr.append(rec.throughput_mbps)
        # overrides
        ooff, onode, oval = [0], [], []
        for res in ov_sets:
            pairs = sorted((rank[nid], val) for nid, val in res.items())
            onode.extend(p for p, _ in pairs)
            oval.extend(v for _, v in pairs)
            ooff.append(len(onode))
        # one bit per node rank: in some override set (the fused engine skips the set's search otherwise)
        oany = np.zeros((N + 31) // 32 + 1, np.uint32)
        if onode:
            hit = np.unique(np.asarray(onode, np.int64))
            np.bitwise_or.at(oany, hit >> 5, (np.uint32(1) << (hit & 31).astype(np.uint32)))

        def srt(keys, *vals):
            if not keys:
                return (np.zeros(1, np.uint64),) + tuple(np.zeros(1, np.asarray(v).dtype if len(v) else np.float64)
                                                          for v in vals)
            o = np.argsort(np.asarray(keys, np.uint64), kind="stable")
            return (np.asarray(keys, np.uint64)[o],) + tuple(np.asarray(v)[o] for v in vals)

        ek, em = srt(ekeys, np.asarray(emeans, np.float64))
        nk, nt = srt(nkeys, np.asarray(nthr, np.float64))
        up = upload(dict(
            op=(op, np.int32), kind=(kind, np.uint8), sig=(sig, np.int32), cbytes=(cbytes, np.int64),
            cok=(cok, np.uint8), gsize=(gsize, np.int32), lthr=(lthr, np.float64), llat=(llat, np.float64),
            soff=(soff, np.int32), sname=(sname, np.int32), sval=(sval, np.float64),
            ek=(ek, np.uint64), em=(em, np.float64),
            mk=(np.asarray(mkeys, np.uint64), np.uint64), moff=(moff, np.int32), mname=(mnames, np.int32),
            mcoef=(mcoef, np.float64), micpt=(micpt, np.float64),
            nk=(nk, np.uint64), nt=(nt, np.float64),
            uok=(uni_ok, np.uint8), uthr=(uni_thr, np.float64), ulat=(uni_lat, np.float64),
            ooff=(ooff, np.int32), onode=(onode, np.int32), oval=(oval, np.float64), oany=(oany, np.uint32),
            s_hw=(self.strat_hw, np.int32), s_gap=(self.strat_gap, np.float64), s_algo=(self.strat_algo, np.uint8),
            s_path=(self.strat_path, np.int32), s_ov=(self.strat_ov, np.int32), s_gv=(self.strat_gv, np.int32)),
            device)
        self.tensors = {k: v for k, v in up.items() if not k.startswith("s_")}
        t = self.tensors
        pp = native.ptr
        self.struct = native.ProfileTables(
            pp(t["op"]), pp(t["kind"]), pp(t["sig"]), pp(t["cbytes"]), pp(t["cok"]), pp(t["gsize"]),
            pp(t["lthr"]), pp(t["llat"]),
            len(flat_uniq) if flat_uniq is not None else len(sig_ids), pp(t["soff"]), pp(t["sname"]),
            pp(t["sval"]),
            len(ekeys), pp(t["ek"]), pp(t["em"]),
            len(mkeys), pp(t["mk"]), pp(t["moff"]), pp(t["mname"]), pp(t["mcoef"]), pp(t["micpt"]),
            len(nkeys), pp(t["nk"]), pp(t["nt"]),
            n_paths, pp(t["uok"]), pp(t["uthr"]), pp(t["ulat"]),
            len(ov_sets), pp(t["ooff"]), pp(t["onode"]), pp(t["oval"]))
        self.n_sims = len(configs)
        self.t_strat = {k[2:]: v for k, v in up.items() if k.startswith("s_")}
        s = self.t_strat
        self.strategies = native.Strategies(self.n_sims, pp(s["hw"]), pp(s["gap"]), pp(s["algo"]), pp(s["path"]),
                                            pp(s["ov"]), pp(s["gv"]))

    def _ops_needing_models(self, h, op, sig, exact_keys, ids, ov_sets) -> set:
        """Op ids (of hardware tag h) with some node that has no exact record in some graph
        variant and is not overridden in every strategy of this tag: one vectorised pass over
        all nodes instead of one per (op, tag)."""
        keys = ((np.uint64(h) << np.uint64(42)) | (op.astype(np.uint64) << np.uint64(21))
                | sig.astype(np.uint64))                                 # [GV, N]
        missing = np.flatnonzero(~np.isin(keys, exact_keys).all(axis=0))
        if missing.size == 0:
            return set()
        ov_h = self.strat_ov[self.strat_hw == h]
        if ov_h.size and (ov_h >= 0).all():  # nodes overridden for every strategy of this tag need nothing
            sets = [ov_sets[k] for k in np.unique(ov_h).tolist()]
            missing = np.asarray([i for i in missing.tolist() if not all(ids[i] in res for res in sets)], np.int64)
        return set(np.unique(op[missing]).tolist()) if missing.size else set()


def _i64(b: int) -> int:
    if not -(2 ** 63) <= b < 2 ** 63:
        raise ValueError(f"bytes {b} outside the int64 range of the device tables")
    return int(b)
