"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference hot path.

This module is the results oracle.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it; the
product package never does.  It restates, in plain Python over the same
duck-typed containers, the reference algorithms of arXiv 2002.06790's ``dfsim``:

* ``expand``      -- strategy.py:170-282 (ids 162-167, patterns 60-87)
* ``estimate``    -- costmodel.py:282-376 with predict 158-165, fit 93-155/253-279,
                     comm formulas 168-223, features 226-246
* ``simulate``    -- engine.py:96-146 and _finalize 69-93
* ``critical_path`` -- graph.py:424-485 (Kahn + suffix DP + min-id walk)
* ``summarize``   -- reporting.py:117-162 (op shares, compute/comm busy, interval
                     overlap 92-114, critical path on finish - start)
* ``to_trace``    -- reporting.py:43-74 (Chrome trace JSON, indent 1)

Pinning: ``tests/test_oracle.py`` checks every function here against the golden
fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced by
running the real reference.  Parity is therefore pinned, not assumed.
"""

from __future__ import annotations

import heapq
import warnings

import numpy as np

COMPUTE, TRANSFER, COLLECTIVE = "Compute", "Transfer", "Collective"
MIB = 2 ** 20


class OracleUnknownOp(Exception):
    def __init__(self, nodes):
        self.nodes = dict(nodes)
        super().__init__(str(sorted(self.nodes)))


class OracleCycle(Exception):
    def __init__(self, ids):
        self.ids = list(ids)
        super().__init__(str(self.ids))


# ----------------------------------------------------------------------------- patterns


def _matches(pattern: str, nid: str) -> bool:
    # strategy.py:69-72
    return nid.startswith(pattern[:-1]) if pattern.endswith("*") else nid == pattern


def _resolved_overrides(overrides: dict, ids: list) -> dict:
    # strategy.py:75-87: dict order, later patterns overwrite earlier ones
    out = {}
    for pattern, value in overrides.items():
        for nid in ids:
            if _matches(pattern, nid):
                out[nid] = float(value)
    return out


# ----------------------------------------------------------------------------- expansion


class _Node:
    __slots__ = ("id", "op_type", "device", "kind", "attrs", "inputs", "output_shapes")

    def __init__(self, id, op_type, device, kind, attrs, inputs, output_shapes):
        self.id, self.op_type, self.device, self.kind = id, op_type, device, kind
        self.attrs, self.inputs, self.output_shapes = attrs, tuple(inputs), tuple(output_shapes)


class _Dev:
    __slots__ = ("id", "kind", "hardware", "throughput_mbps", "latency_us")

    def __init__(self, id, kind, hardware="", throughput_mbps=None, latency_us=0.0):
        self.id, self.kind, self.hardware = id, kind, hardware
        self.throughput_mbps, self.latency_us = throughput_mbps, latency_us


class _Graph:
    def __init__(self, nodes, devices):
        self.nodes, self.devices = nodes, devices


def _byte_size(shape) -> int:
    n = 1
    for d in shape.dims:
        n *= d
    return shape.dtype_bytes * n


def expand(g, cfg):
    """Data-parallel clone + allreduce insertion (strategy.py:170-282).

    Returns (graph, replica_of, collective_ids).  Written as one pass over the
    base graph with a producer->collective rename map, which yields the same
    input lists as the reference's repeated rewiring loop (231-238): a ref to
    any replica of a marked gradient becomes (collective, same slot).
    """
    R = cfg.replicas
    marked = sorted({nid for p in cfg.gradient_markers for nid in g.nodes if _matches(p, nid)})
    for nid in marked:
        n = g.nodes[nid]
        if n.kind != COMPUTE:
            raise ValueError(f"marker on {n.kind} node")
        if not n.output_shapes or _byte_size(n.output_shapes[0]) <= 0:
            raise ValueError("gradient without output")
    rename = {}
    if R > 1:
        for gid in marked:
            for k in range(R):
                rename[f"{gid}@r{k}"] = f"allreduce_{gid}"
    nodes, replica_of = {}, {}
    for k in range(R):
        for nid, n in g.nodes.items():
            dev = cfg.device_map[k] if (cfg.device_map and n.kind == COMPUTE) else n.device
            cid = f"{nid}@r{k}"
            ins = tuple((rename.get(f"{p}@r{k}", f"{p}@r{k}"), s) for p, s in n.inputs)
            nodes[cid] = _Node(cid, n.op_type, dev, n.kind, n.attrs, ins, n.output_shapes)
            replica_of[cid] = (nid, k)
    group = list(cfg.device_map) if cfg.device_map else sorted({n.device for n in nodes.values()})
    fabric = f"collective:{cfg.collective.path}:" + "+".join(group)
    coll = []
    if R > 1:
        for gid in marked:
            grad = g.nodes[gid]
            cid = f"allreduce_{gid}"
            nodes[cid] = _Node(cid, "AllReduce", fabric, COLLECTIVE,
                               {"group": list(group), "bytes": _byte_size(grad.output_shapes[0]),
                                "path": cfg.collective.path},
                               [(f"{gid}@r{k}", 0) for k in range(R)], grad.output_shapes)
            coll.append(cid)
    devices = {}
    for n in nodes.values():
        if n.id in coll or n.device in devices:
            continue
        devices[n.device] = g.devices[n.device] if n.device in g.devices else _Dev(n.device, "Compute", cfg.hardware)
    if coll:
        devices[fabric] = _Dev(fabric, "CollectiveResource", cfg.hardware, 1.0, 0.0)
    return _Graph(nodes, devices), replica_of, coll


# ----------------------------------------------------------------------------- estimation


def _features(g, n):
    # costmodel.py:226-246
    f = {}
    for name, v in n.attrs.items():
        if isinstance(v, (int, float)) and not isinstance(v, bool):
            f[name] = float(v)
    for i, (pid, slot) in enumerate(n.inputs):
        p = g.nodes.get(pid)
        if p is None or slot >= len(p.output_shapes):
            continue
        for j, d in enumerate(p.output_shapes[slot].dims):
            f[f"in{i}_dim{j}"] = float(d)
    return tuple(sorted(f.items()))


def _fit(grid_records):
    """fit_for_grid + fit_linear (costmodel.py:93-141, 253-279): the same numpy calls."""
    if not grid_records:
        return None
    groups = {}
    for rec in grid_records:
        groups.setdefault(tuple(n for n, _ in rec.signature.arg_features), []).append(rec)
    size = max(len(v) for v in groups.values())
    names = min(k for k, v in groups.items() if len(v) == size)
    recs = groups[names]
    n, k = len(recs), len(names)
    if n < k + 1:
        return None
    x = np.array([[v for _, v in r.signature.arg_features] for r in recs], dtype=float)
    y = np.array([r.mean_duration_us for r in recs], dtype=float)
    design = np.hstack([x, np.ones((n, 1))])
    if np.linalg.matrix_rank(design) < k + 1:
        return None
    coef, *_ = np.linalg.lstsq(design, y, rcond=None)
    return names, tuple(float(c) for c in coef[:k]), float(coef[k])


def predict_value(coefs, intercept, feats):
    """predict (costmodel.py:158-165) with CPython's built-in float ``sum``."""
    value = intercept + sum(c * f for c, f in zip(coefs, feats))
    return max(0.0, value)


def predict_neumaier(coefs, intercept, feats):
    """The same value as ``predict_value`` written as the explicit loop CPython 3.12's
    ``sum`` runs for floats (Python/bltinmodule.c, builtin_sum_impl: int start 0,
    first term exact, Neumaier compensation, compensation added only if nonzero
    and finite).  This is the algorithm the device kernel restates."""
    import math
    if not coefs:
        return max(0.0, intercept + 0.0)
    s = 0.0 + coefs[0] * feats[0]
    comp = 0.0
    for c, f in zip(coefs[1:], feats[1:]):
        x = c * f
        t = s + x
        comp += (s - t) + x if abs(s) >= abs(x) else (x - t) + s
        s = t
    if comp != 0.0 and math.isfinite(comp):
        s += comp
    value = intercept + s
    return value if value > 0.0 else 0.0


def _comm(g, n, db, cfg):
    # costmodel.py:334-376 with transfer_time / allreduce_time 168-223
    if n.kind == TRANSFER:
        dev = g.devices.get(n.device)
        b = n.attrs.get("bytes")
        if dev is None or dev.kind != "Link" or not isinstance(b, int):
            return None
        if b <= 0:
            raise ValueError("bytes must be > 0")
        return dev.latency_us + (b / MIB) / dev.throughput_mbps * 1e6
    if n.kind == COLLECTIVE:
        group, b = n.attrs.get("group"), n.attrs.get("bytes")
        if not isinstance(group, (list, tuple)) or not isinstance(b, int):
            return None
        parts = len(group)
        if b <= 0 or parts < 2:
            return None
        path = cfg.collective.path
        uni = db.link_records.get(("gpu-gpu-uni", path, 2))
        if cfg.collective.algo == "MeasuredThroughput":
            rec = db.link_records.get(("nccl-allreduce", path, parts))
            if rec is not None:
                return 0.0 + (b / MIB) / rec.throughput_mbps * 1e6
        if uni is None:
            return None
        ring = 2.0 * (parts - 1) / parts
        return ring * (b / MIB) / uni.throughput_mbps * 1e6 + 2.0 * (parts - 1) * uni.latency_us
    return None


def estimate(g, db, cfg):
    """Fallback chain per node in sorted id order; returns {nid: (us, source)}."""
    ids = sorted(g.nodes)
    ov = _resolved_overrides(cfg.overrides, ids)
    models, out, unknown = {}, {}, {}
    for nid in ids:
        n = g.nodes[nid]
        if nid in ov:
            out[nid] = (ov[nid], "Override")
            continue
        gap = cfg.op_gap_us if n.kind == COMPUTE else 0.0
        feats = _features(g, n)
        grid = db.op_records.get((n.op_type, cfg.hardware))
        rec = grid.get(feats) if grid is not None else None
        if rec is not None:
            out[nid] = (rec.mean_duration_us + gap, "ExactRecord")
            continue
        key = (n.op_type, cfg.hardware)
        if key not in models:
            g_recs = db.op_records.get(key, {})
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                models[key] = _fit([g_recs[k] for k in sorted(g_recs)])
        m = models[key]
        fmap = dict(feats)
        if m is not None and all(name in fmap for name in m[0]):
            out[nid] = (predict_value(m[1], m[2], [fmap[name] for name in m[0]]) + gap, "FittedModel")
            continue
        c = _comm(g, n, db, cfg)
        if c is not None:
            out[nid] = (c, "CommFormula")
            continue
        unknown[nid] = n.op_type
    if unknown:
        raise OracleUnknownOp(unknown)
    return out


# ----------------------------------------------------------------------------- engine


def successors(g):
    # graph.py:122-131: consumers sorted, with multiplicity, dangling refs skipped
    succ = {nid: [] for nid in g.nodes}
    for n in g.nodes.values():
        for pid, _ in n.inputs:
            if pid in succ:
                succ[pid].append(n.id)
    return {k: sorted(v) for k, v in succ.items()}


def simulate(g, durs: dict):
    """Event loop of engine.py:96-146; returns (entries, makespan, busy)."""
    remaining = {nid: len(n.inputs) for nid, n in g.nodes.items()}
    succ = successors(g)
    devs = set(g.devices) | {n.device for n in g.nodes.values()}
    fifo = {d: [] for d in devs}
    head = {d: 0 for d in devs}
    running = {}
    placed = {}
    heap = []

    def push_ready(ids, t):
        for nid in sorted(ids):
            fifo[g.nodes[nid].device].append((nid, t))

    def launch(now):
        for d in sorted(devs):
            if d in running or head[d] == len(fifo[d]):
                continue
            nid, ready = fifo[d][head[d]]
            head[d] += 1
            s = max(free.get(d, 0.0), ready)
            f = s + durs[nid]
            placed[nid] = (s, f)
            running[d] = nid
            heapq.heappush(heap, (f, nid, d))

    free = {}
    push_ready([nid for nid, c in remaining.items() if c == 0], 0.0)
    launch(0.0)
    while heap:
        now = heap[0][0]
        fresh = []
        while heap and heap[0][0] == now:
            _, nid, d = heapq.heappop(heap)
            del running[d]
            free[d] = now
            for m in succ[nid]:
                remaining[m] -= 1
                if remaining[m] == 0:
                    fresh.append(m)
        push_ready(fresh, now)
        launch(now)
    if len(placed) != len(g.nodes):
        raise OracleCycle(sorted(set(g.nodes) - set(placed)))
    entries = sorted(((s, g.nodes[nid].device, nid, f) for nid, (s, f) in placed.items()))
    entries = [(nid, dev, s, f) for s, dev, nid, f in entries]
    makespan = max((e[3] for e in entries), default=0.0)
    busy = {d: 0.0 for d in g.devices}
    for nid, dev, s, f in entries:
        busy[dev] = busy.get(dev, 0.0) + (f - s)
    return entries, makespan, busy


def critical_path(g, durs: dict):
    """graph.py:446-485 on an explicit duration map."""
    if not g.nodes:
        return 0.0, []
    succ = successors(g)
    indeg = {nid: len(n.inputs) for nid, n in g.nodes.items()}
    left = dict(indeg)
    heap = sorted(nid for nid, c in left.items() if c == 0)
    order = []
    while heap:
        nid = heapq.heappop(heap)
        order.append(nid)
        for m in succ[nid]:
            left[m] -= 1
            if left[m] == 0:
                heapq.heappush(heap, m)
    if len(order) != len(g.nodes):
        raise OracleCycle(sorted(nid for nid, c in left.items() if c > 0))
    suffix = {}
    for nid in reversed(order):
        best = 0.0
        for m in succ[nid]:
            if suffix[m] > best:
                best = suffix[m]
        suffix[nid] = durs[nid] + best
    sources = [nid for nid in order if indeg[nid] == 0]
    length = max(suffix[s] for s in sources)
    node = min(s for s in sources if suffix[s] == length)
    path = [node]
    while succ[node]:
        top = max(suffix[m] for m in succ[node])
        node = min(m for m in succ[node] if suffix[m] == top)
        path.append(node)
    return length, path


def run_candidate(g, db, cfg):
    """The reference's per-candidate path (cli.py:83-87 without file I/O)."""
    if cfg.replicas > 1 or cfg.device_map:
        g = expand(g, cfg)[0]
    table = estimate(g, db, cfg)
    durs = {k: v[0] for k, v in table.items()}
    entries, makespan, busy = simulate(g, durs)
    cp = critical_path(g, {nid: f - s for nid, _, s, f in entries})
    return makespan, cp[0], entries, busy, cp[1]


# ----------------------------------------------------------------------------- reporting


def _union(spans):
    """Union components of closed intervals, in start order (reporting.py:92-99)."""
    comps = []
    for lo, hi in sorted(spans):
        if comps and lo <= comps[-1][1]:
            if hi > comps[-1][1]:
                comps[-1][1] = hi
        else:
            comps.append([lo, hi])
    return comps


def _overlap(a, b):
    """Two-pointer intersection length of two component lists (reporting.py:102-114)."""
    i = j = 0
    total = 0.0
    while i < len(a) and j < len(b):
        lo = a[i][0] if a[i][0] >= b[j][0] else b[j][0]
        hi = a[i][1] if a[i][1] <= b[j][1] else b[j][1]
        if hi > lo:
            total += hi - lo
        if a[i][1] <= b[j][1]:
            i += 1
        else:
            j += 1
    return total


def summarize(entries, op_type: dict, kinds: dict, busy: dict, makespan: float, cp, top_k: int = 10):
    """reporting.summarize on oracle entries [(nid, device, start, finish)] in entry order.

    ``op_type[nid]`` is the node's op type, ``kinds[device]`` the device kind of the
    graph's device table (absent -> Compute), ``cp`` the critical_path result on
    finish - start.  Returns the SummaryReport fields as a dict."""
    totals = {}
    compute = comm = 0.0
    cspans, mspans = [], []
    for nid, dev, s, f in entries:
        key = op_type[nid] or nid
        totals[key] = totals.get(key, 0.0) + (f - s)
        if kinds.get(dev, COMPUTE) == COMPUTE:
            compute += f - s
            cspans.append((s, f))
        else:
            comm += f - s
            mspans.append((s, f))
    grand = sum(totals.values())
    ranked = sorted(totals.items(), key=lambda kv: (-kv[1], kv[0]))[: max(0, top_k)]
    return {
        "makespan_us": makespan,
        "per_device_busy_us": dict(busy),
        "utilization": {d: (b / makespan if makespan > 0 else 0.0) for d, b in busy.items()},
        "device_kinds": dict(kinds),
        "top_k_ops": [[k, t, (t / grand if grand > 0 else 0.0)] for k, t in ranked],
        "compute_us": compute,
        "comm_us": comm,
        "overlap_us": _overlap(_union(cspans), _union(mspans)),
        "critical_path_nodes": list(cp[1]),
        "critical_path_us": cp[0],
    }


def _json_str(x: str) -> str:
    out = ['"']
    for ch in x:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch in "\n\r\t\b\f":
            out.append({"\n": "\\n", "\r": "\\r", "\t": "\\t", "\b": "\\b", "\f": "\\f"}[ch])
        elif o < 0x20 or o > 0x7E:
            if o > 0xFFFF:
                o -= 0x10000
                out.append("\\u%04x\\u%04x" % (0xD800 | (o >> 10), 0xDC00 | (o & 0x3FF)))
            else:
                out.append("\\u%04x" % o)
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def to_trace(entries, op_type: dict, source: dict, devices) -> str:
    """reporting.to_trace: ``devices`` = the schedule's busy-dict keys; entries as in summarize."""
    devs = sorted(devices)
    tid = {d: i for i, d in enumerate(devs)}
    parts = []
    for d in devs:
        parts.append(' {\n  "name": "thread_name",\n  "ph": "M",\n  "pid": 0,\n  "tid": %d,\n  "args": {\n'
                     '   "name": %s\n  }\n }' % (tid[d], _json_str(d)))
    for nid, dev, s, f in entries:
        parts.append(' {\n  "name": %s,\n  "ph": "X",\n  "ts": %d,\n  "dur": %d,\n  "pid": 0,\n  "tid": %d,\n'
                     '  "args": {\n   "node": %s,\n   "source": %s\n  }\n }'
                     % (_json_str(op_type[nid] or nid), round(s), round(f - s), tid.get(dev, len(devs)),
                        _json_str(nid), _json_str(source[nid])))
    return ("[\n" + ",\n".join(parts) + "\n]\n") if parts else "[]\n"
