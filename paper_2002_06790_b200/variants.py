"""Graph variants: graphs with identical structure (ids, kinds, devices, inputs) whose
attributes and shapes differ -- e.g. one training graph per batch size.  They share one
topology class; only the per-node estimate inputs (features, comm attributes) are
per variant (``LoweredProfiles(variant_rows=...)``).

Rows of an expanded class are derived from the variant's *base* graph by origin, using
the reference's own ``node_features`` (costmodel.py:226-246) on small stand-in graphs, so
no feature semantics are re-implemented: a clone's features equal its base node's (its
producers are clones or the collective, all carrying the base producers' shapes), a
collective's / PS node's features come from the node built exactly as the expansion
builds it.  ``tests/test_variants.py`` pins the rows against fully materialised graphs.
"""

from __future__ import annotations

import numpy as np

from .lowering import FEATURES, ROW_FIELDS, _i64, base_arrays, node_features, node_rows, row_arrays
from .model import DEVICE_LINK, TRANSFER


class _Stand:
    """Graph stand-in for node_features/node_rows: nodes by id + devices."""

    def __init__(self, nodes, devices):
        self.nodes, self.devices = nodes, devices


class StructureKey:
    """Everything that shapes a topology class (ids, kinds, devices, op types, inputs; not
    attrs or shapes), compared exactly: the hash is computed once, and equal hashes are
    confirmed on the full tuples, so two structures never share a class by a hash collision."""

    __slots__ = ("t", "h")

    def __init__(self, t):
        self.t, self.h = t, hash(t)

    def __hash__(self):
        return self.h

    def __eq__(self, other):
        return self is other or (isinstance(other, StructureKey) and self.h == other.h and self.t == other.t)


def structure_key(g) -> StructureKey:
    return StructureKey((tuple((nid, n.kind, n.device, n.op_type, n.inputs) for nid, n in g.nodes.items()),
                         tuple(sorted((d.id, d.kind) for d in g.devices.values()))))


def rows_for(kind: str, ids, g_b, structure, cfg=None, db=None) -> list:
    """Estimate-input rows (rank order ``ids``) of variant graph ``g_b`` as node_rows tuples
    (reference path of ``variant_arrays``; tests/test_variants.py pins both)."""
    arr = variant_arrays(kind, ids, g_b, structure, cfg, db, {})
    rows = FEATURES.rows
    return [(rows[f], int(ok), int(b), int(gs), float(thr), float(lat))
            for f, ok, b, gs, thr, lat in zip(*(arr[k].tolist() for k in ROW_FIELDS))]


def _special_rows(kind, ids, pos, g_b, structure, cfg, db=None) -> dict:
    """Rows of the nodes a class adds (AllReduce / PS push, aggregate, pull) at positions
    ``pos``, each built exactly as the expansion builds it, with the reference's own
    node_features on a stand-in graph."""
    out = []
    if kind == "dp":
        plan = structure
        for p in pos:
            gid = plan.origin[ids[p]][1]
            grad = g_b.nodes[gid]
            node = plan.collective_node(gid, grad)
            stand = {f"{gid}@r{k}": grad for k in range(plan.R)}
            out.append(node_rows(_Stand({**stand, node.id: node}, {}), [node.id])[0])
    else:
        from .expansion import ps_link_specs
        from .ps import ps_nodes

        from .ps import ps_link_ids

        # the PS links (throughput, latency) of this config's collective path
        specs = ps_link_specs(cfg, db, cfg.ps_device) if db is not None else structure.device_specs
        up, down = ps_link_ids(cfg, cfg.ps_device)
        R = cfg.replicas
        rows0 = {}
        for p in pos:
            cid = ids[p]
            gid = structure.origin[cid][1]
            if gid not in rows0:
                # push_<g>@r<k> / pull_<g>@r<k> differ across k only in their link device (the
                # features -- bytes, the gradient's shapes -- are k-independent): worker 0's nodes
                # and the aggregate are built as the expansion builds them, the other workers' rows
                # are worker 0's with their own link's throughput / latency
                grad = g_b.nodes[gid]
                push0, agg, pull0 = ps_nodes(gid, grad, cfg, cfg.ps_device, replicas=(0,))
                nodes = {f"{gid}@r{k}": grad for k in range(R)}
                nodes.update({f"push_{gid}@r{k}": grad for k in range(R)})  # the aggregate's inputs: shapes only
                nodes.update({push0.id: push0, agg.id: agg, pull0.id: pull0})
                stand = _Stand(nodes, specs)
                rows0[gid] = ({n.id: node_rows(stand, [n.id])[0] for n in (push0, agg, pull0)}, stand)
            r0, stand = rows0[gid]
            if cid.startswith("aggregate_"):
                out.append(r0[cid])
                continue
            push = cid.startswith("push_")
            k = int(cid.rsplit("@r", 1)[1])
            row = r0[f"push_{gid}@r0" if push else f"pull_{gid}@r0"]
            dev = specs.get((up if push else down)[k])
            if row[1] and dev is not None and dev.kind == DEVICE_LINK:
                row = row[:4] + (dev.throughput_mbps, dev.latency_us)
            elif k:  # a link without a Link spec: the row as node_rows gives it for this node
                node = ps_nodes(gid, g_b.nodes[gid], cfg, cfg.ps_device, replicas=(k,))[0 if push else 2]
                row = node_rows(_Stand({**stand.nodes, node.id: node}, specs), [cid])[0]
            out.append(row)
    return row_arrays(out)


def variant_arrays(kind: str, ids, g_b, structure, cfg=None, db=None, cache=None) -> dict:
    """Estimate-input rows (rank order ``ids``) of variant graph ``g_b`` for a class of
    ``kind`` "plain" | "dp" | "ps" (structure: ExpansionPlan), as
    arrays (lowering.ROW_FIELDS; features as FEATURES ids).

    A clone's row is its base node's (its producers are clones or the collective, all carrying
    the base producers' shapes): gathered from the graph's cached base rows.  The rows of the
    added nodes depend on the class and on the output shapes of the marked gradients only, so
    ``cache`` (one dict per class) keeps them per distinct gradient-shape tuple -- graph
    variants that differ in batch size share their weight-gradient shapes."""
    cache = {} if cache is None else cache
    base, index = base_arrays(g_b)
    if "perm" not in cache:  # same structure => same node order in every variant graph
        if kind == "plain":
            perm, special = [index[nid] for nid in ids], []
        else:
            origin = structure.origin
            perm, special = [], []
            for p, cid in enumerate(ids):
                what, gid = origin[cid]
                if what == "clone":
                    perm.append(index[gid])
                else:
                    perm.append(0)
                    special.append(p)
        cache["perm"], cache["special"] = np.asarray(perm, np.int64), np.asarray(special, np.int64)
        cache["grads"] = list(dict.fromkeys(structure.origin[ids[p]][1] for p in special)) if special else []
    perm, special = cache["perm"], cache["special"]
    out = {k: base[k][perm] for k in ROW_FIELDS}
    if len(special):
        nodes = g_b.nodes  # key: the gradients' output shapes as plain tuples (cheap to hash)
        key = tuple((s.dims, s.dtype_bytes) for gid in cache["grads"] for s in nodes[gid].output_shapes)
        rows = cache.get(("special", key))
        if rows is None:
            rows = cache[("special", key)] = _special_rows(kind, ids, special.tolist(), g_b, structure, cfg, db)
        for k in ROW_FIELDS:
            out[k][special] = rows[k]
    return out


__all__ = ["StructureKey", "structure_key", "rows_for", "variant_arrays", "variant_arrays_many", "node_features"]


def variant_arrays_many(kind: str, ids, graphs, structure, cfg=None, db=None, cfgs=None) -> dict:
    """``variant_arrays`` of several graph variants of one class, stacked: each field [GV, N].
    Vectorised over the variants: one gather of the stacked base rows, and the added nodes'
    rows once per distinct gradient-shape tuple (and, for PS classes, collective path:
    ``cfgs[v]`` is variant v's config, whose path sets the PS links' attributes)."""
    cache: dict = {}
    variant_arrays(kind, ids, graphs[0], structure, cfg, db, cache)  # fills perm / special / grads
    perm, special, grads = cache["perm"], cache["special"], cache["grads"]
    bases = [base_arrays(gb)[0] for gb in graphs]
    out = {k: np.stack([b[k] for b in bases])[:, perm] for k in ROW_FIELDS}
    if len(special):
        groups: dict = {}
        gkey = tuple(grads)
        for v, gb in enumerate(graphs):
            memo = gb.__dict__.get("_dfsim_grad_keys")
            if memo is None:
                memo = {}
                try:
                    object.__setattr__(gb, "_dfsim_grad_keys", memo)
                except (AttributeError, TypeError):
                    pass
            key = memo.get(gkey)
            if key is None:
                nodes = gb.nodes
                key = memo[gkey] = tuple((s.dims, s.dtype_bytes) for gid in grads for s in nodes[gid].output_shapes)
            vcfg = cfgs[v] if cfgs is not None else cfg
            groups.setdefault((key, vcfg.collective.path if kind == "ps" else None), []).append(v)
        for (key, _), vs in groups.items():
            vcfg = cfgs[vs[0]] if cfgs is not None else cfg
            same = kind != "ps" or vcfg.collective.path == cfg.collective.path
            rows = cache.get(("special", key)) if same else None
            if rows is None:
                rows = _special_rows(kind, ids, special.tolist(), graphs[vs[0]], structure, vcfg, db)
            sel = np.ix_(np.asarray(vs, np.int64), special)
            for k in ROW_FIELDS:
                out[k][sel] = rows[k]
    if kind != "plain":
        _respec_transfers(out, ids, graphs, structure, [cfgs[v] if cfgs is not None else cfg
                                                        for v in range(len(graphs))], db)
    return out


def _replaced_devices(structure, cfg, db) -> dict:
    """Devices whose spec an expansion under ``cfg`` writes over the base graph's: the
    allreduce fabric (a Collective spec, strategy.py:263-271) when there are collectives; the
    PS device (Compute) and the PS links (the path's Link spec, ps.py)."""
    from .expansion import ps_link_specs
    from .model import DEVICE_COLLECTIVE, DEVICE_COMPUTE, DeviceSpec

    path = cfg.collective.path
    if getattr(cfg, "sync", "allreduce") == "parameter_server":
        out = ps_link_specs(cfg, db, structure.ps_device)
        out[structure.ps_device] = DeviceSpec(structure.ps_device, DEVICE_COMPUTE, cfg.hardware)
        return out
    if not structure.coll_ids:
        return {}
    fabric = f"collective:{path}:" + "+".join(structure.group)
    return {fabric: DeviceSpec(fabric, DEVICE_COLLECTIVE, cfg.hardware, 1.0, 0.0)}


def _respec_transfers(out, ids, graphs, structure, cfgs, db):
    """A base transfer on a device the expansion replaces (a device literally named like the
    fabric, a PS link or the PS device) is estimated against the replacing spec, as the
    reference estimates the expanded graph (costmodel.py:354-359): its clones' rows are
    rewritten.  Such a collision is class-uniform (expansion.path_roles splits the path off),
    so this is a no-op for every class of a normal sweep."""
    g0 = graphs[0]
    tdevs = {n.device for n in g0.nodes.values() if n.kind == TRANSFER}
    if not tdevs:
        return
    pos_of = None
    for v, (gb, cfg) in enumerate(zip(graphs, cfgs)):
        specs = {d: sp for d, sp in _replaced_devices(structure, cfg, db).items() if d in tdevs}
        if not specs:
            continue
        if pos_of is None:
            pos_of = {}
            for p, cid in enumerate(ids):
                what, gid = structure.origin[cid]
                n = g0.nodes[gid] if what == "clone" else None
                if n is not None and n.kind == TRANSFER and n.device in tdevs:
                    pos_of.setdefault(n.device, []).append((p, gid))
        for d, spec in specs.items():
            for p, gid in pos_of.get(d, ()):
                b = gb.nodes[gid].attrs.get("bytes")
                link = spec.kind == DEVICE_LINK and isinstance(b, int)
                out["ok"][v, p] = 1 if link else 0
                out["bytes"][v, p] = _i64(b) if link else 0
                out["gsize"][v, p] = 0
                out["thr"][v, p] = spec.throughput_mbps if link else 1.0
                out["lat"][v, p] = spec.latency_us if link else 0.0

