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

from .lowering import node_features, node_rows


class _Stand:
    """Graph stand-in for node_features/node_rows: nodes by id + devices."""

    def __init__(self, nodes, devices):
        self.nodes, self.devices = nodes, devices


def structure_key(g) -> int:
    """Hash of everything that shapes a topology class (not attrs or shapes)."""
    return hash((tuple((nid, n.kind, n.device, n.op_type, n.inputs) for nid, n in g.nodes.items()),
                 tuple(sorted((d.id, d.kind) for d in g.devices.values()))))


def rows_for(kind: str, ids, g_b, structure, cfg=None, db=None) -> list:
    """Estimate-input rows (rank order ``ids``) of variant graph ``g_b`` for a class of
    ``kind`` "plain" | "dp" (structure: ExpansionPlan) | "ps" (structure: ExpandedGraph)."""
    if kind == "plain":
        return node_rows(g_b, ids)
    base = getattr(g_b, "_dfsim_base_rows", None)  # shared by every class of this graph
    if base is None:
        base = dict(zip(list(g_b.nodes), node_rows(g_b, list(g_b.nodes))))
        try:
            object.__setattr__(g_b, "_dfsim_base_rows", base)
        except (AttributeError, TypeError):
            pass
    out = []
    if kind == "dp":
        plan = structure
        for cid in ids:
            what, gid = plan.origin[cid]
            if what == "clone":
                out.append(base[gid])
                continue
            grad = g_b.nodes[gid]
            node = plan.collective_node(gid, grad)
            stand = _Stand({f"{gid}@r{k}": grad for k in range(plan.R)}, {})
            out.append(node_rows(_Stand({**stand.nodes, node.id: node}, {}), [node.id])[0])
        return out
    if kind == "ps":
        from .ps import ps_nodes

        ex = structure
        gx = ex.graph
        built = {}
        for cid in ids:
            what, gid = ex.origin[cid]
            if what == "clone":
                out.append(base[gid])
                continue
            if gid not in built:
                grad = g_b.nodes[gid]
                nodes = {f"{gid}@r{k}": grad for k in range(cfg.replicas)}
                for n in ps_nodes(gid, grad, cfg, cfg.ps_device):
                    nodes[n.id] = n
                built[gid] = _Stand(nodes, gx.devices)
            stand = built[gid]
            out.append(node_rows(stand, [cid])[0])
        return out
    raise ValueError(kind)


__all__ = ["structure_key", "rows_for", "node_features"]
