"""Drop-in ``expand_data_parallel`` (strategy.py:170-282) with the CSR built on the GPU.

Host side (strings, once per topology class): marker matching (strategy.py:188-200),
clone / collective ids (162-167) and their code-point ranks, device strings, the
validation findings that the reference's ``validate(expanded)`` would raise
(graph.py:331-385) for properties inherited from the base graph.  Device side
(K1, csrc/expand.cu): per-edge rewiring, rank-sorted successor CSR with
multiplicity, in-degree, devices, sources, FIFO capacities, topological order.
The returned ExpandedGraph carries the device CSR, so simulating it needs no
second lowering.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import native
from .errors import ConfigError, DfsimError, PatternWarning
from .lowering import LoweredGraph, _dev_tensor, match_pattern, upload
from .model import (
    COLLECTIVE,
    COMPUTE,
    DEVICE_COLLECTIVE,
    DEVICE_COMPUTE,
    TRANSFER,
    DataflowGraph,
    DeviceSpec,
    ExpandedGraph,
    OpNode,
    check_pattern,
)


def _positive_number(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool) and v > 0


def marked_gradients(g, cfg) -> list[str]:
    """strategy.py:188-200."""
    marked: list[str] = []
    for pattern in cfg.gradient_markers:
        check_pattern(pattern)
        hit = sorted(nid for nid in g.nodes if match_pattern(pattern, nid))
        if not hit:
            warnings.warn(f"gradient marker {pattern!r} matched no node", PatternWarning, stacklevel=3)
        marked.extend(nid for nid in hit if nid not in marked)
    marked.sort()
    for nid in marked:
        node = g.nodes[nid]
        if node.kind != COMPUTE:
            raise ConfigError(f"gradient marker matched {node.kind} node {nid!r}; only Compute nodes are supported")
        if not node.output_shapes or node.output_shapes[0].byte_size() <= 0:
            raise ConfigError(f"gradient node {nid!r} has no positive-size output tensor to reduce")
    return marked


class ExpansionPlan:
    """Strings and ranks of one topology class (host), plus its device CSR (K1).

    ``sync`` "allreduce" is strategy.py:170-282; "parameter_server" is this repo's PS
    expansion (ps.py: push / aggregate / pull nodes on per-worker links), emitted by the
    same K1 launch in PS mode.  Host node objects (``graph``) are built on first use only:
    the batched path needs the ids, ranks and CSR, not the objects."""

    def __init__(self, g, cfg, device: int | None = None, build_objects: bool = True, run_k1: bool = True,
                 db=None, sync: str | None = None):
        R = cfg.replicas
        self.sync = sync or getattr(cfg, "sync", "allreduce")
        ps = self.sync == "parameter_server"
        self.ps_device = getattr(cfg, "ps_device", "ps0")
        path = cfg.collective.path
        link = None
        if ps:  # ps.py's checks, in its order
            from .model import SCENARIO_GPU_GPU_UNI

            if R < 2 or len(cfg.device_map) != R:
                raise ConfigError("parameter-server expansion needs replicas >= 2 and a device_map")
            if self.ps_device in cfg.device_map:
                raise ConfigError(f"PS device {self.ps_device!r} collides with a worker device")
            link = db.link_records.get((SCENARIO_GPU_GPU_UNI, path, 2)) if db is not None else None
            if link is None:
                raise ConfigError(f"no {SCENARIO_GPU_GPU_UNI}/{path}/2 link record for the PS links")
        if cfg.device_map and len(cfg.device_map) != R:
            raise ConfigError(f"device_map has {len(cfg.device_map)} entries for {R} replicas")
        if R > 1 and not cfg.device_map:
            raise ConfigError("device_map is required when replicas > 1")
        self.marked = marked = marked_gradients(g, cfg)
        base_ids = list(g.nodes)
        N0 = len(base_ids)
        base_index = {nid: i for i, nid in enumerate(base_ids)}
        dmap = tuple(cfg.device_map)
        clone_dev = [[(dmap[k] if (dmap and g.nodes[nid].kind == COMPUTE) else g.nodes[nid].device)
                      for nid in base_ids] for k in range(R)]
        group = list(dmap) if dmap else sorted({d for row in clone_dev for d in row})
        self.fabric = fabric = f"collective:{path}:" + "+".join(group)
        clone_ids = [f"{nid}@r{k}" for k in range(R) for nid in base_ids]
        self.origin = dict(zip(clone_ids, [("clone", nid) for nid in base_ids] * R))
        self.link = link
        if ps:  # per gradient: R pushes, the aggregate, R pulls (ps.ps_nodes order)
            self.up_links = [f"link:{path}:{w}->{self.ps_device}" for w in dmap]
            self.down_links = [f"link:{path}:{self.ps_device}->{w}" for w in dmap]
            push_ids = [[f"push_{gid}@r{k}" for k in range(R)] for gid in marked]
            agg_ids = [f"aggregate_{gid}" for gid in marked]
            pull_ids = [[f"pull_{gid}@r{k}" for k in range(R)] for gid in marked]
            coll_ids = agg_ids
            added = [x for gi in range(len(marked)) for x in (push_ids[gi] + [agg_ids[gi]] + pull_ids[gi])]
            for gid, pu, ag, pl in zip(marked, push_ids, agg_ids, pull_ids):
                for cid in pu + [ag] + pl:
                    self.origin[cid] = ("ps", gid)
        else:
            coll_ids = [f"allreduce_{gid}" for gid in marked] if R > 1 else []
            added = coll_ids
            self.origin.update({cid: ("coll", gid) for gid, cid in zip(marked, coll_ids)})
        all_ids = clone_ids + added
        if len(self.origin) != len(all_ids):
            seen = set(clone_ids)
            dup = next(c for c in added if c in seen)
            raise DfsimError(f"collective id {dup!r} collides with an existing node")
        if not ps:
            self._validate_inherited(g, base_index, R, marked, group)
        order = sorted(range(len(all_ids)), key=all_ids.__getitem__)
        self._order = order
        self.ids = [all_ids[i] for i in order]
        rank = np.empty(len(all_ids), dtype=np.int32)
        rank[np.asarray(order, dtype=np.int64)] = np.arange(len(all_ids), dtype=np.int32)
        devset = {d for row in clone_dev for d in row}
        if ps and marked:
            devset.update([self.ps_device] + self.up_links + self.down_links)
        elif coll_ids:
            devset.add(fabric)
        self.devices = sorted(devset)
        drank = {d: i for i, d in enumerate(self.devices)}
        self.R, self.N0, self.G = R, N0, len(coll_ids)
        self.cfg, self.base_ids, self.clone_dev, self.coll_ids, self.group = cfg, base_ids, clone_dev, coll_ids, group
        self._g, self._graph = g, None
        # base arrays
        in_off = np.zeros(N0 + 1, dtype=np.int32)
        in_src, remap, marked_idx, base_dev = [], np.zeros(N0, np.uint8), np.full(N0, -1, np.int32), []
        gidx = {gid: i for i, gid in enumerate(marked)} if R > 1 else {}
        max_in = 0
        for v, nid in enumerate(base_ids):
            node = g.nodes[nid]
            for pid, _ in node.inputs:
                in_src.append(base_index.get(pid, -1))
            in_off[v + 1] = len(in_src)
            max_in = max(max_in, len(node.inputs))
            remap[v] = 1 if (dmap and node.kind == COMPUTE) else 0
            base_dev.append(drank.get(node.device, -1))
            if nid in gidx:
                marked_idx[v] = gidx[nid]
        self.max_indeg = max(max_in, R if coll_ids else 0)
        if not run_k1:  # host strings only (ids, origins, collective nodes); no device arrays
            self.ctx, self.lowered = None, None
            return
        ctx = native.Context.get(device)
        self.ctx = ctx
        d = ctx.device
        n_clone, G = R * N0, len(coll_ids)
        if ps:  # added ids are grouped per gradient: R pushes, aggregate, R pulls
            added_rank = rank[n_clone:].reshape(G, 2 * R + 1) if G else np.zeros((0, 2 * R + 1), np.int32)
            coll_rank = added_rank[:, R]
            push_rank, pull_rank = added_rank[:, :R].ravel(), added_rank[:, R + 1:].ravel()
        else:
            coll_rank, push_rank, pull_rank = rank[n_clone:], np.zeros(1, np.int32), np.zeros(1, np.int32)
        up = upload(dict(
            in_off=(in_off, np.int32), in_src=(in_src, np.int32), base_dev=(base_dev, np.int32),
            remap=(remap, np.uint8), marked=(marked_idx, np.int32), clone_rank=(rank[:n_clone], np.int32),
            coll_rank=(coll_rank, np.int32), map_dev=([drank[x] for x in dmap] if dmap else [0], np.int32),
            push_rank=(push_rank, np.int32), pull_rank=(pull_rank, np.int32),
            up_dev=([drank[x] for x in self.up_links] if ps and G else [0], np.int32),
            down_dev=([drank[x] for x in self.down_links] if ps and G else [0], np.int32)), d)
        self._keep = k = list(up.values())  # one host-to-device copy; order as listed
        base = native.BaseGraph(N0, native.ptr(k[0]), native.ptr(k[1]), native.ptr(k[2]), native.ptr(k[3]),
                                native.ptr(k[4]), len(in_src))
        plan = native.ExpandPlan(R, G, native.ptr(k[5]), native.ptr(k[6]), native.ptr(k[7]), drank.get(fabric, 0),
                                 int(ps), native.ptr(k[8]), native.ptr(k[9]), native.ptr(k[10]), native.ptr(k[11]),
                                 drank.get(self.ps_device, 0))
        self._structs = (base, plan, len(in_src))
        self.lowered = self._run_k1(ctx, base, plan, len(in_src))
        if self.lowered.n_ordered != self.lowered.n:
            raise DfsimError("internal: expansion produced an invalid graph: graph contains a cycle")
        if build_objects:
            _ = self.graph

    @property
    def graph(self) -> DataflowGraph:
        """The expanded graph's host objects (built on first use)."""
        if self._graph is None and getattr(self, "_g", None) is not None:
            self._graph = self._objects(self._g, self.cfg)
        return self._graph

    @property
    def device_specs(self) -> dict:
        """DeviceSpec of every device the expansion adds (PS links need their throughput)."""
        if self.sync != "parameter_server":
            return {}
        return {lid: DeviceSpec(lid, "Link", self.cfg.hardware, self.link.throughput_mbps, self.link.latency_us)
                for lid in self.up_links + self.down_links}

    def op_kind(self):
        """op type and kind code (0 Compute, 1 Transfer, 2 Collective) of every id, without objects:
        the base nodes' once, repeated per replica, the added nodes' by construction (ps.ps_nodes /
        collective_node), then permuted into rank order."""
        from .ps import AGGREGATE_OP, PULL_OP, PUSH_OP

        code = {COMPUTE: 0, TRANSFER: 1, COLLECTIVE: 2}
        base = [self._g.nodes[nid] for nid in self.base_ids]
        ops = [n.op_type for n in base] * self.R
        kinds = [code.get(n.kind, 2) for n in base] * self.R
        if self.sync == "parameter_server":
            per = [PUSH_OP] * self.R + [AGGREGATE_OP] + [PULL_OP] * self.R
            ops += per * self.G
            kinds += ([1] * self.R + [0] + [1] * self.R) * self.G
        else:
            ops += ["AllReduce"] * self.G
            kinds += [2] * self.G
        order = self._order
        return [ops[i] for i in order], [kinds[i] for i in order]

    def _validate_inherited(self, g, base_index, R, marked, group):
        """Findings of validate(expanded) that come from the base graph (graph.py:331-381).
        Every replica clones the same nodes, so one pass decides validity; the findings are
        only spelled out (per replica, in the reference's order) when there are some."""
        if self._inherited_ok(g):
            return
        findings = []
        for k in range(R):
            for nid, node in g.nodes.items():
                cid = f"{nid}@r{k}"
                for pid, slot in node.inputs:
                    if pid not in g.nodes:
                        findings.append(f"node {cid!r} references missing producer {pid + '@r' + str(k)!r}")
                    elif not 0 <= slot < max(1, len(g.nodes[pid].output_shapes)):
                        prod = f"allreduce_{pid}" if (R > 1 and pid in marked) else f"{pid}@r{k}"
                        findings.append(f"node {cid!r} references invalid slot {slot} of {prod!r}")
                if node.kind == COLLECTIVE:
                    grp = node.attrs.get("group")
                    if not isinstance(grp, (list, tuple)) or len(grp) < 2:
                        findings.append(f"collective {cid!r} needs attr 'group' with >= 2 devices")
                    if not _positive_number(node.attrs.get("bytes")):
                        findings.append(f"collective {cid!r} needs attr 'bytes' > 0")
                if node.kind == TRANSFER:
                    src, dst = node.attrs.get("src_device"), node.attrs.get("dst_device")
                    if src is None or dst is None or src == dst:
                        findings.append(f"transfer {cid!r} needs distinct 'src_device' and 'dst_device'")
                    if not _positive_number(node.attrs.get("bytes")):
                        findings.append(f"transfer {cid!r} needs attr 'bytes' > 0")
                if len(findings) >= 5:
                    break
        if findings:
            raise DfsimError("internal: expansion produced an invalid graph: " + "; ".join(findings[:5]))

    @staticmethod
    def _inherited_ok(g) -> bool:
        nodes = g.nodes
        for node in nodes.values():
            for pid, slot in node.inputs:
                prod = nodes.get(pid)
                if prod is None or not 0 <= slot < max(1, len(prod.output_shapes)):
                    return False
            if node.kind == COLLECTIVE:
                grp = node.attrs.get("group")
                if not isinstance(grp, (list, tuple)) or len(grp) < 2 or not _positive_number(node.attrs.get("bytes")):
                    return False
            elif node.kind == TRANSFER:
                src, dst = node.attrs.get("src_device"), node.attrs.get("dst_device")
                if src is None or dst is None or src == dst or not _positive_number(node.attrs.get("bytes")):
                    return False
        return True

    def reexpand(self, topo: bool = True, check: bool = False) -> None:
        """Run K1 again into the same device arrays (timed per-class device work).

        ``topo=False`` skips the Kahn order (the fused path uses the class level order);
        ``check=True`` reads the counts back (synchronising) and compares them."""
        base, plan, n_refs = self._structs
        lg = self.lowered
        N, D = len(self.ids), len(self.devices)
        cap = self.R * n_refs + self.G * self.R * (3 if self.sync == "parameter_server" else 1)
        by = native.ctypes.byref
        P0 = native.P(0)
        if not check:
            self.ctx.call("dfsim_expand_dp", by(base), by(plan), native.ptr(lg.t_succ_off), native.ptr(lg.t_succ_idx),
                          cap, native.ptr(lg.t_indeg), native.ptr(lg.t_dev), native.ptr(lg.t_sources),
                          native.ptr(lg.t_queue_off), native.ptr(lg.t_topo) if topo else P0, D, None, None, None)
            return
        n_edges, n_src, n_ord = native.I64(0), native.I32(0), native.I32(0)
        self.ctx.call("dfsim_expand_dp", by(base), by(plan), native.ptr(lg.t_succ_off), native.ptr(lg.t_succ_idx),
                      cap, native.ptr(lg.t_indeg), native.ptr(lg.t_dev), native.ptr(lg.t_sources),
                      native.ptr(lg.t_queue_off), native.ptr(lg.t_topo) if topo else P0, D, by(n_edges),
                      by(n_src), by(n_ord))
        if (int(n_edges.value), int(n_src.value), int(n_ord.value)) != (lg.n_edges, lg.n_sources,
                                                                         lg.n_ordered if topo else lg.n):
            raise DfsimError("internal: re-expansion disagrees with the first expansion")

    def _run_k1(self, ctx, base, plan, n_refs) -> LoweredGraph:
        import torch

        N = len(self.ids)
        D = len(self.devices)
        dev = f"cuda:{ctx.device}"
        cap = self.R * n_refs + self.G * self.R * (3 if self.sync == "parameter_server" else 1)
        z = lambda n: torch.empty(max(n, 1), dtype=torch.int32, device=dev)  # noqa: E731
        succ_off, succ_idx, indeg, device = z(N + 1), z(cap), z(N), z(N)
        sources, queue_off, topo = z(N), z(D + 1), z(N)
        n_edges, n_src, n_ord = native.I64(0), native.I32(0), native.I32(0)
        by = native.ctypes.byref
        ctx.call("dfsim_expand_dp", by(base), by(plan), native.ptr(succ_off), native.ptr(succ_idx), cap,
                 native.ptr(indeg), native.ptr(device), native.ptr(sources), native.ptr(queue_off), native.ptr(topo),
                 D, by(n_edges), by(n_src), by(n_ord))
        return LoweredGraph.from_arrays(self.ids, self.devices, succ_off, succ_idx, indeg, device, sources, queue_off,
                                        topo, int(n_edges.value), int(n_src.value), self.max_indeg, ctx,
                                        int(n_ord.value))

    def collective_node(self, gid, grad) -> OpNode:
        """AllReduce node of gradient ``gid`` (strategy.py:239-251)."""
        return OpNode(f"allreduce_{gid}", "AllReduce", self.fabric, COLLECTIVE,
                      {"group": list(self.group), "bytes": grad.output_shapes[0].byte_size(),
                       "path": self.cfg.collective.path},
                      tuple((f"{gid}@r{k}", 0) for k in range(self.R)), grad.output_shapes)

    def _objects(self, g, cfg) -> DataflowGraph:
        """Host node/device objects in the reference's insertion order (strategy.py:202-276);
        PS mode: ps.expand_parameter_server's objects."""
        if self.sync == "parameter_server":
            from .ps import expand_parameter_server

            gx = expand_parameter_server(g, cfg, _LinkDB(self.link, cfg.collective.path), self.ps_device).graph
            if self.lowered is not None:
                object.__setattr__(gx, "_dfsim_b200_lowered", ((len(gx.nodes), len(gx.devices), self.ctx.device),
                                                               self.lowered))
            return gx
        R, marked = self.R, set(self.marked) if self.R > 1 else set()
        nodes = {}
        for k in range(R):
            for v, nid in enumerate(self.base_ids):
                n = g.nodes[nid]
                ins = tuple(((f"allreduce_{p}" if p in marked else f"{p}@r{k}"), s) for p, s in n.inputs)
                cid = f"{nid}@r{k}"
                nodes[cid] = OpNode(cid, n.op_type, self.clone_dev[k][v], n.kind, n.attrs, ins, n.output_shapes)
        for gid, cid in zip(self.marked, self.coll_ids):
            nodes[cid] = self.collective_node(gid, g.nodes[gid])
        devices = {}
        coll = set(self.coll_ids)
        for n in nodes.values():
            if n.id in coll or n.device in devices:
                continue
            devices[n.device] = g.devices[n.device] if n.device in g.devices else \
                DeviceSpec(n.device, DEVICE_COMPUTE, cfg.hardware)
        if self.coll_ids:
            devices[self.fabric] = DeviceSpec(self.fabric, DEVICE_COLLECTIVE, cfg.hardware, 1.0, 0.0)
        meta = dict(g.metadata)
        meta["replicas"] = R
        gx = DataflowGraph(nodes=nodes, devices=devices, metadata=meta)
        if self.lowered is not None:
            object.__setattr__(gx, "_dfsim_b200_lowered", ((len(nodes), len(devices), self.ctx.device),
                                                           self.lowered))
        return gx


def expand_data_parallel(g, cfg, device: int | None = None) -> ExpandedGraph:
    """strategy.py:170-282; the expanded graph's CSR is built by K1 on the GPU."""
    plan = ExpansionPlan(g, cfg, device, sync="allreduce")  # the reference has no PS
    replica_of = {f"{nid}@r{k}": (nid, k) for k in range(plan.R) for nid in plan.base_ids}
    return ExpandedGraph(graph=plan.graph, replica_of=replica_of, collective_nodes=list(plan.coll_ids))


def expand_class(g, cfg, device: int | None = None) -> ExpansionPlan:
    return ExpansionPlan(g, cfg, device)


def path_roles(g, cfg, db=None):
    """The sorted device list an expansion of ``g`` under ``cfg`` produces, with the devices it
    adds written with the collective path as a placeholder (ExpansionPlan's device logic).

    Configs of one path-free class key whose roles agree expand to the same ids, CSR and device
    ranks for every path: only the added devices' names and the PS links' attributes depend on
    the path, so they share one topology class (batch.group_classes).  None when the expansion
    would fail -- such configs keep a class of their own, whose construction raises the
    reference's error."""
    from .model import SCENARIO_GPU_GPU_UNI

    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            marked = marked_gradients(g, cfg)
    except DfsimError:
        return None
    R, dmap, path = cfg.replicas, tuple(cfg.device_map), cfg.collective.path
    ps = getattr(cfg, "sync", "allreduce") == "parameter_server"
    psd = getattr(cfg, "ps_device", "ps0")
    base, compute = set(), False
    for n in g.nodes.values():
        if dmap and n.kind == COMPUTE:
            compute = True
        else:
            base.add(n.device)
    if compute:
        base.update(dmap)
    added = {}
    if ps:
        if R < 2 or len(dmap) != R or psd in dmap:
            return None
        if db is None or db.link_records.get((SCENARIO_GPU_GPU_UNI, path, 2)) is None:
            return None
        if marked:
            added[psd] = psd
            for w in dmap:
                added[f"link:{path}:{w}->{psd}"] = f"link:\x00:{w}->{psd}"
                added[f"link:{path}:{psd}->{w}"] = f"link:\x00:{psd}->{w}"
    elif R > 1 and marked:
        group = list(dmap) if dmap else sorted(base)
        added[f"collective:{path}:" + "+".join(group)] = "collective:\x00:" + "+".join(group)
    return tuple(added.get(d, d) for d in sorted(base | set(added)))


def ps_link_specs(cfg, db, ps_device: str) -> dict:
    """DeviceSpec of the PS links an expansion under ``cfg`` adds (ps.py: the path's
    gpu-gpu-uni row gives every link's throughput and latency)."""
    from .model import SCENARIO_GPU_GPU_UNI

    path = cfg.collective.path
    link = db.link_records[(SCENARIO_GPU_GPU_UNI, path, 2)]
    out = {}
    for lid in ([f"link:{path}:{w}->{ps_device}" for w in cfg.device_map]
                + [f"link:{path}:{ps_device}->{w}" for w in cfg.device_map]):
        out[lid] = DeviceSpec(lid, "Link", cfg.hardware, link.throughput_mbps, link.latency_us)
    return out


class _LinkDB:
    """The one profile-DB row expand_parameter_server reads (the PS links' gpu-gpu-uni row)."""

    def __init__(self, link, path):
        from .model import SCENARIO_GPU_GPU_UNI

        self.link_records = {(SCENARIO_GPU_GPU_UNI, path, 2): link}
