"""Parameter-server expansion (SURVEY.md §8a row PS) -- new code.

The reference declares parameter servers a non-goal
and only models allreduce (strategy.py:170-282).  This expansion builds a PS
training step out of the reference's own primitives, so the result is a plain
DataflowGraph that the reference's estimate_all / simulate semantics (and this
framework's kernels) evaluate unchanged:

  clone the graph per replica exactly like expand_data_parallel (strategy.py:202-217);
  for every marked gradient g and replica k:
     push_<g>@r<k>   Transfer  on  link:<path>:<dev_k>->ps   (transfer_time, costmodel.py:176-182)
  aggregate_<g>      Compute   on  the PS device             (profile record / fitted model)
     pull_<g>@r<k>   Transfer  on  link:<path>:ps-><dev_k>
  and every consumer of g@r<k> reads pull_<g>@r<k> instead (slot kept).

Each worker has its own uplink and downlink device (full duplex), so pushes of one
worker serialise on its uplink and pulls on its downlink, while the PS serialises
the aggregations.  Link devices take the throughput and latency of the profile
DB's ``gpu-gpu-uni`` row for the collective path (the row the reference's ring
fallback reads, costmodel.py:334-344).  Parity of the expansion itself is
unpinned (no reference); estimate + simulate of the emitted graph are pinned by
the oracle in tests/test_ps.py and tests/test_gpu_fuzz.py.
"""

from __future__ import annotations

from .errors import ConfigError
from .expansion import marked_gradients
from .model import (
    COMPUTE,
    DEVICE_COMPUTE,
    DEVICE_LINK,
    SCENARIO_GPU_GPU_UNI,
    TRANSFER,
    DataflowGraph,
    DeviceSpec,
    ExpandedGraph,
    OpNode,
)

PUSH_OP, PULL_OP, AGGREGATE_OP = "PushGradient", "PullParameters", "PSAggregate"


def expand_parameter_server(g, cfg, db, ps_device: str = "ps0") -> ExpandedGraph:
    """PS push/aggregate/pull expansion of ``g`` for ``cfg`` (replicas, device_map,
    gradient_markers, collective.path, hardware); see the module docstring."""
    R = cfg.replicas
    if R < 2 or len(cfg.device_map) != R:
        raise ConfigError("parameter-server expansion needs replicas >= 2 and a device_map")
    if ps_device in cfg.device_map:
        raise ConfigError(f"PS device {ps_device!r} collides with a worker device")
    path = cfg.collective.path
    link = db.link_records.get((SCENARIO_GPU_GPU_UNI, path, 2))
    if link is None:
        raise ConfigError(f"no {SCENARIO_GPU_GPU_UNI}/{path}/2 link record for the PS links")
    marked = set(marked_gradients(g, cfg))
    nodes: dict = {}
    replica_of: dict = {}
    for k in range(R):
        for nid, n in g.nodes.items():
            dev = cfg.device_map[k] if n.kind == COMPUTE else n.device
            ins = tuple(((f"pull_{p}@r{k}" if p in marked else f"{p}@r{k}"), s) for p, s in n.inputs)
            cid = f"{nid}@r{k}"
            nodes[cid] = OpNode(cid, n.op_type, dev, n.kind, n.attrs, ins, n.output_shapes)
            replica_of[cid] = (nid, k)
    devices = {}
    for n in list(nodes.values()):
        if n.device not in devices:
            devices[n.device] = g.devices.get(n.device) or DeviceSpec(n.device, DEVICE_COMPUTE, cfg.hardware)
    devices[ps_device] = DeviceSpec(ps_device, DEVICE_COMPUTE, cfg.hardware)
    for w in cfg.device_map:
        for lid in (f"link:{path}:{w}->{ps_device}", f"link:{path}:{ps_device}->{w}"):
            devices[lid] = DeviceSpec(lid, DEVICE_LINK, cfg.hardware, link.throughput_mbps, link.latency_us)
    comm_nodes = []
    origin = {cid: ("clone", nid) for cid, (nid, _k) in replica_of.items()}
    for gid in sorted(marked):
        for node in ps_nodes(gid, g.nodes[gid], cfg, ps_device):
            nodes[node.id] = node
            origin[node.id] = ("ps", gid)
            if node.kind == TRANSFER:
                comm_nodes.append(node.id)
    meta = dict(g.metadata)
    meta.update(replicas=R, sync="parameter_server")
    ex = ExpandedGraph(graph=DataflowGraph(nodes=nodes, devices=devices, metadata=meta),
                       replica_of=replica_of, collective_nodes=comm_nodes)
    ex.origin = origin
    return ex


def ps_link_ids(cfg, ps_device: str) -> tuple[list, list]:
    """(uplink ids, downlink ids) of the PS links, one per worker in device_map order."""
    path = cfg.collective.path
    return ([f"link:{path}:{w}->{ps_device}" for w in cfg.device_map],
            [f"link:{path}:{ps_device}->{w}" for w in cfg.device_map])


def ps_nodes(gid, grad, cfg, ps_device: str, replicas=None) -> list:
    """push_<g>@r<k>, aggregate_<g>, pull_<g>@r<k> for one marked gradient (module docstring);
    ``replicas``: only these workers' push / pull nodes (the aggregate always)."""
    R = cfg.replicas
    ks = range(R) if replicas is None else replicas
    up, down = ps_link_ids(cfg, ps_device)
    nbytes = grad.output_shapes[0].byte_size()
    out = []
    for k in ks:
        w = cfg.device_map[k]
        out.append(OpNode(f"push_{gid}@r{k}", PUSH_OP, up[k], TRANSFER,
                          {"src_device": w, "dst_device": ps_device, "bytes": nbytes},
                          ((f"{gid}@r{k}", 0),), grad.output_shapes))
    aid = f"aggregate_{gid}"
    out.append(OpNode(aid, AGGREGATE_OP, ps_device, COMPUTE,
                      {"replicas": R, "bytes": nbytes, "mflops": round(R * nbytes / 4 / 1e6, 6)},
                      tuple((f"push_{gid}@r{k}", 0) for k in range(R)), grad.output_shapes))
    for k in ks:
        w = cfg.device_map[k]
        out.append(OpNode(f"pull_{gid}@r{k}", PULL_OP, down[k], TRANSFER,
                          {"src_device": ps_device, "dst_device": w, "bytes": nbytes},
                          ((aid, 0),), grad.output_shapes))
    return out
