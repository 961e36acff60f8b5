"""Host-side data model of the drop-in surface.

These are plain containers with the reference's field names, so an object built
with the reference's own classes (``dfsim.graph.DataflowGraph``,
``dfsim.costmodel.DurationTable``, ``dfsim.strategy.StrategyConfig``,
``dfsim.profiledb.ProfileDB``) can be passed to this framework unchanged and
vice versa.  Field lists follow:

* TensorShape / DeviceSpec / OpNode / DataflowGraph -- pkg/src/dfsim/graph.py:32-135
* OpSignature / ProfileRecord / LinkRecord / ProfileDB -- profiledb.py:24-104
* LinearCostModel / DurationEntry / DurationTable -- costmodel.py:50-90
* StrategyConfig / CollectiveConfig / ExpandedGraph -- strategy.py:31-54
* Schedule / ScheduledNode -- engine.py:27-58

The document readers (``parse_graph``, ``load_profiles``, ``parse_config``) are
host I/O run once per input file; they accept the reference's documents
(graph.py:192-293, profiledb.py:164-208, strategy.py:93-142).  No simulation
arithmetic lives here.
"""

from __future__ import annotations

import json
import math
import warnings
from dataclasses import dataclass, field

from .errors import (
    ConfigError,
    GraphFormatError,
    GraphFormatWarning,
    ProfileFormatError,
)

COMPUTE, TRANSFER, COLLECTIVE = "Compute", "Transfer", "Collective"
NODE_KINDS = (COMPUTE, TRANSFER, COLLECTIVE)
DEVICE_COMPUTE, DEVICE_LINK, DEVICE_COLLECTIVE = "Compute", "Link", "CollectiveResource"
DEVICE_KINDS = (DEVICE_COMPUTE, DEVICE_LINK, DEVICE_COLLECTIVE)

SCENARIO_GPU_GPU_UNI = "gpu-gpu-uni"
SCENARIO_GPU_GPU_BI = "gpu-gpu-bi"
SCENARIO_HOST_TO_GPU = "host-to-gpu"
SCENARIO_GPU_TO_HOST = "gpu-to-host"
SCENARIO_NCCL_ALLREDUCE = "nccl-allreduce"

ALGO_MEASURED = "MeasuredThroughput"
ALGO_RING = "RingAnalytic"
COLLECTIVE_ALGOS = (ALGO_MEASURED, ALGO_RING)

SOURCE_OVERRIDE = "Override"
SOURCE_EXACT = "ExactRecord"
SOURCE_FITTED = "FittedModel"
SOURCE_COMM = "CommFormula"
# device-side source tags (u8) -> strings; order is part of the C-ABI
SOURCE_TAGS = (SOURCE_OVERRIDE, SOURCE_EXACT, SOURCE_FITTED, SOURCE_COMM)


# ----------------------------------------------------------------------------- graph


@dataclass(frozen=True)
class TensorShape:
    dims: tuple[int, ...]
    dtype_bytes: int = 4

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        if min(dims, default=0) < 0:
            raise ValueError(f"negative dimension in {dims}")
        if self.dtype_bytes <= 0:
            raise ValueError(f"dtype_bytes must be positive, got {self.dtype_bytes}")
        object.__setattr__(self, "dims", dims)

    def num_elements(self) -> int:
        return math.prod(self.dims)

    def byte_size(self) -> int:
        return self.dtype_bytes * self.num_elements()


@dataclass(frozen=True)
class DeviceSpec:
    id: str
    kind: str
    hardware: str = ""
    throughput_mbps: float | None = None
    latency_us: float = 0.0

    def __post_init__(self):
        if self.kind not in DEVICE_KINDS:
            raise ValueError(f"unknown device kind {self.kind!r}")
        if self.kind == DEVICE_COMPUTE:
            if self.throughput_mbps is not None:
                raise ValueError(f"Compute device {self.id!r} must not carry throughput")
            return
        if self.throughput_mbps is None or self.throughput_mbps <= 0:
            raise ValueError(f"{self.kind} device {self.id!r} needs positive throughput")
        if self.latency_us < 0:
            raise ValueError(f"{self.kind} device {self.id!r} has negative latency")


@dataclass(frozen=True)
class OpNode:
    id: str
    op_type: str
    device: str
    kind: str = COMPUTE
    attrs: dict = field(default_factory=dict)
    inputs: tuple[tuple[str, int], ...] = ()
    output_shapes: tuple[TensorShape, ...] = ()

    def __post_init__(self):
        if not self.id or ":" in self.id:
            raise ValueError(f"bad node id {self.id!r}")
        if self.kind not in NODE_KINDS:
            raise ValueError(f"node {self.id!r}: unknown kind {self.kind!r}")
        object.__setattr__(self, "inputs", tuple((str(p), int(s)) for p, s in self.inputs))
        object.__setattr__(self, "output_shapes", tuple(self.output_shapes))


@dataclass
class DataflowGraph:
    nodes: dict
    devices: dict
    metadata: dict = field(default_factory=dict)

    def in_degree(self) -> dict[str, int]:
        return {nid: len(n.inputs) for nid, n in self.nodes.items()}


def make_graph(nodes, devices, metadata=None) -> DataflowGraph:
    nmap, dmap = {}, {}
    for n in nodes:
        if n.id in nmap:
            raise GraphFormatError(f"duplicate node id {n.id!r}")
        nmap[n.id] = n
    for d in devices:
        if d.id in dmap:
            raise GraphFormatError(f"duplicate device id {d.id!r}")
        dmap[d.id] = d
    return DataflowGraph(nodes=nmap, devices=dmap, metadata=dict(metadata or {}))


def _doc(text: str, err):
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise err(f"syntax error: {exc.msg} (line {exc.lineno})") from exc
    if not isinstance(doc, dict):
        raise err("document must be an object")
    return doc


_NODE_REQUIRED = ("id", "op", "kind", "device")
_NODE_FIELDS = set(_NODE_REQUIRED) | {"attrs", "inputs", "output_shapes"}
_DEVICE_FIELDS = {"id", "kind", "hardware", "throughput_mbps", "latency_us"}


def parse_graph(text: str) -> DataflowGraph:
    """Read a reference graph document (graph.py:192-293 format)."""
    doc = _doc(text, GraphFormatError)
    if "format_version" not in doc:
        raise GraphFormatError("missing required field 'format_version'")
    if str(doc["format_version"]).split(".", 1)[0] != "1":
        raise GraphFormatError(f"unsupported graph format version {doc['format_version']!r}")
    for key in sorted(set(doc) - {"format_version", "metadata", "devices", "nodes"}):
        warnings.warn(f"ignoring unknown graph field {key!r}", GraphFormatWarning, stacklevel=2)
    devices = []
    for i, d in enumerate(doc.get("devices", [])):
        if not isinstance(d, dict) or "id" not in d or "kind" not in d:
            raise GraphFormatError("device entry needs 'id' and 'kind'", location=f"devices[{i}]")
        for key in sorted(set(d) - _DEVICE_FIELDS):  # graph.py:217-219
            warnings.warn(f"ignoring unknown device field {key!r}", GraphFormatWarning, stacklevel=2)
        try:
            devices.append(DeviceSpec(d["id"], d["kind"], d.get("hardware", ""),
                                      d.get("throughput_mbps"), d.get("latency_us", 0.0)))
        except (KeyError, TypeError, ValueError) as exc:
            raise GraphFormatError(str(exc), location=f"devices[{i}]") from exc
    nodes = []
    for i, nd in enumerate(doc.get("nodes", [])):
        loc = f"nodes[{i}]"
        if not isinstance(nd, dict):
            raise GraphFormatError("node entry must be an object", location=loc)
        for fieldname in _NODE_REQUIRED:  # graph.py:230-233
            if fieldname not in nd:
                raise GraphFormatError(f"missing required node field {fieldname!r}", location=loc)
        for key in sorted(set(nd) - _NODE_FIELDS):  # graph.py:234-236
            warnings.warn(f"ignoring unknown node field {key!r}", GraphFormatWarning, stacklevel=2)
        try:
            refs = []
            for ref in nd.get("inputs", []):
                pid, sep, slot = ref.rpartition(":")
                if not sep:
                    raise GraphFormatError(f"input reference {ref!r} is not 'nodeId:slot'", loc)
                refs.append((pid, int(slot)))
            shapes = tuple(TensorShape(tuple(s["dims"]), s.get("dtype_bytes", 4))
                           for s in nd.get("output_shapes", []))
            nodes.append(OpNode(nd["id"], nd["op"], nd["device"], nd["kind"],
                                dict(nd.get("attrs", {})), tuple(refs), shapes))
        except GraphFormatError:
            raise
        except (KeyError, TypeError, ValueError) as exc:
            raise GraphFormatError(str(exc), location=loc) from exc
    g = make_graph(nodes, devices, doc.get("metadata", {}))
    for n in g.nodes.values():
        for pid, slot in n.inputs:
            if pid not in g.nodes:
                raise GraphFormatError(f"node {n.id!r} references missing producer {pid!r}", n.id)
            if not 0 <= slot < max(1, len(g.nodes[pid].output_shapes)):
                raise GraphFormatError(f"node {n.id!r} references bad slot {slot} of {pid!r}", n.id)
    return g


def serialize_graph(g) -> str:
    """Write a graph in the reference document format (graph.py:296-325)."""
    devs = []
    for d in g.devices.values():
        e = {"id": d.id, "kind": d.kind, "hardware": d.hardware}
        if d.kind != DEVICE_COMPUTE:
            e["throughput_mbps"], e["latency_us"] = d.throughput_mbps, d.latency_us
        devs.append(e)
    nodes = [{"id": n.id, "op": n.op_type, "kind": n.kind, "device": n.device,
              "attrs": dict(n.attrs), "inputs": [f"{p}:{s}" for p, s in n.inputs],
              "output_shapes": [{"dims": list(s.dims), "dtype_bytes": s.dtype_bytes}
                                for s in n.output_shapes]}
             for n in g.nodes.values()]
    return json.dumps({"format_version": 1, "metadata": dict(g.metadata),
                       "devices": devs, "nodes": nodes}, indent=2) + "\n"


# ----------------------------------------------------------------------------- profiles


@dataclass(frozen=True)
class OpSignature:
    op_type: str
    hardware: str
    arg_features: tuple = ()

    def __post_init__(self):
        feats = tuple(sorted((str(n), float(v)) for n, v in self.arg_features))
        names = [n for n, _ in feats]
        if len(set(names)) != len(names):
            raise ValueError(f"duplicate feature names in {names}")
        if not all(math.isfinite(v) for _, v in feats):
            raise ValueError(f"non-finite feature value in {feats}")
        object.__setattr__(self, "arg_features", feats)


@dataclass(frozen=True)
class ProfileRecord:
    signature: OpSignature
    mean_duration_us: float
    stderr_us: float = 0.0
    samples: int = 1

    def __post_init__(self):
        if self.mean_duration_us <= 0:
            raise ValueError(f"mean_duration must be > 0, got {self.mean_duration_us}")
        if self.stderr_us < 0 or self.samples < 1:
            raise ValueError("bad stderr/samples")


@dataclass(frozen=True)
class LinkRecord:
    scenario: str
    path: str
    participants: int
    throughput_mbps: float
    latency_us: float = 0.0

    def __post_init__(self):
        if self.participants < 1:
            raise ValueError(f"participants must be >= 1, got {self.participants}")
        if not math.isfinite(self.throughput_mbps) or self.throughput_mbps <= 0:
            raise ValueError(f"throughput must be finite and > 0, got {self.throughput_mbps}")
        if self.latency_us < 0:
            raise ValueError(f"latency must be >= 0, got {self.latency_us}")


@dataclass
class ProfileDB:
    op_records: dict = field(default_factory=dict)     # (op, hw) -> {features: record}
    link_records: dict = field(default_factory=dict)   # (scenario, path, n) -> LinkRecord
    hardware_tags: list = field(default_factory=list)
    provenance: str = ""
    replaced: int = 0


def db_insert(db: ProfileDB, rec) -> None:
    """In-place insert; identical keys collapse, last wins (profiledb.py:128-158)."""
    if isinstance(rec, LinkRecord) or hasattr(rec, "scenario"):
        key = (rec.scenario, rec.path, rec.participants)
        db.replaced += key in db.link_records
        db.link_records[key] = rec
    else:
        sig = rec.signature
        grid = db.op_records.setdefault((sig.op_type, sig.hardware), {})
        db.replaced += sig.arg_features in grid
        grid[sig.arg_features] = rec


def load_profiles(text: str) -> ProfileDB:
    """Read a reference profile-db document (profiledb.py:164-208 format)."""
    doc = _doc(text, ProfileFormatError)
    if str(doc.get("format_version", "")).split(".", 1)[0] != "1":
        raise ProfileFormatError(f"unsupported profile-db format version {doc.get('format_version')!r}")
    db = ProfileDB(hardware_tags=list(doc.get("hardware_tags", [])), provenance=doc.get("provenance", ""))
    for i, r in enumerate(doc.get("op_records", [])):
        try:
            s = r["signature"]
            db_insert(db, ProfileRecord(
                OpSignature(s["op_type"], s["hardware"], tuple((n, v) for n, v in s.get("arg_features", []))),
                r["mean_duration"], r.get("stderr", 0.0), r.get("samples", 1)))
        except (KeyError, TypeError, ValueError) as exc:
            raise ProfileFormatError(f"op_records[{i}]: {exc}") from exc
    for i, r in enumerate(doc.get("link_records", [])):
        try:
            db_insert(db, LinkRecord(r["scenario"], r["path"], r["participants"],
                                     r["throughput"], r.get("latency", 0.0)))
        except (KeyError, TypeError, ValueError) as exc:
            raise ProfileFormatError(f"link_records[{i}]: {exc}") from exc
    return db


def save_profiles(db) -> str:
    ops = []
    for key in sorted(db.op_records):
        for feats in sorted(db.op_records[key]):
            r = db.op_records[key][feats]
            ops.append({"signature": {"op_type": r.signature.op_type, "hardware": r.signature.hardware,
                                      "arg_features": [[n, v] for n, v in r.signature.arg_features]},
                        "mean_duration": r.mean_duration_us, "stderr": r.stderr_us, "samples": r.samples})
    links = [{"scenario": r.scenario, "path": r.path, "participants": r.participants,
              "throughput": r.throughput_mbps, "latency": r.latency_us}
             for _, r in sorted(db.link_records.items())]
    return json.dumps({"format_version": 1, "hardware_tags": list(db.hardware_tags),
                       "provenance": db.provenance, "op_records": ops, "link_records": links},
                      indent=2) + "\n"


# ----------------------------------------------------------------------------- cost model types


@dataclass(frozen=True)
class FitStats:
    r_squared: float
    max_rel_residual: float
    n_points: int


@dataclass(frozen=True)
class LinearCostModel:
    op_type: str
    hardware: str
    feature_names: tuple
    coefficients: tuple
    intercept: float
    fit_stats: FitStats

    def __post_init__(self):
        if len(self.coefficients) != len(self.feature_names):
            raise ValueError("one coefficient per feature required")


@dataclass(frozen=True)
class DurationEntry:
    duration_us: float
    source: str

    def __post_init__(self):
        if not self.duration_us >= 0.0:
            raise ValueError(f"durations are nonnegative microseconds, got {self.duration_us}")


@dataclass
class DurationTable:
    entries: dict = field(default_factory=dict)

    def durations(self) -> dict[str, float]:
        return {nid: e.duration_us for nid, e in self.entries.items()}


# ----------------------------------------------------------------------------- strategy


@dataclass(frozen=True)
class CollectiveConfig:
    algo: str = ALGO_MEASURED
    path: str = "PCIeSwitch"


@dataclass(frozen=True)
class StrategyConfig:
    replicas: int = 1
    device_map: tuple = ()
    collective: CollectiveConfig = CollectiveConfig()
    gradient_markers: tuple = ()
    overrides: dict = field(default_factory=dict)
    hardware: str = ""
    op_gap_us: float = 0.0
    # extension (not in the reference; its parse_config ignores unknown keys, strategy.py:93-142):
    # "allreduce" (strategy.py:170-282) or "parameter_server" (ps.py)
    sync: str = "allreduce"
    ps_device: str = "ps0"


SYNC_ALLREDUCE, SYNC_PS = "allreduce", "parameter_server"


@dataclass
class ExpandedGraph:
    graph: DataflowGraph
    replica_of: dict
    collective_nodes: list


def check_pattern(pattern: str) -> None:
    """Literal id or prefix + one trailing '*' (strategy.py:60-66)."""
    if not pattern:
        raise ConfigError("empty pattern")
    star = pattern.find("*")
    if star not in (-1, len(pattern) - 1):
        raise ConfigError(f"pattern {pattern!r}: '*' is only allowed as a trailing glob")


def parse_config(text: str) -> StrategyConfig:
    """Read a reference strategy document (strategy.py:93-142 format)."""
    doc = _doc(text, ConfigError)
    if str(doc.get("format_version", 1)).split(".", 1)[0] != "1":
        raise ConfigError(f"unsupported config format version {doc.get('format_version')!r}")
    replicas = doc.get("replicas", 1)
    if not isinstance(replicas, int) or replicas < 1:
        raise ConfigError(f"replicas must be an integer >= 1, got {replicas!r}")
    dmap = tuple(doc.get("device_map", ()))
    if dmap and len(dmap) != replicas:
        raise ConfigError(f"device_map has {len(dmap)} entries for {replicas} replicas")
    if replicas > 1 and not dmap:
        raise ConfigError("device_map is required when replicas > 1")
    if len(set(dmap)) != len(dmap):
        raise ConfigError("device_map entries must be distinct")
    coll = doc.get("collective", {})
    algo = coll.get("algo", ALGO_MEASURED)
    if algo not in COLLECTIVE_ALGOS:
        raise ConfigError(f"unknown collective algo {algo!r}; expected one of {COLLECTIVE_ALGOS}")
    markers = tuple(doc.get("gradient_markers", ()))
    for p in markers:
        check_pattern(p)
    overrides = dict(doc.get("overrides", {}))
    for p, v in overrides.items():
        check_pattern(p)
        if not isinstance(v, (int, float)) or isinstance(v, bool) or v < 0:
            raise ConfigError(f"override for {p!r} must be a duration >= 0, got {v!r}")
    gap = doc.get("op_gap_us", 0.0)
    if not isinstance(gap, (int, float)) or gap < 0:
        raise ConfigError(f"op_gap_us must be >= 0, got {gap!r}")
    sync = doc.get("sync", SYNC_ALLREDUCE)
    if sync not in (SYNC_ALLREDUCE, SYNC_PS):
        raise ConfigError(f"unknown sync {sync!r}; expected {SYNC_ALLREDUCE!r} or {SYNC_PS!r}")
    return StrategyConfig(replicas, dmap, CollectiveConfig(algo, coll.get("path", "PCIeSwitch")),
                          markers, {k: float(v) for k, v in overrides.items()},
                          doc.get("hardware", ""), float(gap), sync, doc.get("ps_device", "ps0"))


# ----------------------------------------------------------------------------- schedule


@dataclass(frozen=True)
class ScheduledNode:
    node_id: str
    device: str
    start_us: float
    finish_us: float
    source: str
    op_type: str = ""


@dataclass
class Schedule:
    entries: list
    makespan_us: float
    per_device_busy_us: dict = field(default_factory=dict)

    def by_node(self) -> dict:
        return {e.node_id: e for e in self.entries}

    def to_json(self) -> str:
        """Canonical form, byte-compatible with engine.py:48-58."""
        return json.dumps({
            "makespan_us": self.makespan_us,
            "per_device_busy_us": dict(sorted(self.per_device_busy_us.items())),
            "entries": [[e.node_id, e.device, e.start_us, e.finish_us, e.source, e.op_type]
                        for e in self.entries],
        })


def utilization(s) -> dict[str, float]:
    """Busy fraction per device (engine.py:218-222); host-side ratio of kernel outputs."""
    if s.makespan_us <= 0:
        return {d: 0.0 for d in s.per_device_busy_us}
    return {d: b / s.makespan_us for d, b in s.per_device_busy_us.items()}
