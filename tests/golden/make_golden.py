"""Generate golden fixtures by running the REAL reference (dfsim) in this container.

Usage (only where /root/reference exists; the GPU box never runs this):

    python tests/golden/make_golden.py

Writes ``engine_cases.json.gz`` and ``pipeline_cases.json.gz`` next to this file.
Every expected value below is produced by the reference's own public functions:
``simulate`` (engine.py:96-146), ``critical_path`` (graph.py:446-485) applied to
``finish - start`` like ``summarize`` does (reporting.py:128,154),
``expand_data_parallel`` (strategy.py:170-282) and ``estimate_all``
(costmodel.py:282-331).  Inputs come from the reference's own generators
(synth.py) and the instance families of its tests (test_engine.py:33-36,
test_acceptance.py:40-48, test_costmodel.py, test_strategy.py).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
import warnings
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent


def _import_reference():
    if not REF.exists():
        sys.exit("reference not present; fixtures are generated only in the build container")
    sys.path.insert(0, str(REF / "src"))
    import dfsim  # noqa: F401
    return dfsim


dfsim = _import_reference()
from dfsim.costmodel import SOURCE_OVERRIDE, DurationEntry, DurationTable, estimate_all, node_signature  # noqa: E402
from dfsim.engine import simulate  # noqa: E402
from dfsim.errors import CycleError, DfsimError, MissingDurationError, UnknownOpError  # noqa: E402
from dfsim.graph import (  # noqa: E402
    COLLECTIVE, COMPUTE, TRANSFER, DeviceSpec, OpNode, TensorShape, critical_path, make_graph, serialize_graph,
)
from dfsim.reporting import summarize, to_trace  # noqa: E402
from dfsim.profiledb import LinkRecord, OpSignature, ProfileDB, ProfileRecord, _insert_inplace, load_profiles, save_profiles  # noqa: E402
from dfsim.strategy import CollectiveConfig, StrategyConfig, expand_data_parallel, parse_config, serialize_config  # noqa: E402
from dfsim.synth import DurationLaw, SplitMix64, SynthSpec, gen_durations, gen_graph, gen_profiles, parse_synth_spec  # noqa: E402


def mk_node(nid, inputs=(), device="gpu0", op="Op", kind=COMPUTE, attrs=None, shapes=None):
    # same builder as the reference's tests/conftest.py:29-38
    return OpNode(id=nid, op_type=op, device=device, kind=kind, attrs=dict(attrs or {}),
                  inputs=tuple((p, 0) for p in inputs),
                  output_shapes=tuple(shapes) if shapes else (TensorShape((4, 4), 4),))


def mk_graph(nodes, extra_devices=(), hardware="test-hw"):
    devices = {}
    for n in nodes:
        devices.setdefault(n.device, DeviceSpec(id=n.device, kind="Compute", hardware=hardware))
    for d in extra_devices:
        devices[d.id] = d
    return make_graph(list(nodes), list(devices.values()))


def mk_table(durs):
    return DurationTable(entries={k: DurationEntry(float(v), SOURCE_OVERRIDE) for k, v in durs.items()})


def table_doc(t: DurationTable):
    return {nid: [e.duration_us, e.source] for nid, e in t.entries.items()}


def run_engine(g, table):
    """Expected outputs: schedule (canonical json) + CP over finish-start, or the error."""
    try:
        s = simulate(g, table)
    except CycleError as exc:
        return {"error": "CycleError", "ids": exc.cycle}
    except MissingDurationError as exc:
        return {"error": "MissingDurationError", "ids": exc.node_ids}
    durs = {e.node_id: e.finish_us - e.start_us for e in s.entries}
    cp_len, cp_path = critical_path(g, durs)
    return {"schedule": json.loads(s.to_json()), "cp": [cp_len, cp_path], "summary": summary_doc(s, g),
            **trace_doc(s)}


def summary_doc(s, g, top_k=10):
    """reporting.summarize (reporting.py:117-162) of the schedule, JSON-ready."""
    r = summarize(s, g, top_k=top_k)
    return {"makespan_us": r.makespan_us, "per_device_busy_us": r.per_device_busy_us, "utilization": r.utilization,
            "device_kinds": r.device_kinds, "top_k_ops": [list(t) for t in r.top_k_ops], "compute_us": r.compute_us,
            "comm_us": r.comm_us, "overlap_us": r.overlap_us, "critical_path_nodes": r.critical_path_nodes,
            "critical_path_us": r.critical_path_us}


def trace_doc(s):
    """reporting.to_trace (reporting.py:43-74): sha256 of the document; the text itself for small schedules."""
    text = to_trace(s)
    out = {"trace_sha256": hashlib.sha256(text.encode()).hexdigest(), "trace_bytes": len(text.encode())}
    if len(s.entries) <= 12:
        out["trace"] = text
    return out


# ----------------------------------------------------------------------------- engine cases


def engine_cases():
    cases = []

    def add(name, g, table):
        cases.append({"name": name, "graph": serialize_graph(g), "durations": table_doc(table),
                      "expect": run_engine(g, table)})

    chain = mk_graph([mk_node("A"), mk_node("B", ["A"]), mk_node("C", ["B"])])
    add("chain", chain, mk_table({"A": 2, "B": 3, "C": 5}))
    add("parallel", mk_graph([mk_node("A", device="gpu0"), mk_node("B", device="gpu1")]),
        mk_table({"A": 3, "B": 5}))
    for two in (True, False):
        db_, dc_ = ("gpu0", "gpu1") if two else ("gpu0", "gpu0")
        g = mk_graph([mk_node("A"), mk_node("B", ["A"], device=db_), mk_node("C", ["A"], device=dc_),
                      mk_node("D", ["B", "C"])])
        add(f"diamond_{'two' if two else 'one'}", g, mk_table({"A": 1, "B": 2, "C": 4, "D": 1}))
    add("fifo_tiebreak", mk_graph([mk_node("A"), mk_node("z", ["A"]), mk_node("b", ["A"])]),
        mk_table({"A": 1, "z": 1, "b": 1}))
    zc = mk_graph([mk_node("A"), mk_node("B", ["A"]), mk_node("C", ["B"]), mk_node("D", ["C"])])
    add("zero_duration_chain", zc, mk_table({"A": 0, "B": 2, "C": 0, "D": 1}))
    add("all_zero", chain, mk_table({"A": 0, "B": 0, "C": 0}))
    anomaly = mk_graph([mk_node("n0", device="gpu1"), mk_node("n1", device="gpu0"),
                        mk_node("n2", ["n1"], device="gpu1"), mk_node("n3", ["n0"], device="gpu1"),
                        mk_node("n4", ["n2"], device="gpu0")])
    add("anomaly_base", anomaly, mk_table({"n0": 3, "n1": 4, "n2": 4, "n3": 3, "n4": 3}))
    add("anomaly_bumped", anomaly, mk_table({"n0": 4, "n1": 4, "n2": 4, "n3": 3, "n4": 3}))
    add("cycle", mk_graph([mk_node("A", ["B"]), mk_node("B", ["A"]), mk_node("C")]),
        mk_table({"A": 1, "B": 1, "C": 1}))
    add("missing_duration", chain, mk_table({"A": 1, "B": 1}))
    add("empty", make_graph([], []), mk_table({}))
    # duplicate references: one producer feeding the same consumer twice
    dup = mk_graph([mk_node("p"), OpNode("c", "Op", "gpu1", inputs=(("p", 0), ("p", 0))), mk_node("q", ["c"])])
    add("duplicate_refs", dup, mk_table({"p": 1.5, "c": 2.25, "q": 0.5}))
    # rank inversions of expanded ids (F4e): "a0@r0" < "a@r0", "x@r10" < "x@r2"
    inv_nodes = [mk_node(n, device=f"gpu{i % 3}") for i, n in enumerate(["a@r0", "a0@r0", "x@r10", "x@r2", "x@r1"])]
    add("rank_inversions", mk_graph(inv_nodes), mk_table({n.id: 1.0 for n in inv_nodes}))

    # summary / trace coverage: link + collective devices, empty op types (key = node id),
    # zero durations, start ties across devices, non-ASCII and escaped characters in ids
    links = [DeviceSpec(id="link:a", kind="Link", hardware="test-hw", throughput_mbps=1000.0, latency_us=1.0),
             DeviceSpec(id="fabric", kind="CollectiveResource", hardware="test-hw", throughput_mbps=1.0,
                        latency_us=0.0)]
    mixed = [mk_node("c0", op="Conv2D"), mk_node("c1", ["c0"], op=""), mk_node("t0", ["c0"], device="link:a",
             kind=TRANSFER, op="Send"), mk_node("t1", ["t0"], device="link:a", kind=TRANSFER, op="Send"),
             mk_node("ar", ["c1", "t1"], device="fabric", kind=COLLECTIVE, op="AllReduce"),
             mk_node("c2", ["c0"], device="gpu1", op="Conv2D"), mk_node("z\u00e9\"q", ["c2"], device="gpu1", op=""),
             mk_node("c3", ["ar"], op="Conv2D"), mk_node("c4", ["c2"], device="gpu1", op="MatMul")]
    add("summary_mixed", mk_graph(mixed, extra_devices=links),
        mk_table({"c0": 2.5, "c1": 0.0, "t0": 3.25, "t1": 1.5, "ar": 4.0, "c2": 1.0, "z\u00e9\"q": 2.0, "c3": 0.5,
                  "c4": 0.0}))
    for seed in range(6):
        rng = SplitMix64(seed + 77)
        g0 = gen_graph(SynthSpec(kind="RandomDAG", nodes=50 + 20 * seed, density=0.08, seed=500 + seed, num_devices=4))
        devs = [DeviceSpec(id=f"link:{k}", kind="Link", hardware="test-hw", throughput_mbps=100.0, latency_us=1.0)
                for k in range(2)]
        nodes = []
        for nid in sorted(g0.nodes):
            n = g0.nodes[nid]
            r = rng.randint(0, 9)
            if r < 3:
                n = OpNode(n.id, ("Send", "Recv", "")[r], f"link:{r % 2}", TRANSFER, n.attrs, n.inputs, n.output_shapes)
            elif r == 3:
                n = OpNode(n.id, "", n.device, n.kind, n.attrs, n.inputs, n.output_shapes)
            nodes.append(n)
        durs = {}
        for nid in sorted(g0.nodes):
            u = rng.uniform()
            durs[nid] = 0.0 if u < 0.1 else (float(rng.randint(1, 3)) * 0.1 if u < 0.3 else u * 7.0)
        add(f"summary_random_{seed}", mk_graph(nodes, extra_devices=devs), mk_table(durs))

    # random DAG families of the reference tests
    for seed in range(25):  # test_engine.random_instance
        g = gen_graph(SynthSpec(kind="RandomDAG", nodes=60, density=0.1, seed=seed, num_devices=3))
        add(f"random60_{seed}", g, gen_durations(g, DurationLaw("uniform", low=1, high=8), seed=seed ^ 0xBEEF))
    for seed in range(100):  # test_acceptance.oracle_instance (C1)
        nodes = 20 + (seed * 13) % 181
        devices = 1 + seed % 4
        density = 0.02 + (seed % 5) * 0.03
        g = gen_graph(SynthSpec(kind="RandomDAG", nodes=nodes, density=density, seed=seed, num_devices=devices))
        add(f"c1_{seed}", g, gen_durations(g, DurationLaw("uniform", low=1, high=8), seed=seed ^ 0x5EED))

    # float durations: exercises start+dur rounding, CP right-fold and exact == batching
    for seed in range(20):
        ndev = 1 + seed % 6
        g = gen_graph(SynthSpec(kind="RandomDAG", nodes=40 + 7 * seed, density=0.08, seed=1000 + seed, num_devices=ndev))
        rng = SplitMix64(seed * 7919 + 1)
        durs = {}
        for nid in sorted(g.nodes):
            r = rng.uniform()
            if r < 0.1:
                durs[nid] = 0.0
            elif r < 0.3:
                durs[nid] = float(rng.randint(1, 4)) * 0.1      # ties that are not exact in binary
            else:
                durs[nid] = rng.uniform() * 10.0
        add(f"float_{seed}", g, mk_table(durs))
    # one larger instance (still seconds for the reference)
    g = gen_graph(SynthSpec(kind="RandomDAG", nodes=1500, density=0.004, seed=4242, num_devices=8))
    rng = SplitMix64(99)
    add("float_large", g, mk_table({nid: rng.uniform() * 100.0 for nid in sorted(g.nodes)}))
    return cases


# ----------------------------------------------------------------------------- pipeline cases


def run_pipeline(g, db, cfg):
    """cli._run_one_simulation (cli.py:71-116) without file I/O."""
    out = {}
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            if cfg.replicas > 1 or cfg.device_map:
                ex = expand_data_parallel(g, cfg)
                g = ex.graph
                out["expanded"] = serialize_graph(g)
                out["collective_nodes"] = list(ex.collective_nodes)
                out["replica_of"] = {k: list(v) for k, v in ex.replica_of.items()}
            table = estimate_all(g, db, cfg)
    except UnknownOpError as exc:
        out["error"] = "UnknownOpError"
        out["nodes"] = exc.nodes
        return out
    except DfsimError as exc:
        out["error"] = type(exc).__name__
        out["message"] = str(exc)
        return out
    out["durations"] = table_doc(table)
    out.update(run_engine(g, table))
    return out


def pipeline_cases():
    cases = []

    def add(name, g, db, cfg):
        cases.append({"name": name, "graph": serialize_graph(g), "profiles": save_profiles(db),
                      "config": serialize_config(cfg), "expect": run_pipeline(g, db, cfg)})

    samples = REF / "samples"
    chain_spec = parse_synth_spec((samples / "chain.synth.json").read_text())
    add("chain_demo", gen_graph(chain_spec), gen_profiles(chain_spec),
        parse_config((samples / "single_replica.config.json").read_text()))
    cnn_spec = parse_synth_spec((samples / "layered_cnn.synth.json").read_text())
    add("layered_cnn_sample", gen_graph(cnn_spec), gen_profiles(cnn_spec),
        parse_config((samples / "layered_cnn.config.json").read_text()))

    spec16 = SynthSpec(kind="LayeredCNN", layers=16)
    g16, db16 = gen_graph(spec16), gen_profiles(spec16)
    for r in (1, 2, 4):  # C7 (test_acceptance.py:233-256)
        cfg = StrategyConfig(replicas=r, device_map=tuple(f"gpu{i}" for i in range(r)),
                             gradient_markers=("grad_conv_*",), overrides={"allreduce_*": 0.0} if r > 1 else {},
                             hardware=spec16.hardware)
        add(f"c7_r{r}", g16, db16, cfg)

    nvl = ProfileDB(op_records={k: dict(v) for k, v in db16.op_records.items()},
                    link_records=dict(db16.link_records), hardware_tags=list(db16.hardware_tags))
    _insert_inplace(nvl, LinkRecord("gpu-gpu-uni", "NVLink", 2, 858306.0, 2.0))
    for r, gap in ((8, 0.125), (3, 0.0), (5, 1e-3)):
        cfg = StrategyConfig(replicas=r, device_map=tuple(f"gpu{i}" for i in range(r)),
                             collective=CollectiveConfig("RingAnalytic", "NVLink"),
                             gradient_markers=("grad_conv_*",), hardware="synth-hw", op_gap_us=gap)
        add(f"layered_ring_nvlink_r{r}", g16, nvl, cfg)
    # Measured with the 8-participant record present, and without (ring fallback / unknown)
    for r, path in ((8, "PCIeSwitch"), (3, "PCIeSwitch"), (3, "NVLink"), (2, "RDMA")):
        cfg = StrategyConfig(replicas=r, device_map=tuple(f"gpu{i}" for i in range(r)),
                             collective=CollectiveConfig("MeasuredThroughput", path),
                             gradient_markers=("grad_conv_*",), hardware="synth-hw", op_gap_us=0.5)
        add(f"layered_measured_{path}_r{r}", g16, nvl, cfg)

    # Table 1 links + planted ops
    t1 = load_profiles((samples / "v100_table1.profdb").read_text())
    for key, grid in db16.op_records.items():
        for rec in grid.values():
            _insert_inplace(t1, rec)
    for r in (2, 4, 8):
        cfg = StrategyConfig(replicas=r, device_map=tuple(f"gpu{i}" for i in range(r)),
                             collective=CollectiveConfig("MeasuredThroughput", "PCIeSwitch"),
                             gradient_markers=("grad_conv_*", "grad_conv_0*"), hardware="synth-hw")
        add(f"table1_measured_r{r}", gen_graph(SynthSpec(kind="LayeredCNN", layers=5)), t1, cfg)

    # random DAG families with expansion (test_strategy.py:165-184) and planted profiles
    for seed in range(6):
        spec = SynthSpec(kind="RandomDAG", nodes=30, density=0.15, seed=seed, num_devices=1 + seed % 3)
        g = gen_graph(spec)
        db = gen_profiles(spec)
        for r in (1, 2, 4):
            markers = tuple(sorted(g.nodes)[::7])
            cfg = StrategyConfig(replicas=r, device_map=tuple(f"gpu{i}" for i in range(r)),
                                 gradient_markers=markers, hardware=spec.hardware, op_gap_us=0.25 * seed,
                                 collective=CollectiveConfig("MeasuredThroughput", "PCIeSwitch"))
            add(f"random30_s{seed}_r{r}", g, db, cfg)

    # --- estimate precedence (test_costmodel.py:263-413)
    HW = "test-hw"

    def grid_records(op, feat, slope, icpt, grid):
        return [ProfileRecord(OpSignature(op, HW, ((feat, x),)), slope * x + icpt) for x in grid]

    def db_of(records=(), links=()):
        db = ProfileDB()
        for r in list(records) + list(links):
            _insert_inplace(db, r)
        return db

    grid = [2.0 ** i for i in range(16)]
    solo = mk_graph([mk_node("solo", op="Conv2D", attrs={"in_channels": 24})])
    add("fitted_interp", solo, db_of(grid_records("Conv2D", "in_channels", 12.5, 40.0, grid)),
        StrategyConfig(hardware=HW))
    g8 = mk_graph([mk_node("solo", op="Conv2D", attrs={"in_channels": 8})])
    db = db_of(grid_records("Conv2D", "in_channels", 12.5, 40.0, grid))
    _insert_inplace(db, ProfileRecord(node_signature(g8, g8.nodes["solo"], HW), 777.0))
    add("exact_beats_model", g8, db, StrategyConfig(hardware=HW, op_gap_us=0.75))
    add("override_beats_exact", g8, db, StrategyConfig(hardware=HW, overrides={"solo": 5.0}))
    add("model_only", mk_graph([mk_node("solo", op="Conv2D", attrs={"in_channels": 7})]), db,
        StrategyConfig(hardware=HW, op_gap_us=0.1))
    add("unknown_op", mk_graph([mk_node("solo", op="MyCustomOp")]), ProfileDB(), StrategyConfig(hardware=HW))
    add("partial_unknown", mk_graph([mk_node("known", op="Conv2D", attrs={"in_channels": 8}), mk_node("weird", op="Mystery")]),
        db_of(grid_records("Conv2D", "in_channels", 2.0, 3.0, grid)), StrategyConfig(hardware=HW))
    link = DeviceSpec(id="pci", kind="Link", throughput_mbps=10000.0, latency_us=1.0)
    tnode = mk_node("t", kind=TRANSFER, device="pci", attrs={"src_device": "cpu0", "dst_device": "gpu0", "bytes": 2 ** 20})
    add("transfer_link", mk_graph([tnode], extra_devices=[link]), ProfileDB(), StrategyConfig(hardware=HW, op_gap_us=3.0))
    fabric = DeviceSpec(id="fabric", kind="CollectiveResource", throughput_mbps=1.0)
    c2 = mk_node("ar", kind=COLLECTIVE, device="fabric", attrs={"group": ["gpu0", "gpu1"], "bytes": 100 * 2 ** 20})
    add("collective_measured", mk_graph([c2], extra_devices=[fabric]),
        db_of(links=[LinkRecord("nccl-allreduce", "PCIeSwitch", 2, 11598.12)]), StrategyConfig(hardware=HW))
    c3 = mk_node("ar", kind=COLLECTIVE, device="fabric", attrs={"group": ["gpu0", "gpu1", "gpu2"], "bytes": 2 ** 20})
    add("collective_ring_fallback", mk_graph([c3], extra_devices=[fabric]),
        db_of(links=[LinkRecord("gpu-gpu-uni", "PCIeSwitch", 2, 12000.0, 0.5)]), StrategyConfig(hardware=HW))
    add("collective_ring_algo", mk_graph([c3], extra_devices=[fabric]),
        db_of(links=[LinkRecord("gpu-gpu-uni", "QPI", 2, 10948.81, 1.25), LinkRecord("nccl-allreduce", "QPI", 3, 5000.0)]),
        StrategyConfig(hardware=HW, collective=CollectiveConfig("RingAnalytic", "QPI")))
    add("collective_unknown", mk_graph([mk_node("ar", kind=COLLECTIVE, device="fabric", attrs={"group": ["g0", "g1"], "bytes": 4})],
                                       extra_devices=[fabric]), ProfileDB(), StrategyConfig(hardware=HW))
    # collective exact record overrides the formula (costmodel.py:307-311 before 323)
    cg = mk_graph([c2], extra_devices=[fabric])
    dbx = db_of(links=[LinkRecord("nccl-allreduce", "PCIeSwitch", 2, 11598.12)])
    _insert_inplace(dbx, ProfileRecord(node_signature(cg, cg.nodes["ar"], HW), 42.5))
    add("collective_exact_record", cg, dbx, StrategyConfig(hardware=HW, op_gap_us=9.0))
    # overlapping override patterns, last listed wins (test_strategy.py:207-226)
    og = mk_graph([mk_node("conv_a", op="Conv2D", attrs={"in_channels": 3}), mk_node("conv_b", ["conv_a"], op="Conv2D", attrs={"in_channels": 5}),
                   mk_node("conv_ax", ["conv_a"], op="Conv2D", attrs={"in_channels": 9}), mk_node("other", ["conv_b", "conv_ax"], op="Conv2D", attrs={"in_channels": 1})])
    add("override_last_wins", og, db_of(grid_records("Conv2D", "in_channels", 1.5, 2.0, grid)),
        StrategyConfig(hardware=HW, overrides={"conv_*": 10.0, "conv_a*": 20.0, "conv_ax": 30.0}, op_gap_us=0.5))
    # two-feature grid: predict's Neumaier sum over c*f terms (costmodel.py:164)
    rng = SplitMix64(31337)
    recs = []
    for i in range(24):
        x, y = float(rng.randint(1, 4096)), float(rng.randint(1, 512))
        recs.append(ProfileRecord(OpSignature("MatMul", HW, (("k", x), ("m", y))), 0.0173 * x + 3.1e-7 * x * y + 0.9 * y + 11.0))
    nodes = []
    for i in range(40):
        attrs = {"k": rng.randint(1, 100000) + rng.uniform(), "m": rng.randint(1, 700) * 1.0001}
        nodes.append(mk_node(f"mm{i:02d}", [f"mm{i - 1:02d}"] if i else [], op="MatMul", attrs=attrs,
                             device=f"gpu{i % 3}"))
    add("two_feature_fit", mk_graph(nodes), db_of(recs), StrategyConfig(hardware=HW, op_gap_us=1e-3))
    # negative-intercept law clamped at zero (predict's max(0.0, .))
    neg = [ProfileRecord(OpSignature("Sub", HW, (("n", x),)), 3.0 * x - 2.5) for x in (1.0, 2.0, 3.0, 4.0)]
    add("clamp_zero", mk_graph([mk_node("s0", op="Sub", attrs={"n": 0.25}), mk_node("s1", ["s0"], op="Sub", attrs={"n": 5.5})]),
        db_of(neg), StrategyConfig(hardware=HW, op_gap_us=0.2))
    # parameter-server-shaped graph: transfers on link devices, aggregate compute
    links = [DeviceSpec(id=f"link:pcie{i}", kind="Link", throughput_mbps=12347.09 + i, latency_us=0.5 * i) for i in range(3)]
    ps_nodes = []
    for w in range(3):
        ps_nodes.append(mk_node(f"fwd{w}", device=f"gpu{w}", op="Conv2D", attrs={"in_channels": 16 + w}))
        ps_nodes.append(mk_node(f"push{w}", [f"fwd{w}"], device=f"link:pcie{w}", kind=TRANSFER, op="Send",
                                attrs={"src_device": f"gpu{w}", "dst_device": "ps0", "bytes": (w + 1) * 3 * 2 ** 18}))
    ps_nodes.append(mk_node("agg", [f"push{w}" for w in range(3)], device="ps0", op="Conv2D", attrs={"in_channels": 4}))
    for w in range(3):
        ps_nodes.append(mk_node(f"pull{w}", ["agg"], device=f"link:pcie{w}", kind=TRANSFER, op="Recv",
                                attrs={"src_device": "ps0", "dst_device": f"gpu{w}", "bytes": 2 ** 20 + w}))
        ps_nodes.append(mk_node(f"apply{w}", [f"pull{w}"], device=f"gpu{w}", op="Conv2D", attrs={"in_channels": 2}))
    add("ps_transfers", mk_graph(ps_nodes, extra_devices=links),
        db_of(grid_records("Conv2D", "in_channels", 12.5, 40.0, grid)), StrategyConfig(hardware=HW, op_gap_us=0.3))
    return cases


def main():
    for name, fn in (("engine_cases", engine_cases), ("pipeline_cases", pipeline_cases)):
        data = fn()
        path = OUT / f"{name}.json.gz"
        with gzip.open(path, "wt") as fh:
            json.dump(data, fh)
        print(f"{path.name}: {len(data)} cases, {path.stat().st_size} bytes")
    kat = SplitMix64(0)
    print("splitmix64 seed0:", [hex(kat.next_u64()) for _ in range(3)])


if __name__ == "__main__":
    main()
