"""GPU parity of the whole per-candidate path (cli.py:83-87) against the reference:
K1 expand_data_parallel -> K2 estimate_all -> K3 simulate -> K4 critical_path,
checked on every golden pipeline case (tests/golden/pipeline_cases.json.gz)."""

from __future__ import annotations

import json
import warnings

import pytest

pytestmark = pytest.mark.gpu


def _run(case):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import load_profiles, parse_config, parse_graph

    g, db, cfg = parse_graph(case["graph"]), load_profiles(case["profiles"]), parse_config(case["config"])
    exp = case["expect"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if cfg.replicas > 1 or cfg.device_map:
            ex = fw.expand_data_parallel(g, cfg)
            ref = parse_graph(exp["expanded"])
            assert list(ex.graph.nodes) == list(ref.nodes), case["name"]
            for nid, n in ref.nodes.items():
                m = ex.graph.nodes[nid]
                assert (m.op_type, m.device, m.kind, m.inputs, dict(m.attrs), m.output_shapes) == \
                       (n.op_type, n.device, n.kind, n.inputs, dict(n.attrs), n.output_shapes), (case["name"], nid)
            assert list(ex.graph.devices) == list(ref.devices)
            assert ex.graph.devices == ref.devices
            assert ex.collective_nodes == exp["collective_nodes"]
            assert {k: list(v) for k, v in ex.replica_of.items()} == exp["replica_of"]
            g = ex.graph
        if exp.get("error") == "UnknownOpError":
            with pytest.raises(fw.UnknownOpError) as err:
                fw.estimate_all(g, db, cfg)
            assert err.value.nodes == exp["nodes"], case["name"]
            return
        table = fw.estimate_all(g, db, cfg)
    assert {k: [e.duration_us, e.source] for k, e in table.entries.items()} == exp["durations"], case["name"]
    assert list(table.entries) == list(exp["durations"])
    s = fw.simulate(g, table)
    assert s.to_json() == json.dumps(exp["schedule"]), case["name"]
    cp = fw.critical_path(g, {e.node_id: e.finish_us - e.start_us for e in s.entries})
    assert [cp[0], cp[1]] == exp["cp"], case["name"]


def test_pipeline_golden_cases(pipeline_cases):
    for case in pipeline_cases:
        _run(case)


def test_sweep_matches_reference_pipeline(pipeline_cases):
    """The batched sweep over many configs reproduces each single-candidate result."""
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import load_profiles, parse_config, parse_graph

    by_graph = {}
    for case in pipeline_cases:
        if case["expect"].get("error"):
            continue
        by_graph.setdefault((case["graph"], case["profiles"]), []).append(case)
    for (gtxt, dbtxt), cases in by_graph.items():
        g, db = parse_graph(gtxt), load_profiles(dbtxt)
        cfgs = [parse_config(c["config"]) for c in cases]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = fw.sweep(g, db, cfgs, keep_schedules=True)
        for i, c in enumerate(cases):
            e = c["expect"]
            assert res.makespan[i] == e["schedule"]["makespan_us"], c["name"]
            assert res.cp_len[i] == e["cp"][0], c["name"]
            assert res.schedule(i).to_json() == json.dumps(e["schedule"]), c["name"]
            assert res.critical_path(i) == (e["cp"][0], e["cp"][1]), c["name"]
        ms = [c["expect"]["schedule"]["makespan_us"] for c in cases]
        assert res.best_index == min(range(len(ms)), key=ms.__getitem__)


def test_estimate_errors():
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, ProfileDB, StrategyConfig, make_graph

    link = DeviceSpec("l0", "Link", "", 100.0, 0.0)
    g = make_graph([OpNode("t", "Send", "l0", "Transfer", {"src_device": "a", "dst_device": "b", "bytes": 0}),
                    OpNode("u", "Mystery", "gpu0")], [link, DeviceSpec("gpu0", "Compute")])
    with pytest.raises(ValueError, match="bytes must be > 0"):
        fw.estimate_all(g, ProfileDB(), StrategyConfig())
    g2 = make_graph([OpNode("u", "Mystery", "gpu0")], [DeviceSpec("gpu0", "Compute")])
    with pytest.raises(ValueError, match="nonnegative"):
        fw.estimate_all(g2, ProfileDB(), StrategyConfig(overrides={"u": -1.0}))


def test_sweep_concurrent_streams_match_serial():
    """Many small topology classes launched on 8 streams == one after another on one stream
    (per-stream scratch in the context), and AR candidates match the oracle."""
    import numpy as np

    import paper_2002_06790_b200 as fw
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    graphs = [W.vgg16_training(batch=b) for b in (8, 32)]
    db = W.model_profiles(graphs[0], ["hw0"])
    cfgs, gof = [], []
    for gi in range(2):
        for R in (1, 2, 4):
            for sync in ("allreduce", "parameter_server"):
                for path in ("NVLink", "PCIeSwitch"):
                    for gap in (0.0, 0.5):
                        cfgs.append(StrategyConfig(replicas=R, device_map=tuple(f"gpu{k}" for k in range(R)),
                                                   collective=CollectiveConfig("MeasuredThroughput", path),
                                                   gradient_markers=("wgrad_*",), hardware="hw0", op_gap_us=gap,
                                                   sync=sync if R > 1 else "allreduce"))
                        gof.append(gi)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = fw.sweep_variants(graphs, db, cfgs, gof, streams=1)
        b = fw.sweep_variants(graphs, db, cfgs, gof, streams=8)
    assert len(b.classes) == 5  # R = 1 | (2, 4 workers) x (allreduce, PS); both paths share each class
    assert np.array_equal(a.makespan, b.makespan) and np.array_equal(a.cp_len, b.cp_len)
    assert (a.best_index, a.best_makespan) == (b.best_index, b.best_makespan)
    for i in (0, 5, 17, 40):
        if cfgs[i].sync == "allreduce":
            ms, cp, *_ = O.run_candidate(graphs[gof[i]], db, cfgs[i])
            assert (b.makespan[i], b.cp_len[i]) == (ms, cp), i


def test_sweep_edge_cases():
    """Empty graph, a single node, no configs: the reference's answers (cli.py:123-149)."""
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, ProfileDB, StrategyConfig, make_graph

    empty = make_graph([], [])
    res = fw.sweep(empty, ProfileDB(), [StrategyConfig(), StrategyConfig(op_gap_us=1.0)], keep_schedules=True)
    assert list(res.makespan) == [0.0, 0.0] and list(res.cp_len) == [0.0, 0.0] and res.best_index == 0
    s = res.schedule(0)
    assert s.entries == [] and s.makespan_us == 0.0
    assert fw.to_trace(s) == "[]\n"
    one = make_graph([OpNode("a", "Op", "gpu0")], [DeviceSpec("gpu0", "Compute")])
    cfgs = [StrategyConfig(overrides={"a": 2.5}), StrategyConfig(overrides={"a": 1.5})]
    res = fw.sweep(one, ProfileDB(), cfgs, keep_schedules=True)
    assert list(res.makespan) == [2.5, 1.5] and res.best_index == 1
    rep = res.summary(1)
    assert rep.critical_path_nodes == ["a"] and rep.critical_path_us == 1.5 and rep.top_k_ops == [("Op", 1.5, 1.0)]
    none = fw.sweep(one, ProfileDB(), [])
    assert none.best_index == -1 and len(none.makespan) == 0


def test_sweep_rejects_nan_or_negative_values_like_the_reference():
    """A NaN op_gap_us or a negative override passes the config parser (NaN < 0 is False) but
    not DurationEntry (costmodel.py:78-80): sweep must raise that ValueError instead of
    running the fused engine on a NaN/negative duration (which never terminates)."""
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200 import workloads as W

    g = W.layered_cnn(6)
    db = W.planted_profiles(W.CNN_LAWS)
    base = dict(replicas=4, device_map=("gpu0", "gpu1", "gpu2", "gpu3"), gradient_markers=("grad_conv_*",),
                hardware="synth-hw")
    good = fw.StrategyConfig(**base, op_gap_us=0.5)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert fw.TopologyClass(g, db, [good]).fused
        for bad in (fw.StrategyConfig(**base, op_gap_us=float("nan")),
                    fw.StrategyConfig(**base, op_gap_us=-1e9),
                    fw.StrategyConfig(**base, overrides={"conv_01@r2": -2.0}),
                    fw.StrategyConfig(**base, overrides={"conv_*": float("nan")})):
            assert not fw.TopologyClass(g, db, [good, bad]).fused
            with pytest.raises(ValueError, match="nonnegative"):
                fw.sweep(g, db, [good, bad])


def test_sweep_error_precedence_construction_vs_runtime():
    """The first failing config in list order raises (cli.py:132-145), whether its class failed
    to build (expansion ConfigError) or at run time (UnknownOpError)."""
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, ProfileDB, make_graph

    g = make_graph([OpNode("a", "Mystery", "gpu0"),
                    OpNode("t", "Send", "l0", "Transfer", {"src_device": "gpu0", "dst_device": "gpu1", "bytes": 8},
                           inputs=(("a", 0),))],
                   [DeviceSpec("gpu0", "Compute"), DeviceSpec("gpu1", "Compute"), DeviceSpec("l0", "Link", "", 100.0, 0.0)])
    plain = fw.StrategyConfig()
    bad_dp = fw.StrategyConfig(replicas=2, device_map=("gpu0", "gpu1"), gradient_markers=("t",))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with pytest.raises(fw.UnknownOpError):
            fw.sweep(g, ProfileDB(), [plain, bad_dp])
        with pytest.raises(fw.ConfigError):
            fw.sweep(g, ProfileDB(), [bad_dp, plain])
