"""GPU parity of the schedule consumers: summarize (reporting.py:117-162)
through K6 + K4, and to_trace (43-74), against the reference's own reports in
tests/golden/ and against the oracle on the headline ResNet-50 DP8 class."""

from __future__ import annotations

import hashlib
import json
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _doc(r):
    return {"makespan_us": r.makespan_us, "per_device_busy_us": r.per_device_busy_us, "utilization": r.utilization,
            "device_kinds": r.device_kinds, "top_k_ops": [list(t) for t in r.top_k_ops], "compute_us": r.compute_us,
            "comm_us": r.comm_us, "overlap_us": r.overlap_us, "critical_path_nodes": r.critical_path_nodes,
            "critical_path_us": r.critical_path_us}


def _schedule(doc, g):
    """The Schedule object the reference held: Schedule.to_json sorts the busy dict, the
    in-memory one lists g.devices first, then other devices in entry order (engine.py:88-92)."""
    from paper_2002_06790_b200.model import Schedule, ScheduledNode

    entries = [ScheduledNode(*e) for e in doc["entries"]]
    busy = {d: doc["per_device_busy_us"][d] for d in g.devices if d in doc["per_device_busy_us"]}
    for e in entries:
        busy.setdefault(e.device, doc["per_device_busy_us"][e.device])
    assert busy.keys() == doc["per_device_busy_us"].keys()
    return Schedule(entries=entries, makespan_us=doc["makespan_us"], per_device_busy_us=busy)


def test_summarize_dropin_matches_golden(engine_cases, pipeline_cases):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import parse_graph

    n = 0
    for case in list(engine_cases) + list(pipeline_cases):
        exp = case["expect"]
        if "summary" not in exp:
            continue
        g = parse_graph(exp["expanded"]) if "expanded" in exp else parse_graph(case["graph"])
        rep = fw.summarize(_schedule(exp["schedule"], g), g)
        assert json.dumps(_doc(rep)) == json.dumps(exp["summary"]), case["name"]
        n += 1
    assert n > 200


def test_summarize_rejects_foreign_schedule(engine_cases):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import parse_graph

    case = next(c for c in engine_cases if c["name"] == "chain")
    g = parse_graph(case["graph"])
    s = _schedule(case["expect"]["schedule"], g)
    s.entries = s.entries[:-1]
    with pytest.raises(fw.DfsimError, match="node sets differ"):
        fw.summarize(s, g)


def test_sweep_summaries_and_traces_match_golden(pipeline_cases):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import load_profiles, parse_config, parse_graph

    by_graph = {}
    for case in pipeline_cases:
        if "summary" in case["expect"]:
            by_graph.setdefault((case["graph"], case["profiles"]), []).append(case)
    for (gtxt, dbtxt), cases in by_graph.items():
        g, db = parse_graph(gtxt), load_profiles(dbtxt)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = fw.sweep(g, db, [parse_config(c["config"]) for c in cases], keep_schedules=True)
        reps = res.summaries(range(len(cases)))
        for i, c in enumerate(cases):
            assert json.dumps(_doc(reps[i])) == json.dumps(c["expect"]["summary"]), c["name"]
            assert hashlib.sha256(res.trace(i).encode()).hexdigest() == c["expect"]["trace_sha256"], c["name"]


def test_sweep_summaries_resnet_dp8_vs_oracle():
    """Fused sweep on the headline class: batched K6 reports == the oracle's summarize/to_trace."""
    import paper_2002_06790_b200 as fw
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    g = W.resnet50_training(batch=32)
    db = W.model_profiles(g, ["hw0", "hw1"])
    dmap = tuple(f"gpu{i}" for i in range(8))
    cfgs = [StrategyConfig(replicas=8, device_map=dmap, collective=CollectiveConfig("RingAnalytic", "NVLink"),
                           gradient_markers=("wgrad_*",), hardware=f"hw{i % 2}", op_gap_us=0.25 * i,
                           overrides={"wgrad_l1_*": 3.25} if i == 3 else {}) for i in range(6)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = fw.sweep(g, db, cfgs, keep_schedules=True)
        reps = res.summaries(range(len(cfgs)), top_k=12)
        for i, cfg in enumerate(cfgs):
            gx = O.expand(g, cfg)[0]
            table = O.estimate(gx, db, cfg)
            entries, makespan, busy = O.simulate(gx, {k: v for k, (v, _) in table.items()})
            cp = O.critical_path(gx, {nid: f - s for nid, _, s, f in entries})
            op = {nid: n.op_type for nid, n in gx.nodes.items()}
            kinds = {d: spec.kind for d, spec in gx.devices.items()}
            want = O.summarize(entries, op, kinds, busy, makespan, cp, top_k=12)
            assert json.dumps(_doc(reps[i])) == json.dumps(want), i
            assert res.trace(i) == O.to_trace(entries, op, {k: s for k, (_, s) in table.items()}, busy), i


@pytest.mark.parametrize("seed", range(10))
def test_summarize_random_schedules_vs_oracle(seed):
    """K6 on random schedules: link / collective devices, empty op types, zero durations, ties."""
    import paper_2002_06790_b200 as fw
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200.model import (DeviceSpec, DurationEntry, DurationTable, OpNode, make_graph)

    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    devs = [DeviceSpec(f"gpu{k}", "Compute") for k in range(int(rng.integers(1, 6)))]
    devs += [DeviceSpec(f"link{k}", "Link", "", 100.0, 0.5) for k in range(int(rng.integers(0, 3)))]
    devs += [DeviceSpec("fabric", "CollectiveResource", "", 1.0, 0.0)] if rng.random() < 0.5 else []
    nodes, durs = [], {}
    for i in range(n):
        d = devs[int(rng.integers(0, len(devs)))]
        kind = {"Compute": "Compute", "Link": "Transfer", "CollectiveResource": "Collective"}[d.kind]
        ins = tuple((f"v{j:04d}", 0) for j in sorted(set(rng.integers(0, i, size=int(rng.integers(0, 3))).tolist()))) if i else ()
        nodes.append(OpNode(f"v{i:04d}", str(rng.choice(["MatMul", "Add", "", "Send"])), d.id, kind, {}, ins))
        durs[f"v{i:04d}"] = float(rng.choice([0.0, 1.0, 2.5, rng.uniform(0, 10)]))
    g = make_graph(nodes, devs)
    table = DurationTable(entries={k: DurationEntry(v, "Override") for k, v in durs.items()})
    s = fw.simulate(g, table)
    rep = fw.summarize(s, g, top_k=int(rng.integers(0, 6)))
    entries, ms, busy = O.simulate(g, durs)
    cp = O.critical_path(g, {nid: f - st for nid, _, st, f in entries})
    want = O.summarize(entries, {k: v.op_type for k, v in g.nodes.items()}, {d: sp.kind for d, sp in g.devices.items()},
                       s.per_device_busy_us, ms, cp, top_k=len(rep.top_k_ops) if rep.top_k_ops else 0)
    got = _doc(rep)
    for k in ("compute_us", "comm_us", "overlap_us", "critical_path_us", "critical_path_nodes", "makespan_us"):
        assert got[k] == want[k], (seed, k)
    assert got["top_k_ops"] == want["top_k_ops"][: len(got["top_k_ops"])]
