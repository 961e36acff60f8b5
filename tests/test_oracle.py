"""Pin the oracle (oracle/) against the reference's own outputs (tests/golden/).

CPU only: the Python restatement and the C engine restatement must reproduce
every golden fixture bit-for-bit before either is trusted as a parity checker.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import case_graph, case_table
from oracle import dfsim_oracle as O
from oracle import native_oracle as NO
from paper_2002_06790_b200.model import parse_config, load_profiles, parse_graph


def _expected_entries(exp):
    return [tuple(e[:4]) for e in exp["schedule"]["entries"]]


def test_python_engine_matches_golden(engine_cases):
    for case in engine_cases:
        g, exp = case_graph(case), case["expect"]
        durs = {k: v for k, (v, _) in case["durations"].items()}
        if exp.get("error") == "MissingDurationError":
            assert set(g.nodes) - set(durs) == set(exp["ids"])
            continue
        if exp.get("error") == "CycleError":
            with pytest.raises(O.OracleCycle) as err:
                O.simulate(g, durs)
            assert err.value.ids == exp["ids"], case["name"]
            continue
        entries, makespan, busy = O.simulate(g, durs)
        assert entries == _expected_entries(exp), case["name"]
        assert makespan == exp["schedule"]["makespan_us"]
        assert busy == exp["schedule"]["per_device_busy_us"]
        cp = O.critical_path(g, {nid: f - s for nid, _, s, f in entries})
        assert [cp[0], cp[1]] == exp["cp"], case["name"]


def test_c_engine_matches_golden(engine_cases):
    for case in engine_cases:
        exp = case["expect"]
        if exp.get("error") == "MissingDurationError":
            continue
        g = case_graph(case)
        csr = NO.Csr(g)
        dur = np.array([case["durations"][nid][0] for nid in csr.ids])
        rc, start, finish, busy, ms, order = NO.simulate(csr, dur)
        if exp.get("error") == "CycleError":
            assert rc == 1
            assert [csr.ids[v] for v in np.nonzero(np.isnan(start))[0]] == exp["ids"]
            continue
        assert rc == 0, case["name"]
        got = [(csr.ids[v], csr.devices[csr.dev[v]], start[v], finish[v]) for v in order]
        assert got == _expected_entries(exp), case["name"]
        assert ms == exp["schedule"]["makespan_us"]
        exp_busy = exp["schedule"]["per_device_busy_us"]
        assert {d: busy[i] for i, d in enumerate(csr.devices) if d in exp_busy} == exp_busy
        rc, length, path = NO.critical_path(csr, finish - start)
        assert rc == 0
        assert [length, [csr.ids[v] for v in path]] == exp["cp"], case["name"]


def test_python_pipeline_matches_golden(pipeline_cases):
    for case in pipeline_cases:
        g, db, cfg = parse_graph(case["graph"]), load_profiles(case["profiles"]), parse_config(case["config"])
        exp = case["expect"]
        if exp.get("error") == "UnknownOpError":
            gg = O.expand(g, cfg)[0] if (cfg.replicas > 1 or cfg.device_map) else g
            with pytest.raises(O.OracleUnknownOp) as err:
                O.estimate(gg, db, cfg)
            assert err.value.nodes == exp["nodes"], case["name"]
            continue
        assert "error" not in exp, case["name"]
        if "expanded" in exp:
            gx, replica_of, coll = O.expand(g, cfg)
            ref = parse_graph(exp["expanded"])
            assert list(gx.nodes) == list(ref.nodes), case["name"]
            for nid, n in ref.nodes.items():
                m = gx.nodes[nid]
                assert (m.op_type, m.device, m.kind, m.inputs, dict(m.attrs)) == \
                       (n.op_type, n.device, n.kind, n.inputs, dict(n.attrs)), (case["name"], nid)
            assert sorted(gx.devices) == sorted(ref.devices)
            assert coll == exp["collective_nodes"]
            g = gx
        table = O.estimate(g, db, cfg)
        assert {k: [v, s] for k, (v, s) in table.items()} == exp["durations"], case["name"]
        entries, makespan, busy = O.simulate(g, {k: v for k, (v, _) in table.items()})
        assert entries == _expected_entries(exp), case["name"]
        assert makespan == exp["schedule"]["makespan_us"]
        cp = O.critical_path(g, {nid: f - s for nid, _, s, f in entries})
        assert [cp[0], cp[1]] == exp["cp"], case["name"]


def _summary_and_trace(g, durs, sources):
    entries, makespan, busy = O.simulate(g, durs)
    cp = O.critical_path(g, {nid: f - s for nid, _, s, f in entries})
    op = {nid: n.op_type for nid, n in g.nodes.items()}
    kinds = {d: spec.kind for d, spec in g.devices.items()}
    return (O.summarize(entries, op, kinds, busy, makespan, cp), O.to_trace(entries, op, sources, busy))


def _check_report(case, g, durs, sources):
    import hashlib
    import json

    exp = case["expect"]
    rep, trace = _summary_and_trace(g, durs, sources)
    # dict order matters (the reference's report iterates these dicts)
    assert json.dumps(rep) == json.dumps(exp["summary"]), case["name"]
    if "trace" in exp:
        assert trace == exp["trace"], case["name"]
    assert hashlib.sha256(trace.encode()).hexdigest() == exp["trace_sha256"], case["name"]


def test_python_summary_and_trace_match_golden(engine_cases, pipeline_cases):
    """summarize (reporting.py:117-162) and to_trace (43-74) restated, pinned on every fixture."""
    n = 0
    for case in engine_cases:
        if "summary" not in case["expect"]:
            continue
        d = case["durations"]
        _check_report(case, case_graph(case), {k: v for k, (v, _) in d.items()}, {k: s for k, (_, s) in d.items()})
        n += 1
    for case in pipeline_cases:
        exp = case["expect"]
        if "summary" not in exp:
            continue
        g = parse_graph(exp["expanded"]) if "expanded" in exp else parse_graph(case["graph"])
        d = exp["durations"]
        _check_report(case, g, {k: v for k, (v, _) in d.items()}, {k: s for k, (_, s) in d.items()})
        n += 1
    assert n > 150


def test_python_predict_is_cpython_sum():
    """predict's sum is CPython's float sum (Neumaier since 3.12); pinned here on random data."""
    rng = np.random.default_rng(7)
    for _ in range(2000):
        k = int(rng.integers(1, 6))
        coefs = [float(x) for x in rng.normal(size=k) * 10.0 ** rng.integers(-8, 8, size=k)]
        feats = [float(x) for x in rng.normal(size=k) * 10.0 ** rng.integers(-3, 9, size=k)]
        icpt = float(rng.normal() * 100)
        want = max(0.0, icpt + sum(c * f for c, f in zip(coefs, feats)))
        assert O.predict_value(coefs, icpt, feats) == want
        # the explicit compensated loop the CUDA kernel implements
        assert O.predict_neumaier(coefs, icpt, feats) == want
