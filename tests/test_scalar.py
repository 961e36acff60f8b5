"""The scalar drop-in functions (scalar.py) against golden vectors produced by the real
reference (tests/golden/make_scalar_golden.py): predict, transfer_time, allreduce_time
(device formula kernels, GPU), topological_order (host C++), query_*, apply_overrides."""

from __future__ import annotations

import gzip
import json
import warnings
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden" / "scalar_cases.json.gz"


@pytest.fixture(scope="module")
def cases():
    return json.load(gzip.open(GOLDEN))


def _run(fn):
    try:
        return {"value": fn()}
    except Exception as e:  # noqa: BLE001 -- compared with the reference's exception
        return {"error": type(e).__name__, "message": str(e)}


def test_topological_order_matches_reference(cases):
    import paper_2002_06790_b200 as fw

    for c in cases["topo"]:
        g = fw.parse_graph(json.dumps(c["graph"]))
        assert _run(lambda: fw.topological_order(g)) == c["expect"]


def test_oracle_predict_pinned(cases):
    from oracle import dfsim_oracle as O

    for c in cases["predict"]:
        assert O.predict_neumaier(c["coefs"], c["intercept"], c["features"]) == c["expect"]


def test_queries_and_apply_overrides(cases):
    import paper_2002_06790_b200 as fw

    db = fw.load_profiles(json.dumps(cases["profiles"]))
    assert fw.query_link(db, "nccl-allreduce", "PCIeSwitch", 4).throughput_mbps == 8048.35
    assert fw.query_link(db, "nccl-allreduce", "QPI", 4) is None
    with pytest.raises(ValueError, match="participants must be >= 1"):
        fw.query_link(db, "nccl-allreduce", "QPI", 0)
    assert fw.query_grid(db, "Conv", "hw") == []
    sig = fw.OpSignature("Conv", "hw", (("k", 3.0),))
    assert fw.query_exact(db, sig) is None
    g = fw.make_graph([fw.OpNode("a", "Op", "gpu0"), fw.OpNode("ab", "Op", "gpu0", inputs=(("a", 0),))],
                      [fw.DeviceSpec("gpu0", "Compute")])
    t = fw.DurationTable(entries={"a": fw.DurationEntry(1.0, "ExactRecord"), "ab": fw.DurationEntry(2.0, "FittedModel")})
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = fw.apply_overrides(t, fw.StrategyConfig(overrides={"a*": 5.0, "ab": 7.0, "zz": 1.0}), g)
    assert {k: (e.duration_us, e.source) for k, e in out.entries.items()} == {"a": (5.0, "Override"),
                                                                             "ab": (7.0, "Override")}
    with pytest.raises(fw.MissingDurationError):
        fw.apply_overrides(fw.DurationTable(entries={}), fw.StrategyConfig(), g)


@pytest.mark.gpu
def test_predict_kernel_matches_reference(cases):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import LinearCostModel

    for c in cases["predict"]:
        m = LinearCostModel("Op", "hw", tuple(f"f{i}" for i in range(len(c["coefs"]))), tuple(c["coefs"]),
                            c["intercept"], None)
        assert fw.predict(m, c["features"]) == c["expect"]
    # one launch for many rows of one model
    c = [x for x in cases["predict"] if len(x["coefs"]) == 3]
    m = LinearCostModel("Op", "hw", ("f0", "f1", "f2"), tuple(c[0]["coefs"]), c[0]["intercept"], None)
    rows = [x["features"] for x in c]
    from oracle import dfsim_oracle as O

    want = [O.predict_value(c[0]["coefs"], c[0]["intercept"], r) for r in rows]
    assert fw.predict_batch(m, rows).tolist() == want
    with pytest.raises(ValueError, match="expected 3 features, got 2"):
        fw.predict(m, [1.0, 2.0])


@pytest.mark.gpu
def test_comm_kernels_match_reference(cases):
    import paper_2002_06790_b200 as fw

    db = fw.load_profiles(json.dumps(cases["profiles"]))
    for c in cases["comm"]:
        if c["fn"] == "transfer_time":
            link = fw.DeviceSpec("l", "Link", "", c["thr"], c["lat"])
            got = _run(lambda: fw.transfer_time(c["bytes"], link))
        else:
            fb = fw.DeviceSpec("f", "Link", "", *c["fallback"]) if c["fallback"] else None
            got = _run(lambda: fw.allreduce_time(c["bytes"], c["n"], db, algo=c["algo"], path=c["path"],
                                                 fallback_link=fb))
        assert got == c["expect"], c
    # the acceptance numbers (test_acceptance.py:209-210)
    qpi = fw.query_link(db, "host-to-gpu", "QPI", 1)
    assert abs(fw.transfer_time(2 ** 20, fw.DeviceSpec("l", "Link", "", qpi.throughput_mbps, qpi.latency_us))
               - 83.635) < 1e-3
    assert abs(fw.allreduce_time(100 * 2 ** 20, 4, db, path="PCIeSwitch") - 12424.90) < 1e-2
    assert np.isfinite(fw.comm_time_us(1, 1.0))
