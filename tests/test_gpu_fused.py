"""GPU: the fused hot path (K2a + K3 v2 + K4 v2) equals the unfused kernels and the oracle.

The unfused path is itself pinned to the reference's golden outputs
(test_gpu_engine.py, test_gpu_pipeline.py); here the fused engine must reproduce
it bit-for-bit on the headline ResNet-50 DP8 class, including candidates with
overrides, and including the exact-engine fallback after a FIFO ring overflow.
"""

from __future__ import annotations

import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _configs(n, overrides_every=5):
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    dmap = tuple(f"gpu{i}" for i in range(8))
    out = []
    for i in range(n):
        ov = {"wgrad_l1_*": 3.25, "l2_b0_conv1@r3": 0.0} if i % overrides_every == min(3, overrides_every - 1) else {}
        algo = "RingAnalytic" if i % 3 else "MeasuredThroughput"
        out.append(StrategyConfig(replicas=8, device_map=dmap, collective=CollectiveConfig(algo, "NVLink"),
                                  gradient_markers=("wgrad_*",), hardware=f"hw{i % 4}", op_gap_us=1e-3 * (i // 4),
                                  overrides=ov))
    return out


@pytest.fixture(scope="module")
def resnet():
    from paper_2002_06790_b200 import workloads as W

    g = W.resnet50_training(batch=32)
    return g, W.model_profiles(g, [f"hw{i}" for i in range(4)])


def _rank_rows(tc, o):
    return [tuple(t.cpu().numpy() for t in tc.rows_by_rank(o, r)) for r in range(tc.lp.n_sims)]


def _compare(tc_f, tc_u):
    of, ou = tc_f.run(), tc_u.run()
    assert tc_f.fused and not tc_u.fused
    assert np.array_equal(of["makespan"].cpu().numpy(), ou["makespan"].cpu().numpy())
    assert np.array_equal(of["busy"].cpu().numpy(), ou["busy"].cpu().numpy())
    assert np.array_equal(of["cp_len"].cpu().numpy(), ou["cp_len"].cpu().numpy())
    assert (of["n_placed"].cpu().numpy() == tc_f.lg.n).all()
    for (sf, ff), (su, fu) in zip(_rank_rows(tc_f, of), _rank_rows(tc_u, ou)):
        assert np.array_equal(sf, su) and np.array_equal(ff, fu)
    return of


def test_fused_equals_unfused_resnet_dp8(resnet):
    from paper_2002_06790_b200.batch import TopologyClass

    g, db = resnet
    cfgs = _configs(96)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tf = TopologyClass(g, db, cfgs, fused=True)
        tu = TopologyClass(g, db, cfgs, fused=False)
    of = _compare(tf, tu)
    assert not of.get("fallback_rows")
    src = of["cp_src"].cpu().numpy()
    assert (src >= 0).all()


@pytest.mark.parametrize("search_all", [False, True])
def test_fused_override_rows_equal_unfused(resnet, monkeypatch, search_all):
    """Overrides in the fused engine, both ways: few (variant, override set) combinations get
    their own duration rows (dfsim_override_rows: no lookup in the engine), otherwise the
    engine searches the set per popped node (skipping nodes in no set).  Both must equal the
    unfused kernels bit for bit (costmodel.py:302-304: an override replaces the estimate)."""
    from paper_2002_06790_b200.batch import TopologyClass

    if search_all:
        monkeypatch.setenv("DFSIM_OV_SEARCH_ALL", "1")
    g, db = resnet
    cfgs = _configs(256, overrides_every=2)  # 4 hw x 2 algos x {none, one set}: 16 combinations
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tf = TopologyClass(g, db, cfgs, fused=True)
        tu = TopologyClass(g, db, cfgs, fused=False)
    assert (tf.combo is None) == search_all
    _compare(tf, tu)


def test_reexpand_async_reproduces_first_expansion(resnet):
    """K1 re-run without host round-trips (n_refs given, no count read-back) rewrites
    the same CSR; the synchronising variant (n_refs = -1, counts read back) agrees."""
    import torch

    from paper_2002_06790_b200.batch import TopologyClass

    g, db = resnet
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tu = TopologyClass(g, db, _configs(8), fused=False)
    lg, plan = tu.lg, tu.plan
    names = ("t_succ_off", "t_succ_idx", "t_indeg", "t_dev", "t_sources", "t_queue_off")
    used = dict(t_succ_idx=lg.n_edges, t_sources=lg.n_sources)

    def view(k):
        t = getattr(lg, k)
        return t[: used[k]] if k in used else t

    before = {k: view(k).clone() for k in names}
    for k in names:
        getattr(lg, k).fill_(-7)
    plan.reexpand(topo=True)
    torch.cuda.synchronize()
    for k in names:
        assert torch.equal(view(k), before[k]), k
    _assert_topological(lg)
    plan._structs[0].n_refs = -1
    plan.reexpand(topo=True, check=True)
    for k in names:
        assert torch.equal(view(k), before[k]), k
    _assert_topological(lg)


def _assert_topological(lg):
    """The Kahn order may differ run to run (frontier order); it must be a topological order."""
    topo = lg.t_topo[: lg.n].cpu().numpy()
    off, idx = lg.t_succ_off.cpu().numpy(), lg.t_succ_idx[: lg.n_edges].cpu().numpy()
    pos = np.full(lg.n, -1)
    pos[topo] = np.arange(lg.n)
    assert (pos >= 0).all()
    src = np.repeat(np.arange(lg.n), np.diff(off[: lg.n + 1]))
    assert (pos[src] < pos[idx]).all()


def test_fused_ring_overflow_falls_back_exactly(resnet, monkeypatch):
    from paper_2002_06790_b200.batch import TopologyClass
    from paper_2002_06790_b200.prepare import ClassTables

    g, db = resnet
    cfgs = _configs(40)
    monkeypatch.setattr(ClassTables, "QCAP", 2)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tf = TopologyClass(g, db, cfgs, fused=True)
        tu = TopologyClass(g, db, cfgs, fused=False)
    of = _compare(tf, tu)
    assert of.get("fallback_rows"), "QCAP=2 must overflow on this graph"


@pytest.mark.parametrize("n", [1, 2, 4, 97])
def test_fused_overflow_in_partial_warps(resnet, monkeypatch, n):
    """Chunks whose warps hold flagged and idle candidate groups side by side (three groups
    per warp): every lane must reach the warp-wide votes (regression: a short-circuited vote
    deadlocked such warps)."""
    from paper_2002_06790_b200.batch import TopologyClass
    from paper_2002_06790_b200.prepare import ClassTables

    g, db = resnet
    cfgs = _configs(n)
    monkeypatch.setattr(ClassTables, "QCAP", 2)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tf = TopologyClass(g, db, cfgs, fused=True)
        tu = TopologyClass(g, db, cfgs, fused=False)
    _compare(tf, tu)


def test_fused_spot_check_against_oracle(resnet):
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import sweep

    g, db = resnet
    cfgs = _configs(12)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = sweep(g, db, cfgs, keep_schedules=True)
        for i in (0, 3, 7, 11):
            ms, cp_len, entries, busy, cp_path = O.run_candidate(g, db, cfgs[i])
            assert res.makespan[i] == ms and res.cp_len[i] == cp_len
            s = res.schedule(i)
            assert [(e.node_id, e.device, e.start_us, e.finish_us) for e in s.entries] == entries
            assert res.critical_path(i) == (cp_len, cp_path)
    ms_all = res.makespan
    assert res.best_index == int(np.argmin(ms_all))


def test_sweep_unfused_matches_fused_on_layered(pipeline_cases):
    import json

    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.model import load_profiles, parse_config, parse_graph

    cases = [c for c in pipeline_cases if c["name"].startswith(("layered_ring", "random30", "c7_r"))]
    for c in cases:
        g, db, cfg = parse_graph(c["graph"]), load_profiles(c["profiles"]), parse_config(c["config"])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = fw.sweep(g, db, [cfg] * 3, keep_schedules=True)
        assert r.schedule(2).to_json() == json.dumps(c["expect"]["schedule"]), c["name"]
        assert r.cp_len[1] == c["expect"]["cp"][0]


def test_fused_row_layout_with_level_kernel(resnet, monkeypatch):
    """A class without a K4 v3 plan keeps row-layout schedules and K4 v2 (level groups):
    forced here; results must still equal the unfused kernels, overflow fallback included."""
    from paper_2002_06790_b200.batch import TopologyClass
    from paper_2002_06790_b200.prepare import ClassTables

    g, db = resnet
    monkeypatch.setenv("DFSIM_CP_KERNEL", "levels")
    for qcap in (16, 2):
        monkeypatch.setattr(ClassTables, "QCAP", qcap)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            tf = TopologyClass(g, db, _configs(40), fused=True)
            tu = TopologyClass(g, db, _configs(40), fused=False)
        assert tf.tables.lane is None and tf.tables.cp_struct is not None
        _compare(tf, tu)


def test_lane_kernel_partial_warps(resnet, monkeypatch):
    """Candidate counts that leave the last 32-candidate warp of K4 v3 partly empty, and one
    candidate alone, must agree with the unfused kernels (K4 v3 forced below its class-size
    threshold)."""
    from paper_2002_06790_b200 import prepare
    from paper_2002_06790_b200.batch import TopologyClass

    monkeypatch.setattr(prepare, "LANE_MIN_SIMS", 1)
    g, db = resnet
    for n in (1, 33, 70):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            tf = TopologyClass(g, db, _configs(n), fused=True)
            tu = TopologyClass(g, db, _configs(n), fused=False)
        assert tf.tables.lane is not None
        _compare(tf, tu)


def test_lane_kernel_with_overflow_reruns(resnet, monkeypatch):
    """K4 v3 (forced) after ring-overflow re-runs: the critical paths of just the re-run
    candidates are redone through the candidate-list entry (dfsim_critical_path_lanes_ex)."""
    from paper_2002_06790_b200 import prepare
    from paper_2002_06790_b200.batch import TopologyClass
    from paper_2002_06790_b200.prepare import ClassTables

    monkeypatch.setattr(prepare, "LANE_MIN_SIMS", 1)
    monkeypatch.setattr(ClassTables, "QCAP", 2)
    g, db = resnet
    cfgs = _configs(45)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tf = TopologyClass(g, db, cfgs, fused=True)
        tu = TopologyClass(g, db, cfgs, fused=False)
    assert tf.tables.lane is not None
    o = tf.run(defer_fallback=True)
    assert tf.fallback_if_needed(o) and o["fallback_rows"]
    tf.critical_path_only(o)
    ou = tu.run()
    assert np.array_equal(o["makespan"].cpu().numpy(), ou["makespan"].cpu().numpy())
    assert np.array_equal(o["cp_len"].cpu().numpy(), ou["cp_len"].cpu().numpy())
