"""Parameter-server expansion (new code, ps.py): structure on CPU; estimate + simulate of the
emitted graph against the oracle on the GPU (the expansion itself has no reference)."""

from __future__ import annotations

import warnings

import numpy as np
import pytest


def _setup(R=4, path="NVLink"):
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    g = W.vgg16_training(batch=16)
    db = W.model_profiles(g, ["hw0", "hw1"])
    cfg = StrategyConfig(replicas=R, device_map=tuple(f"gpu{i}" for i in range(R)),
                         collective=CollectiveConfig("RingAnalytic", path), gradient_markers=("wgrad_*",),
                         hardware="hw0", op_gap_us=0.25, sync="parameter_server")
    return g, db, cfg


def test_ps_expansion_structure():
    from paper_2002_06790_b200.ps import expand_parameter_server

    g, db, cfg = _setup()
    ex = expand_parameter_server(g, cfg, db)
    gx = ex.graph
    G = sum(1 for n in g.nodes if n.startswith("wgrad_"))
    assert len(gx.nodes) == cfg.replicas * len(g.nodes) + G * (2 * cfg.replicas + 1)
    assert len(ex.collective_nodes) == 2 * cfg.replicas * G
    for nid, node in gx.nodes.items():
        for pid, _ in node.inputs:
            assert pid in gx.nodes, (nid, pid)
            assert not (pid.startswith("wgrad_") and not nid.startswith("push_")), "consumer not rewired"
    agg = gx.nodes["aggregate_wgrad_fc3"]
    assert agg.device == "ps0" and len(agg.inputs) == cfg.replicas
    assert gx.devices["link:NVLink:gpu1->ps0"].kind == "Link"
    assert gx.nodes["apply_fc3@r2"].inputs == (("pull_wgrad_fc3@r2", 0),)


@pytest.mark.gpu
def test_ps_sweep_matches_oracle():
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import sweep
    from paper_2002_06790_b200.ps import expand_parameter_server

    g, db, cfg = _setup()
    cfgs = [cfg, cfg.__class__(**{**cfg.__dict__, "hardware": "hw1", "op_gap_us": 0.0}),
            cfg.__class__(**{**cfg.__dict__, "op_gap_us": 1.5})]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = sweep(g, db, cfgs, keep_schedules=True)
        for i, c in enumerate(cfgs):
            gx = expand_parameter_server(g, c, db).graph
            table = O.estimate(gx, db, c)
            entries, ms, busy = O.simulate(gx, {k: v[0] for k, v in table.items()})
            cp = O.critical_path(gx, {nid: f - s for nid, _, s, f in entries})
            assert res.makespan[i] == ms and res.cp_len[i] == cp[0]
            s = res.schedule(i)
            assert [(e.node_id, e.device, e.start_us, e.finish_us) for e in s.entries] == entries
    assert res.best_index == int(np.argmin(res.makespan))


@pytest.mark.gpu
def test_ps_r8_wide_device_set_fused_equals_unfused():
    """8 workers + 16 links + PS = 25 devices: exercises the 32-lane engine group."""
    from paper_2002_06790_b200.batch import TopologyClass

    g, db, cfg = _setup(R=8)
    cfgs = [cfg.__class__(**{**cfg.__dict__, "hardware": f"hw{i % 2}", "op_gap_us": 0.01 * i}) for i in range(40)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tf = TopologyClass(g, db, cfgs, fused=True)
        tu = TopologyClass(g, db, cfgs, fused=False)
    assert tf.fused and tf.lg.n_devices == 25
    of, ou = tf.run(), tu.run()
    assert np.array_equal(of["makespan"].cpu().numpy(), ou["makespan"].cpu().numpy())
    assert np.array_equal(of["cp_len"].cpu().numpy(), ou["cp_len"].cpu().numpy())
    assert np.array_equal(of["busy"].cpu().numpy(), ou["busy"].cpu().numpy())
    for r in range(len(cfgs)):
        for a, b in zip(tf.rows_by_rank(of, r), tu.rows_by_rank(ou, r)):
            assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())
