"""GPU: candidates that differ only in their collective path share one topology class
(batch.group_classes: the path names the devices an expansion adds and sets the PS links'
attributes, but not ids, CSR or device ranks).  Every candidate's schedule, summary and trace
rebuilt from such a class must equal the drop-in path run on that candidate's own expansion
(estimate_all -> simulate -> summarize / to_trace on expand_data_parallel or the PS
expansion), which is itself pinned to the reference's golden outputs."""

from __future__ import annotations

import hashlib
import sys
import warnings
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def bert_sweep():
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2002_06790_b200 as fw

    graphs, db, configs, graph_of = bench.build_workload(0, 36, "bert-large-ps-ar")  # 2 per (R, sync, path)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = fw.sweep_variants(graphs, db, configs, graph_of, keep_schedules=True)
    return graphs, db, configs, graph_of, res


def test_paths_share_classes(bert_sweep):
    from paper_2002_06790_b200.batch import group_classes

    graphs, db, configs, graph_of, res = bert_sweep
    groups = group_classes(graphs, configs, graph_of, db)
    assert len(groups) == 6  # (2, 4, 8 workers) x (allreduce, PS); 3 paths each
    for idx in groups:
        assert len({configs[i].collective.path for i in idx}) == 3


def _own_expansion(g, cfg, db):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200.ps import expand_parameter_server

    if cfg.sync == "parameter_server":
        return expand_parameter_server(g, cfg, db, cfg.ps_device).graph
    return fw.expand_data_parallel(g, cfg).graph


def test_every_path_rebuilds_its_own_schedule(bert_sweep):
    import paper_2002_06790_b200 as fw

    graphs, db, configs, graph_of, res = bert_sweep
    for i in range(0, len(configs), 1):
        cfg = configs[i]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            gx = _own_expansion(graphs[graph_of[i]], cfg, db)
            want = fw.simulate(gx, fw.estimate_all(gx, db, cfg))
        got = res.schedule(i)
        assert [(e.node_id, e.device, e.start_us, e.finish_us, e.source) for e in got.entries] == \
               [(e.node_id, e.device, e.start_us, e.finish_us, e.source) for e in want.entries], i
        assert got.per_device_busy_us == want.per_device_busy_us and list(got.per_device_busy_us) == \
            list(want.per_device_busy_us)
        assert got.makespan_us == want.makespan_us == res.makespan[i]
        if i % 6 == 5:  # reports of one candidate per (R, sync) group and path
            assert res.summary(i) == fw.summarize(want, gx)
            h = lambda t: hashlib.sha256(t.encode()).hexdigest()  # noqa: E731
            assert h(res.trace(i)) == h(fw.to_trace(want))


def test_grouping_grid_rebuilds_every_schedule():
    """The grid of tests/test_group_classes.py (6 graphs incl. three with a link named like a
    device an expansion adds, R in {2, 3}, allreduce / PS, 4 paths) through sweep_variants:
    every candidate's schedule and summary equal the drop-in path on its own expansion, and a
    candidate whose drop-in path raises (no link rows for QPI; a transfer whose link the
    expansion turns into the fabric or the PS device) raises the same error in a sweep."""
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200 import workloads as W

    sys.path.insert(0, str(ROOT / "tests"))
    from test_group_classes import _configs, _graphs

    db = W.planted_profiles(W.CNN_LAWS, links=W.SYNTH_LINKS + W.SYNTH_FABRIC_LINKS)
    graphs = _graphs()
    ok, failing = [], []
    for cfg, gi in _configs():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                g = graphs[gi]
                gx = _own_expansion(g, cfg, db) if cfg.replicas > 1 else g
                ok.append((cfg, gi, fw.simulate(gx, fw.estimate_all(gx, db, cfg))))
            except fw.DfsimError as e:
                failing.append((cfg, gi, e))
    # 24 QPI (allreduce + PS), the NVLink fabric collision (g3, R = 2), g5 under PS (3 paths x 2 R)
    assert len(ok) == 66 and len(failing) == 31, [(c.sync, c.collective.path, c.replicas, gi) for c, gi, _ in failing]
    for cfg, gi, e in failing:
        with warnings.catch_warnings(), pytest.raises(type(e)) as got:
            warnings.simplefilter("ignore")
            fw.sweep_variants(graphs, db, [cfg], [gi])
        assert str(got.value) == str(e)
    configs, graph_of = [c for c, _, _ in ok], [gi for _, gi, _ in ok]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = fw.sweep_variants(graphs, db, configs, graph_of, keep_schedules=True)
    for i, (cfg, gi, want) in enumerate(ok):
        got = res.schedule(i)
        assert [(e.node_id, e.device, e.start_us, e.finish_us, e.source) for e in got.entries] == \
               [(e.node_id, e.device, e.start_us, e.finish_us, e.source) for e in want.entries], i
        assert got.makespan_us == want.makespan_us == res.makespan[i]
        assert got.per_device_busy_us == want.per_device_busy_us
        if gi >= 3:
            gx = _own_expansion(graphs[gi], cfg, db) if cfg.replicas > 1 else graphs[gi]
            assert res.summary(i) == fw.summarize(want, gx)
