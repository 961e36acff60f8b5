"""GPU: sweeps over graphs loaded by the C++ document loader equal sweeps over
parse_graph's objects (plain classes take the loader's CSR / signature tables directly;
expanded classes materialise nodes on demand)."""

from __future__ import annotations

import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _configs(dp: bool):
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    if dp:
        return [StrategyConfig(replicas=4, device_map=tuple(f"gpu{i}" for i in range(4)),
                               collective=CollectiveConfig("RingAnalytic", "NVLink"), gradient_markers=("wgrad_*",),
                               hardware=f"hw{i % 2}", op_gap_us=0.1 * i) for i in range(6)]
    return [StrategyConfig(hardware=f"hw{i % 2}", op_gap_us=0.1 * i,
                           overrides={"n0001*": 2.5} if i == 3 else {}) for i in range(6)]


@pytest.mark.parametrize("name", ["layered", "resnet"])
def test_sweep_on_loaded_document_equals_parsed(name):
    import paper_2002_06790_b200 as fw
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import parse_graph, serialize_graph

    if name == "layered":
        g0 = W.layered_dag(20_000, 200, devices=8)
        db = W.dag_profiles(["hw0", "hw1"])
        cfgs = _configs(False)
    else:
        g0 = W.resnet50_training(batch=8)
        db = W.model_profiles(g0, ["hw0", "hw1"])
        cfgs = _configs(True)
    text = serialize_graph(g0)
    gd, gp = fw.load_graph(text), parse_graph(text)
    assert isinstance(gd, fw.DocumentGraph)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = fw.sweep(gd, db, cfgs, keep_schedules=True)
        b = fw.sweep(gp, db, cfgs, keep_schedules=True)
    assert np.array_equal(a.makespan, b.makespan) and np.array_equal(a.cp_len, b.cp_len)
    assert (a.best_index, a.best_makespan) == (b.best_index, b.best_makespan)
    assert a.schedule(a.best_index).to_json() == b.schedule(b.best_index).to_json()
    t_doc = fw.estimate_all(gd, db, cfgs[0]) if name == "layered" else None
    if t_doc is not None:
        t_ref = fw.estimate_all(gp, db, cfgs[0])
        assert {k: (e.duration_us, e.source) for k, e in t_doc.entries.items()} == \
               {k: (e.duration_us, e.source) for k, e in t_ref.entries.items()}
