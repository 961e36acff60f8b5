"""GPU parity: K3 simulate + K4 critical path vs the reference's own outputs.

Every golden engine case (tests/golden/engine_cases.json.gz, produced by the
real dfsim) goes through the drop-in ``simulate`` / ``critical_path`` and must
match bit-for-bit: entry order, start/finish, makespan, busy, CP length + path.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import case_graph, case_table

pytestmark = pytest.mark.gpu


def _check_case(case):
    import paper_2002_06790_b200 as fw

    g, table, exp = case_graph(case), case_table(case), case["expect"]
    if exp.get("error") == "MissingDurationError":
        with pytest.raises(fw.MissingDurationError) as err:
            fw.simulate(g, table)
        assert err.value.node_ids == exp["ids"]
        return
    if exp.get("error") == "CycleError":
        with pytest.raises(fw.CycleError) as err:
            fw.simulate(g, table)
        assert err.value.cycle == exp["ids"]
        return
    s = fw.simulate(g, table)
    assert [[e.node_id, e.device, e.start_us, e.finish_us, e.source, e.op_type] for e in s.entries] == \
        exp["schedule"]["entries"], case["name"]
    assert s.makespan_us == exp["schedule"]["makespan_us"]
    assert s.per_device_busy_us == exp["schedule"]["per_device_busy_us"]
    assert s.to_json() == __import__("json").dumps(exp["schedule"])
    cp = fw.critical_path(g, {e.node_id: e.finish_us - e.start_us for e in s.entries})
    assert [cp[0], cp[1]] == exp["cp"], case["name"]


def test_engine_golden_cases(engine_cases):
    for case in engine_cases:
        _check_case(case)


def test_batched_engine_matches_c_oracle():
    """Many duration rows through one launch vs the C oracle, incl. ties and zeros."""
    import torch

    from oracle import native_oracle as NO
    from paper_2002_06790_b200.lowering import LoweredGraph
    from paper_2002_06790_b200.simulator import critical_path_arrays, simulate_arrays
    from paper_2002_06790_b200.workloads import random_dag

    g = random_dag(400, 0.02, seed=3, num_devices=7)
    lg = LoweredGraph(g)
    csr = NO.Csr(g)
    assert csr.ids == lg.ids
    rng = np.random.default_rng(0)
    S = 96
    dur = rng.uniform(0, 5, size=(S, lg.n))
    dur[rng.uniform(size=dur.shape) < 0.15] = 0.0
    dur[rng.uniform(size=dur.shape) < 0.2] = 1.0
    t = torch.from_numpy(dur).cuda()
    o = simulate_arrays(lg, t)
    cp = critical_path_arrays(lg, o["start"], o["finish"], paths=True)
    start, finish = o["start"].cpu().numpy(), o["finish"].cpu().numpy()
    for s in range(S):
        rc, st, fi, busy, ms, _ = NO.simulate(csr, dur[s])
        assert rc == 0
        assert np.array_equal(st, start[s]) and np.array_equal(fi, finish[s]), s
        assert ms == o["makespan"][s].item()
        assert np.array_equal(busy, o["busy"][s].cpu().numpy())
        rc, length, path = NO.critical_path(csr, fi - st)
        assert length == cp["cp_len"][s].item()
        k = cp["cp_path_len"][s].item()
        assert list(path) == cp["cp_path"][s, :k].cpu().tolist()
