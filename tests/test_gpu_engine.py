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


@pytest.mark.parametrize("ndev", [33, 100, 256])
def test_engine_many_devices_matches_c_oracle(ndev):
    """More devices than warp lanes (wide PS / DP expansions): lane l owns l, l+32, ..."""
    import torch

    from oracle import native_oracle as NO
    from paper_2002_06790_b200.lowering import LoweredGraph
    from paper_2002_06790_b200.simulator import critical_path_arrays, simulate_arrays
    from paper_2002_06790_b200.workloads import random_dag

    g = random_dag(700, 0.01, seed=ndev, num_devices=ndev)
    lg = LoweredGraph(g)
    csr = NO.Csr(g)
    assert csr.ids == lg.ids and lg.n_devices > 32
    rng = np.random.default_rng(ndev)
    rows = [rng.uniform(0, 9, lg.n), rng.integers(0, 3, lg.n).astype(np.float64)]
    o = simulate_arrays(lg, torch.tensor(np.stack(rows), device="cuda:0"))
    cp = critical_path_arrays(lg, o["start"], o["finish"])["cp_len"].cpu().numpy()
    for s, row in enumerate(rows):
        rc, ws, wf, wbusy, wms, _ = NO.simulate(csr, row)
        assert rc == 0 and int(o["n_placed"][s]) == lg.n
        assert np.array_equal(o["start"][s, : lg.n].cpu().numpy(), ws)
        assert np.array_equal(o["finish"][s, : lg.n].cpu().numpy(), wf)
        assert float(o["makespan"][s]) == wms
        got = dict(zip(lg.devices, o["busy"][s, : lg.n_devices].cpu().numpy().tolist()))
        want = dict(zip(csr.devices, wbusy.tolist()))
        assert got == {d: b for d, b in want.items() if d in got} and all(want[d] == 0.0 for d in want if d not in got)
        assert cp[s] == NO.critical_path(csr, wf - ws)[1]


def test_parameter_server_sixteen_workers_vs_oracle():
    """PS with 16 workers has 49 devices (PS + 16 GPUs + 32 links): the wide-device engine."""
    import warnings

    import paper_2002_06790_b200 as fw
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig
    from paper_2002_06790_b200.ps import expand_parameter_server

    g = W.vgg16_training(batch=16)
    db = W.model_profiles(g, ["hw0"])
    cfgs = [StrategyConfig(replicas=16, device_map=tuple(f"gpu{k}" for k in range(16)),
                           collective=CollectiveConfig("MeasuredThroughput", "NVLink"), gradient_markers=("wgrad_*",),
                           hardware="hw0", op_gap_us=0.1 * i, sync="parameter_server") for i in range(3)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = fw.sweep(g, db, cfgs, keep_schedules=True)
    for i, cfg in enumerate(cfgs):
        gx = expand_parameter_server(g, cfg, db).graph
        assert len(gx.devices) > 32
        table = O.estimate(gx, db, cfg)
        entries, ms, busy = O.simulate(gx, {k: v for k, (v, _) in table.items()})
        cp = O.critical_path(gx, {nid: f - s for nid, _, s, f in entries})
        assert res.makespan[i] == ms and res.cp_len[i] == cp[0], i


@pytest.mark.parametrize("n", [1, 1000, 16384, 16385, 65536, 1_000_003])
def test_argmin_first_minimum(n):
    """K5: first minimum of (value, index) -- single-CTA and two-pass paths, ties across slices."""
    import torch

    from paper_2002_06790_b200 import native

    rng = np.random.default_rng(n)
    vals = rng.integers(0, 50, n).astype(np.float64)
    vals[rng.integers(0, n, 5)] = -1.0  # several tying minima
    t = torch.tensor(vals, device="cuda:0")
    rec = torch.empty(2, dtype=torch.float64, device="cuda:0")
    ctx = native.Context.get(0)
    ctx.call("dfsim_argmin", n, native.ptr(t), 7, native.ptr(rec))
    r = rec.cpu()
    assert float(r[0]) == vals.min() and int(r[1:2].view(torch.int64)) == 7 + int(np.argmin(vals))
