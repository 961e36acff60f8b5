"""GPU: the bench configurations at FULL size against the oracle, every candidate.

* C2 (headline): ResNet-50 DP8, 65,536 candidates, N = 4,619, run exactly as bench.py runs
  it -- every schedule, makespan, busy row, critical path and the best index bit for bit.
* C3 / C4: all 10,032 / 16,384 candidates (45 / 18 topology classes) through
  sweep_variants -- makespans, critical paths, busy, best index; plus the engine invariants
  (engine.py:96-146) on every schedule.
* C5 (tests/test_gpu_dag1m.py): the 1M-node DAG.
Oracle: oracle/parity.py (estimate_all restated in Python, C simulate + critical path)."""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_headline_class_full_size_properties():
    """Every one of the 65,536 candidates of the headline class (exactly as bench.py builds and
    runs it) against the oracle: the complete schedule (start and finish of all 4,619 nodes),
    the makespan, per-device busy, the critical-path length and its first node, bit for bit,
    and the best index (first minimum, K5).  Oracle: estimate_all restated in Python once per
    hardware tag (+ op_gap as the reference's one IEEE add, oracle/parity.py) and the C
    restatement of simulate + critical_path on all host cores."""
    import torch

    sys.path.insert(0, str(ROOT))
    import bench
    from oracle import parity
    from paper_2002_06790_b200.batch import TopologyClass

    graphs, db, configs, _ = bench.build_workload(0, 65536, "resnet50-dp8")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tc = TopologyClass(graphs[0], db, configs, 0)
    assert tc.fused
    tc.expand()
    o = tc.run(schedules=True)
    rec = tc.best(o).cpu()
    lg, S, N = tc.lg, len(configs), tc.lg.n
    st, fi = tc.rows_by_rank_batch(o, range(S))   # node-rank order
    assert int((o["n_placed"] == N).sum()) == S
    assert torch.equal(o["makespan"], fi.max(dim=1).values)
    ref = parity.oracle_grid_isolated("resnet50-dp8", sims=65536, schedules=True)
    assert ref["classes"][0][0] == list(lg.ids) and len(ref["classes"]) == 1
    ost, ofi = ref["start"](0), ref["finish"](0)
    for a in range(0, S, 4096):  # every schedule, bit for bit (oracle rows by rank, like st / fi)
        assert np.array_equal(st[a:a + 4096].cpu().numpy(), ost[a:a + 4096]), a
        assert np.array_equal(fi[a:a + 4096].cpu().numpy(), ofi[a:a + 4096]), a
    assert np.array_equal(o["makespan"].cpu().numpy(), ref["makespan"])
    assert np.array_equal(o["cp_len"].cpu().numpy(), ref["cp_len"])
    src = o["cp_src"].cpu().numpy()
    assert [lg.ids[v] for v in src.tolist()] == ref["cp_src_id"]
    busy = o["busy"][:, : lg.n_devices].cpu().numpy()
    want_busy = np.array([[b[d] for d in lg.devices] for b in ref["busy"]])
    assert np.array_equal(busy, want_busy)
    assert float(rec[0]) == ref["makespan"].min()
    assert int(rec[1:2].view(torch.int64)) == parity.first_minimum(ref["makespan"])


def _class_invariants(tc, o):
    """Engine invariants of one topology class's schedules (see the module docstring)."""
    import torch

    lg, N = tc.lg, tc.lg.n
    st, fi = tc.rows_by_rank_batch(o, range(tc.lp.n_sims))
    assert bool((o["n_placed"] == N).all())
    assert bool((fi >= st).all())
    assert torch.equal(o["makespan"], fi.max(dim=1).values)
    off = lg.t_succ_off[: N + 1].long()
    idx = lg.t_succ_idx[: lg.n_edges].long()
    src = torch.repeat_interleave(torch.arange(N, device=st.device), off[1:] - off[:-1])
    assert bool((st[:, idx] >= fi[:, src]).all())
    dev = lg.t_dev[:N].long()
    for d in range(lg.n_devices):
        nodes = torch.nonzero(dev == d).flatten()
        s_d, order = st[:, nodes].sort(dim=1, stable=True)
        f_d = fi[:, nodes].gather(1, order)
        assert bool((s_d[:, 1:] >= f_d[:, :-1]).all())
    assert bool((o["cp_len"] <= o["makespan"] * (1 + 1e-12)).all())


@pytest.mark.parametrize("workload", ["bert-large-ps-ar", "vgg16-sweep"])
def test_multiclass_workloads_full_size(workload):
    """C4 (16,384 candidates, 18 classes) and C3 (10,032 candidates, 45 classes) exactly as the
    bench builds them: per-class invariants on every schedule, oracle bit-parity on a sample."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2002_06790_b200 import sweep_variants

    graphs, db, configs, graph_of = bench.build_workload(0, bench.WORKLOADS[workload][1], workload)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = sweep_variants(graphs, db, configs, graph_of, keep_schedules=True)
    for tc, _, o in res.classes:
        _class_invariants(tc, o)
    # every candidate against the oracle (oracle/parity.py: Python estimate once per class and
    # (hardware, collective) variant, C simulate + critical path on all host cores)
    from oracle import parity

    ref = parity.oracle_grid_isolated(workload)
    assert np.array_equal(res.makespan, ref["makespan"])
    assert np.array_equal(res.cp_len, ref["cp_len"])
    assert res.best_index == parity.first_minimum(ref["makespan"])
    assert res.best_makespan == ref["makespan"].min()
    for tc, idx, o in res.classes:  # per-device busy of every candidate
        busy = o["busy"][:, : tc.lg.n_devices].cpu().numpy()
        for row, i in enumerate(idx):
            names = tc.objects_for(row)[1]  # device names of this candidate's collective path
            assert [busy[row, d] for d in range(tc.lg.n_devices)] == [ref["busy"][i][d] for d in names]


def test_global_duration_row_class_matches_exact_engine():
    """C4's R=8 parameter-server classes (N = 9,474, 25 devices) leave room for only 13
    candidates per CTA with the duration row in smem, so the fused engine reads that row from
    global memory instead (fused.cu kBaseG). Every schedule must equal the exact engine's and a
    sample the oracle's."""
    import torch

    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2002_06790_b200.batch import TopologyClass

    graphs, db, configs, _ = bench.build_workload(0, 2048, "bert-large-ps-ar")
    configs = [c for c in configs if c.replicas == 8 and c.sync == "parameter_server"
               and c.collective.path == "NVLink"]
    assert len(configs) > 100
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tc = TopologyClass(graphs[0], db, configs, 0)
        ref = TopologyClass(graphs[0], db, configs, 0, fused=False)
    assert tc.fused and tc.lg.n > 8192 and tc.lg.n_devices > 16
    assert tc.chunk_capacity > 13  # the smem-row layout's capacity for this class
    for c in (tc, ref):
        c.expand()
    o, r = tc.run(schedules=True), ref.run(schedules=True)
    N = tc.lg.n
    st, fi = tc.rows_by_rank_batch(o, range(len(configs)))
    assert torch.equal(st, r["start"][:, :N]) and torch.equal(fi, r["finish"][:, :N])
    assert torch.equal(o["makespan"], r["makespan"])
    assert torch.equal(o["cp_len"], r["cp_len"])
    for i in (0, len(configs) // 2, len(configs) - 1):
        assert float(o["makespan"][i]) == bench._run_candidate_ps_aware(graphs[0], db, configs[i])
