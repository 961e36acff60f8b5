"""GPU: size-independent properties at the headline configuration's FULL size.

The bench's C2 class (ResNet-50 DP8, 65,536 candidates, N = 4,619) is run exactly as
bench.py runs it; every candidate's schedule must then satisfy the engine's invariants
(engine.py:96-146): dependencies respected, no two nodes overlapping on one device,
makespan = max finish, busy = per-device sum of (finish - start), the critical path no
longer than the makespan -- and a sample of candidates spread over the grid must equal
the oracle bit for bit."""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_headline_class_full_size_properties():
    import torch

    sys.path.insert(0, str(ROOT))
    import bench
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200.batch import TopologyClass

    graphs, db, configs, _ = bench.build_workload(0, 65536, "resnet50-dp8")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tc = TopologyClass(graphs[0], db, configs, 0)
    assert tc.fused
    tc.expand()
    o = tc.run(schedules=True)
    lg, S, N = tc.lg, len(configs), tc.lg.n
    pos = torch.as_tensor(tc.tables.pos, device="cuda:0")
    st = o["start"][:, :N].index_select(1, pos)   # node-rank order
    fi = o["finish"][:, :N].index_select(1, pos)
    assert int((o["n_placed"] == N).sum()) == S
    assert bool((fi >= st).all())
    assert torch.equal(o["makespan"], fi.max(dim=1).values)
    # dependencies: start of every consumer >= finish of each producer
    off = lg.t_succ_off[: N + 1].long()
    idx = lg.t_succ_idx[: lg.n_edges].long()
    src = torch.repeat_interleave(torch.arange(N, device="cuda:0"), off[1:] - off[:-1])
    for a in range(0, S, 8192):
        assert bool((st[a:a + 8192, idx] >= fi[a:a + 8192, src]).all())
    # one node at a time per device, busy = sum of durations per device
    dev = lg.t_dev[:N].long()
    busy = o["busy"]
    for d in range(lg.n_devices):
        nodes = torch.nonzero(dev == d).flatten()
        s_d, order = st[:, nodes].sort(dim=1, stable=True)
        f_d = fi[:, nodes].gather(1, order)
        assert bool((s_d[:, 1:] >= f_d[:, :-1]).all()), d
        tot = (f_d - s_d).sum(dim=1)
        assert torch.allclose(busy[:, d], tot, rtol=1e-12, atol=0.0), d
    assert bool((o["cp_len"] <= o["makespan"] * (1 + 1e-12)).all())
    # oracle bit-parity on candidates spread over hardware tags and the op_gap grid
    for i in np.linspace(0, S - 1, 12).astype(int).tolist():
        ms, cp, entries, _, _ = O.run_candidate(graphs[0], db, configs[i])
        assert float(o["makespan"][i]) == ms and float(o["cp_len"][i]) == cp, i
        rank = lg.rank_of()
        got_s, got_f = st[i].cpu().numpy(), fi[i].cpu().numpy()
        for nid, _, s, f in entries:
            assert got_s[rank[nid]] == s and got_f[rank[nid]] == f, (i, nid)


def _class_invariants(tc, o):
    """Engine invariants of one topology class's schedules (see the module docstring)."""
    import torch

    lg, N = tc.lg, tc.lg.n
    st, fi = o["start"][:, :N], o["finish"][:, :N]
    if o.get("layout") == "position":
        pos = torch.as_tensor(tc.tables.pos, device=st.device)
        st, fi = st.index_select(1, pos), fi.index_select(1, pos)
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
    ms = res.makespan
    assert res.best_index == int(np.lexsort((np.arange(len(ms)), ms))[0])
    n_check = 24 if workload == "vgg16-sweep" else 8  # oracle seconds per candidate: ~0.05 (C3), ~0.5 (C4)
    for i in np.linspace(0, len(configs) - 1, n_check).astype(int).tolist():
        want = bench._run_candidate_ps_aware(graphs[graph_of[i]], db, configs[i])
        assert res.makespan[i] == want, (workload, i)


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
    pos = torch.as_tensor(tc.tables.pos, device="cuda:0")
    assert torch.equal(o["start"][:, :N].index_select(1, pos), r["start"][:, :N])
    assert torch.equal(o["finish"][:, :N].index_select(1, pos), r["finish"][:, :N])
    assert torch.equal(o["makespan"], r["makespan"])
    assert torch.equal(o["cp_len"], r["cp_len"])
    for i in (0, len(configs) // 2, len(configs) - 1):
        assert float(o["makespan"][i]) == bench._run_candidate_ps_aware(graphs[0], db, configs[i])
