"""CPU: the K4 v3 storage plan (dfsim_cp_lanes_plan, host C++ in libdfsim_b200.so).

The kernel keeps a suffix value in a shared-memory slot while it is read within the writer's
prefetch chunk or the next one, and in a global spill row otherwise, prefetched into a
stage with the reading chunk *before* the previous chunk runs.  A wrong plan (a slot reused
while still needed, a spill value prefetched before it is written, a stage row overwritten)
would read a stale value.  Here the kernel's exact data movement is emulated in numpy --
NaN-poisoned storage, prefetch timing as in the kernel -- and the critical-path length and
start node must equal the C oracle (graph.py:446-485) on DAGs with long-lived values, fan-outs
wider than the spill stage, ties and zeros.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import native_oracle as NO
from paper_2002_06790_b200.prepare import Tables, lane_plan


class _Csr:
    def __init__(self, off, idx, indeg):
        self.n = len(indeg)
        self.off, self.idx, self.indeg = (np.ascontiguousarray(a, np.int32) for a in (off, idx, indeg))


def emulate(t, plan, d_by_pos):
    NS, RM = plan["n_slots"], plan["rmax"]
    rows = np.full(NS + 2 * RM, np.nan)
    spill = np.full(max(plan["n_long"], 1), np.nan)
    rec = plan["rec"].reshape(-1, 2)
    succ, b, so, sl = plan["succ"], plan["bounds"], plan["spill_off"], plan["spill_list"]
    NQ = plan["n_chunks"]

    def prefetch(q):  # issued before chunk q - 1 runs (kernel: one chunk ahead)
        for r in range(so[q], so[q + 1]):
            rows[NS + (q & 1) * RM + (r - so[q])] = spill[sl[r]]

    length, src = 0.0, None
    prefetch(0)
    for q in range(NQ):
        if q + 1 < NQ:
            prefetch(q + 1)
        assert b[q] - b[q + 1] <= plan["K"]
        for p in range(b[q] - 1, b[q + 1] - 1, -1):
            x, y = int(rec[p, 0]), int(rec[p, 1])
            best = 0.0
            for j in range(x & 0xFFFFFF, (x & 0xFFFFFF) + (x >> 24)):
                v = rows[succ[j]]
                assert not np.isnan(v), ("stale read", p, j)
                best = v if v > best else best
            sv = d_by_pos[p] + best
            if y & (1 << 12):
                rows[y & 0xFFF] = sv
            if y & (1 << 14):
                spill[y >> 15] = sv
            if y & (1 << 13):
                rk = t.rank_of_pos[p]
                if src is None or sv > length or (sv == length and rk < src):
                    length, src = sv, rk
    return length, src


def _random_dag(n, rng, window, max_in=3, hub_every=0):
    ins = [[] for _ in range(n)]
    for v in range(1, n):
        k = int(rng.integers(0, max_in + 1))
        lo = max(0, v - window)
        ins[v] = sorted(set(int(p) for p in rng.integers(lo, v, k)))
        if hub_every and v % hub_every == 0:
            ins[v].append(0)  # everything also depends on node 0: a very wide fan-out
    succ = [[] for _ in range(n)]
    for v in range(n):
        for p in ins[v]:
            succ[p].append(v)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in succ])
    idx = np.asarray([m for s in succ for m in sorted(s)], np.int64)
    indeg = np.asarray([len(i) for i in ins], np.int64)
    return off, idx, indeg


def _check(off, idx, indeg, rng, K):
    n = len(indeg)
    t = Tables(n, 1, off, idx, indeg, np.zeros(n, np.int64))
    plan = lane_plan(t, K=K)
    assert plan is not None
    csr = _Csr(off, idx, indeg)
    for trial in range(3):
        d = [rng.uniform(0, 10, n), np.round(rng.uniform(0, 3, n)), np.where(rng.random(n) < 0.4, 0.0, 1.0)][trial]
        rc, length, path = NO.critical_path(csr, d)
        assert rc == 0
        assert emulate(t, plan, d[t.rank_of_pos]) == (length, path[0])
    return plan


@pytest.mark.parametrize("K", [8, 16])
@pytest.mark.parametrize("seed", range(4))
def test_plan_random_dags(K, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    off, idx, indeg = _random_dag(n, rng, window=int(rng.integers(2, 800)))
    _check(off, idx, indeg, rng, K)


def test_plan_wide_fanout_widens_stage():
    rng = np.random.default_rng(7)
    off, idx, indeg = _random_dag(1500, rng, window=5, hub_every=20)  # node 0 feeds ~75 far nodes
    plan = _check(off, idx, indeg, rng, 16)
    assert plan["n_long"] > 0


@pytest.mark.parametrize("n", [1, 2, 7, 17])
def test_plan_tiny_graphs(n):
    rng = np.random.default_rng(n)
    off, idx, indeg = _random_dag(n, rng, window=3)
    _check(off, idx, indeg, rng, 16)


def test_plan_resnet50_dp8_class():
    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    g = W.resnet50_training(batch=32)
    cfg = StrategyConfig(replicas=8, device_map=tuple(f"gpu{i}" for i in range(8)),
                         collective=CollectiveConfig("RingAnalytic", "NVLink"), gradient_markers=("wgrad_*",))
    c = NO.Csr(O.expand(g, cfg)[0])
    plan = _check(c.off.astype(np.int64), c.idx.astype(np.int64), c.indeg.astype(np.int64),
                  np.random.default_rng(0), 16)
    assert plan["n_slots"] <= 32 and plan["rmax"] == 16 and plan["n_long"] > 1000
