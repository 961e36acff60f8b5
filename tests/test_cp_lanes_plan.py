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
    """The kernel's data movement for one candidate (one lane): value rows [slots | spill
    stages], chunk blocks and spill values prefetched ``stages - 1`` chunks ahead."""
    NS, RM, ST = plan["n_slots"], plan["rmax"], plan["smem_stages"]
    rows = np.full(NS + ST * RM, np.nan)
    spill = np.full(max(plan["n_long"], 1), np.nan)
    blocks = plan["blocks"].reshape(-1, 4)
    boff, b, so, sl = plan["block_off"], plan["bounds"], plan["spill_off"], plan["spill_list"]
    NQ = plan["n_chunks"]
    staged = {}

    def prefetch(q):  # the chunk's block and spill values, into stage q % ST
        staged[q % ST] = blocks[boff[q]:boff[q + 1]].copy()
        for r in range(so[q], so[q + 1]):
            rows[NS + (q % ST) * RM + (r - so[q])] = spill[sl[r]]

    length, src = 0.0, None
    for q in range(min(ST - 1, NQ)):
        prefetch(q)
    for q in range(NQ):
        if q + ST - 1 < NQ:
            prefetch(q + ST - 1)
        assert b[q] - b[q + 1] <= plan["K"]
        blk = staged[q % ST]
        ext = blk.view(np.uint16).reshape(-1)
        for i, p in enumerate(range(b[q] - 1, b[q + 1] - 1, -1)):
            x, y, z, w = (int(v) for v in blk[i])
            deg = y & 0xFF
            succ = [z & 0xFFFF, z >> 16, w & 0xFFFF, w >> 16][: min(deg, 4)]
            succ += [int(ext[(y >> 8) + k]) for k in range(deg - 4)] if deg > 4 else []
            best = 0.0
            for e in succ:
                v = rows[e]
                assert not np.isnan(v), ("stale read", p, e)
                best = v if v > best else best
            sv = d_by_pos[p] + best
            if x & (1 << 12):
                rows[x & 0xFFF] = sv
            if x & (1 << 14):
                spill[x >> 15] = sv
            if x & (1 << 13):
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


def _check(off, idx, indeg, rng, K, stages=3, rmax=8, near=1):
    n = len(indeg)
    t = Tables(n, 1, off, idx, indeg, np.zeros(n, np.int64))
    plan = lane_plan(t, K=K, rmax_min=rmax, stages=stages, near=near)
    assert plan is not None
    csr = _Csr(off, idx, indeg)
    for trial in range(3):
        d = [rng.uniform(0, 10, n), np.round(rng.uniform(0, 3, n)), np.where(rng.random(n) < 0.4, 0.0, 1.0)][trial]
        rc, length, path = NO.critical_path(csr, d)
        assert rc == 0
        assert emulate(t, plan, d[t.rank_of_pos]) == (length, path[0])
    return plan


@pytest.mark.parametrize("K, stages, near", [(8, 0, 1), (8, 0, 8), (8, 2, 3), (8, 3, 1), (16, 2, 1), (16, 3, 5)])
@pytest.mark.parametrize("seed", range(4))
def test_plan_random_dags(K, stages, near, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    off, idx, indeg = _random_dag(n, rng, window=int(rng.integers(2, 800)), max_in=int(rng.integers(1, 7)))
    _check(off, idx, indeg, rng, K, stages, near=near)


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
                  np.random.default_rng(0), 8, stages=0, near=8)
    assert plan["n_slots"] <= 40 and plan["n_long"] > 1000
