"""GPU: configuration C5 at full size -- the 1M-node layered DAG (bench.py ``dag1m``).

* The large-graph engine (K3 large) and the wide critical path (K4 wide) on three duration
  rows -- continuous, tie-heavy integers, zero-heavy -- against the C oracle: every start and
  finish of the 1,000,000 nodes, makespan, busy, critical-path length and first node.
* The bench's own candidate path (estimate on the device -> simulate -> critical path) for
  two candidates of one hardware tag against the oracle's estimate + C engine.
* A forced ring overflow at full size (``DFSIM_LARGE_QCAP=16``: a level of 1,000 nodes over
  8 devices queues ~125 nodes per device) must re-run exactly and change nothing.
"""

from __future__ import annotations

import os
import subprocess
import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def dag():
    from oracle import native_oracle as NO
    from paper_2002_06790_b200 import workloads as W

    g = W.layered_dag(1_000_000, 1000, devices=8)
    return g, NO.Csr(g)


def _rows(n, seed=3):
    rng = np.random.default_rng(seed)
    return np.stack([rng.uniform(0.5, 30, n), rng.integers(1, 5, n).astype(np.float64),
                     np.where(rng.random(n) < 0.3, 0.0, rng.uniform(0, 3, n))])


def check_engine_full(g, csr, rows):
    import torch

    from oracle import native_oracle as NO
    from paper_2002_06790_b200.lowering import LoweredGraph
    from paper_2002_06790_b200.simulator import critical_path_arrays, simulate_arrays

    lg = LoweredGraph(g, 0)
    assert list(csr.ids) == list(lg.ids) and lg.n == 1_000_000
    from paper_2002_06790_b200 import native

    o = simulate_arrays(lg, torch.tensor(rows, device="cuda:0"))
    cp = critical_path_arrays(lg, o["start"], o["finish"], paths=True)  # K4 v1 (+ path walk)
    order, loff, nl = lg.levels()  # K4 wide: the bench's critical path at this size
    S = len(rows)
    wide = torch.empty(S, dtype=torch.float64, device="cuda:0")
    wsrc = torch.empty(S, dtype=torch.int32, device="cuda:0")
    lg.ctx.call("dfsim_critical_path_wide", native.ctypes.byref(lg.struct), native.ptr(order), native.ptr(loff), nl,
                S, native.ptr(o["start"]), native.ptr(o["finish"]), native.ptr(wide), native.ptr(wsrc))
    rc, ms, cpl, st, fi, busy, src = NO.simulate_batch_full(csr, rows, threads=len(rows))
    assert rc == 0
    assert (o["n_placed"].cpu().numpy() == lg.n).all()
    assert np.array_equal(o["start"][:, : lg.n].cpu().numpy(), st)
    assert np.array_equal(o["finish"][:, : lg.n].cpu().numpy(), fi)
    assert np.array_equal(o["makespan"].cpu().numpy(), ms)
    assert np.array_equal(o["busy"][:, : lg.n_devices].cpu().numpy(), busy)
    assert np.array_equal(cp["cp_len"].cpu().numpy(), cpl)
    assert np.array_equal(cp["cp_path"][:, 0].cpu().numpy(), src)
    assert np.array_equal(wide.cpu().numpy(), cpl) and np.array_equal(wsrc.cpu().numpy(), src)


def test_dag1m_engine_and_critical_path_full_size(dag):
    g, csr = dag
    check_engine_full(g, csr, _rows(csr.n))


def test_dag1m_bench_candidates_full_size(dag):
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle import parity
    from paper_2002_06790_b200.batch import TopologyClass

    g, _ = dag
    _, db, configs, _ = bench.build_workload(0, 2 * bench.N_HW, "dag1m")
    pick = [configs[0], configs[bench.N_HW]]  # one hardware tag, op_gap 0 and 1e-3
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        tc = TopologyClass(g, db, pick, 0)
    o = tc.run(schedules=False)
    ref = parity.oracle_grid_isolated("dag1m", sims=2 * bench.N_HW, select=[0, bench.N_HW])
    assert np.array_equal(o["makespan"].cpu().numpy(), ref["makespan"])
    assert np.array_equal(o["cp_len"].cpu().numpy(), ref["cp_len"])


def test_dag1m_forced_ring_overflow_full_size():
    """The exact re-run after a ring overflow, at full size, in a fresh process (the ring
    capacity is read once per process)."""
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import numpy as np, test_gpu_dag1m as T\n"
            "from paper_2002_06790_b200 import workloads as W\n"
            "from oracle import native_oracle as NO\n"
            "g = W.layered_dag(1_000_000, 1000, devices=8); csr = NO.Csr(g)\n"
            "T.check_engine_full(g, csr, T._rows(csr.n, seed=4)[:2])\n"
            "print('overflow-ok')\n") % (str(ROOT), str(ROOT / "tests"))
    env = dict(os.environ, DFSIM_LARGE_QCAP="16")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "overflow-ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
