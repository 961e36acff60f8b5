"""GPU: the large-graph kernels agree bit-for-bit with the exact kernels and the oracle.

K4 wide (dfsim_critical_path_wide, one CTA per candidate over the reverse level order)
must give the same critical-path length and start node as K4 v1 (itself pinned on the
reference's golden cases) on general DAGs -- edges spanning many levels, ties, zero
durations -- and on the C5-style layered DAG."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _both(lg, st, fi):
    import torch

    from paper_2002_06790_b200 import native
    from paper_2002_06790_b200.simulator import critical_path_arrays

    ref = critical_path_arrays(lg, st, fi, paths=True)
    order, loff, nl = lg.levels()
    S = fi.shape[0]
    cp = torch.empty(S, dtype=torch.float64, device=fi.device)
    src = torch.empty(S, dtype=torch.int32, device=fi.device)
    lg.ctx.call("dfsim_critical_path_wide", native.ctypes.byref(lg.struct), native.ptr(order), native.ptr(loff), nl,
                S, native.ptr(st), native.ptr(fi), native.ptr(cp), native.ptr(src))
    return ref, cp, src


@pytest.mark.parametrize("seed", range(4))
def test_wide_cp_matches_v1_random_dags(seed):
    import torch

    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.lowering import LoweredGraph

    g = W.random_dag(1200 + 200 * seed, 0.004 * (seed + 1), seed=seed, num_devices=4)
    lg = LoweredGraph(g, 0)
    rng = np.random.default_rng(seed)
    S, N = 7, lg.n
    fi = rng.uniform(0, 10, size=(S, N))
    fi[:, rng.random(N) < 0.2] = 0.0           # zero durations
    fi[1] = np.round(fi[1])                     # ties
    st = np.where(rng.random((S, N)) < 0.5, 0.0, rng.uniform(0, 1, size=(S, N)))
    fi_t = torch.tensor(fi + st, device="cuda:0")
    st_t = torch.tensor(st, device="cuda:0")
    for start in (st_t, None):
        ref, cp, src = _both(lg, start, fi_t if start is not None else torch.tensor(fi, device="cuda:0"))
        assert torch.equal(cp, ref["cp_len"])
        assert torch.equal(src, ref["cp_path"][:, 0])


def test_wide_cp_layered_dag_vs_oracle():
    import torch

    from oracle import dfsim_oracle as O
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.lowering import LoweredGraph

    g = W.layered_dag(60_000, 300, devices=8)
    lg = LoweredGraph(g, 0)
    rng = np.random.default_rng(11)
    d = rng.uniform(0.5, 30, size=(3, lg.n))
    ref, cp, src = _both(lg, None, torch.tensor(d, device="cuda:0"))
    assert torch.equal(cp, ref["cp_len"]) and torch.equal(src, ref["cp_path"][:, 0])
    want = O.critical_path(g, {nid: d[0, i] for i, nid in enumerate(lg.ids)})
    assert float(cp[0]) == want[0] and lg.ids[int(src[0])] == want[1][0]


def _check_engine(g, rows):
    import torch

    from oracle import native_oracle as NO
    from paper_2002_06790_b200.lowering import LoweredGraph
    from paper_2002_06790_b200.simulator import critical_path_arrays, simulate_arrays

    lg = LoweredGraph(g, 0)
    csr = NO.Csr(g)
    assert list(csr.ids) == list(lg.ids)
    o = simulate_arrays(lg, torch.tensor(np.stack(rows), device="cuda:0"))
    cp = critical_path_arrays(lg, o["start"], o["finish"])["cp_len"].cpu().numpy()
    st, fi = o["start"].cpu().numpy(), o["finish"].cpu().numpy()
    for s, row in enumerate(rows):
        rc, ws, wf, wbusy, wms, _ = NO.simulate(csr, row)
        assert rc == 0 and int(o["n_placed"][s]) == lg.n
        assert np.array_equal(st[s, : lg.n], ws) and np.array_equal(fi[s, : lg.n], wf), s
        assert float(o["makespan"][s]) == wms
        assert np.array_equal(o["busy"][s, : lg.n_devices].cpu().numpy(), wbusy)
        assert cp[s] == NO.critical_path(csr, wf - ws)[1]


def test_large_engine_matches_c_oracle():
    """K3 large (smem rings, prefetched successors, plain counters) == the C oracle."""
    from paper_2002_06790_b200 import workloads as W

    g = W.layered_dag(150_000, 500, devices=8)
    rng = np.random.default_rng(5)
    n = len(g.nodes)
    rows = [rng.uniform(0.5, 30, n), rng.integers(1, 5, n).astype(np.float64),
            np.where(rng.random(n) < 0.3, 0.0, rng.uniform(0, 3, n)), np.round(rng.uniform(0, 8, n) * 4) / 4]
    _check_engine(g, rows)


def test_large_engine_ring_overflow_falls_back():
    """A fan-out of 9,000 ready nodes on one device and 100,000 sources on another overflow
    the shared-memory rings; those candidates are re-run exactly."""
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, make_graph

    nodes = [OpNode("a", "Op", "gpu0")]
    nodes += [OpNode(f"b{i:05d}", "Op", "gpu0", inputs=(("a", 0),)) for i in range(9000)]
    nodes += [OpNode(f"c{i:06d}", "Op", "gpu1") for i in range(100_000)]
    g = make_graph(nodes, [DeviceSpec("gpu0", "Compute"), DeviceSpec("gpu1", "Compute")])
    rng = np.random.default_rng(2)
    n = len(nodes)
    _check_engine(g, [rng.uniform(0.5, 3, n), np.ones(n)])


def test_large_engine_duplicate_edges_and_wide_fanout():
    """Repeated producers (two slots of one node: duplicate edges) and hub nodes with
    fan-outs far beyond the kPre carried successors, on the large engine."""
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, TensorShape, make_graph

    rng = np.random.default_rng(9)
    n, D = 150_000, 6
    shapes = (TensorShape((4,), 4), TensorShape((4,), 4))
    nodes = []
    for i in range(n):
        ins = []
        if i:
            for _ in range(int(rng.integers(1, 4))):
                p = int(rng.integers(max(0, i - 1500), i))
                ins.append((f"v{p:06d}", 0))
                if rng.random() < 0.3:
                    ins.append((f"v{p:06d}", 1))  # the same producer again
            if i % 97 == 0 and i % 1000:
                ins.append((f"v{(i // 1000) * 1000:06d}", 0))  # hubs: every 1000th node
        uniq = tuple(dict.fromkeys(ins))
        nodes.append(OpNode(f"v{i:06d}", "Op", f"gpu{i % D}", inputs=uniq, output_shapes=shapes))
    g = make_graph(nodes, [DeviceSpec(f"gpu{k}", "Compute") for k in range(D)])
    rows = [rng.uniform(0.5, 30, n), np.round(rng.uniform(0, 4, n)) / 2]
    _check_engine(g, rows)


@pytest.mark.parametrize("seed", range(3))
def test_large_engine_random_local_dags(seed):
    """Random DAGs beyond the shared-memory engines (producers within a sliding window,
    random devices incl. skewed loads, 1-20 devices): tie-heavy integer durations, zeros,
    and continuous ones, against the C oracle."""
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, make_graph

    rng = np.random.default_rng(100 + seed)
    n, D = 80_000 + 20_000 * seed, int(rng.integers(1, 21))
    win = int(rng.integers(20, 3000))
    devs = rng.integers(0, D, n)
    if seed == 1:
        devs = np.where(rng.random(n) < 0.6, 0, devs)  # one device takes most of the work
    nodes = []
    for i in range(n):
        k = int(rng.integers(0, 4)) if i else 0
        ins = sorted({int(p) for p in rng.integers(max(0, i - win), i, k)}) if i else []
        nodes.append(OpNode(f"x{i:06d}", "Op", f"gpu{devs[i]}", inputs=tuple((f"x{p:06d}", 0) for p in ins)))
    g = make_graph(nodes, [DeviceSpec(f"gpu{d}", "Compute") for d in range(D)])
    rows = [rng.integers(0, 4, n).astype(np.float64), rng.uniform(0.1, 9, n),
            np.where(rng.random(n) < 0.5, 0.0, rng.integers(1, 3, n)).astype(np.float64)]
    _check_engine(g, rows)
