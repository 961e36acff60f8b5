"""CPU: the per-class tables of the fused kernels (prepare.Tables).  An exact emulation of
K4 v2 (reverse level order, smem slots, spill rows, one-chunk-ahead prefetch) driven by
the tables must reproduce the oracle's critical path, and the engine's packed successor /
counter encodings must decode back to the CSR.  The kernels execute these tables as-is,
so this pins the host-side construction independently of a GPU."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import dfsim_oracle as O
from oracle import native_oracle as NO
from paper_2002_06790_b200 import workloads as W
from paper_2002_06790_b200.lowering import host_csr
from paper_2002_06790_b200.prepare import Tables


def emulate_cp(t: Tables, start_by_pos, finish_by_pos):
    """K4 v2 semantics: reverse chunks, reverse groups, slots + spill row + per-chunk prefetch."""
    N = t.n
    region = np.full(t.slot_region + 2 * t.stage_doubles, np.nan)
    spill = np.full(max(t.n_long, 1), np.nan)
    best_len, best_src = None, None
    K = t.chunk

    def prefetch(c):
        p0, p1 = t.group_off[t.chunk_off[c]], t.group_off[t.chunk_off[c + 1]]
        base = t.slot_region + (c & 1) * t.stage_doubles
        for p in range(p0, p1):
            region[base + 2 * (p - p0)] = start_by_pos[p]
            region[base + 2 * (p - p0) + 1] = finish_by_pos[p]
        for r in range(t.spill_off[c], t.spill_off[c + 1]):
            region[base + 2 * K + (r - t.spill_off[c])] = spill[t.spill_list[r]]

    if t.n_chunks:
        prefetch(t.n_chunks - 1)
    for c in range(t.n_chunks - 1, -1, -1):
        if c > 0:
            prefetch(c - 1)
        base = t.slot_region + (c & 1) * t.stage_doubles
        p0 = t.group_off[t.chunk_off[c]]
        for gi in range(t.chunk_off[c + 1] - 1, t.chunk_off[c] - 1, -1):
            vals = []
            for p in range(t.group_off[gi], t.group_off[gi + 1]):
                m = int(t.cp_meta[p])
                j0, j1 = m & 0xFFFF, (m & 0xFFFF) + ((m >> 16) & 0xFF)
                best = 0.0
                for j in range(j0, j1):
                    x = region[int(t.cp_succ_abs[j])]
                    assert not np.isnan(x), "read a value that was never written/prefetched"
                    best = x if x > best else best
                d = region[base + 2 * (p - p0) + 1] - region[base + 2 * (p - p0)]
                vals.append((p, d + best, m))
            for p, sv, m in vals:  # the group's writes land after all its reads (no intra-level edges)
                info = int(t.pinfo[p])
                if info & 0x8000:
                    region[info & 0x7FFF] = sv
                if info >> 31:
                    spill[(info >> 16) & 0x7FFF] = sv
                if (m >> 24) & 1:
                    r = int(t.rank_of_pos[p])
                    if best_len is None or sv > best_len or (sv == best_len and r < best_src):
                        best_len, best_src = sv, r
    return (0.0 if best_len is None else best_len), best_src


@pytest.mark.parametrize("seed", range(6))
def test_cp_tables_reproduce_oracle(seed):
    g = W.random_dag(120 + 40 * seed, 0.03, seed=seed, num_devices=1 + seed % 4)
    h = host_csr(g)
    rng = np.random.default_rng(seed)
    for chunk in (16, 32):
        t = Tables(len(h["ids"]), len(h["devices"]), h["succ_off"], h["succ_idx"], h["indeg"], h["device"],
                   group=16, chunk=chunk)
        assert t.acyclic
        csr = NO.Csr(g)
        dur = rng.uniform(0, 5, size=t.n)
        dur[rng.uniform(size=t.n) < 0.2] = 0.0
        rc, st, fi, _, _, _ = NO.simulate(csr, dur)
        want = O.critical_path(g, {nid: fi[i] - st[i] for i, nid in enumerate(csr.ids)})
        length, src = emulate_cp(t, st[t.rank_of_pos], fi[t.rank_of_pos])
        assert length == want[0]
        assert csr.ids[src] == want[1][0]


def test_cp_tables_resnet_dp8_spill_windows():
    g = W.resnet50_training(batch=8)
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig

    cfg = StrategyConfig(replicas=8, device_map=tuple(f"gpu{i}" for i in range(8)),
                         collective=CollectiveConfig("RingAnalytic", "NVLink"), gradient_markers=("wgrad_*",))
    gx = O.expand(g, cfg)[0]
    h = host_csr(gx)
    t = Tables(len(h["ids"]), len(h["devices"]), h["succ_off"], h["succ_idx"], h["indeg"], h["device"])
    assert t.fused_ok and t.n_long > 1000 and t.n_slots < 100
    csr = NO.Csr(gx)
    rng = np.random.default_rng(3)
    dur = rng.uniform(0.5, 50, size=t.n)
    rc, st, fi, _, _, _ = NO.simulate(csr, dur)
    want = O.critical_path(gx, {nid: fi[i] - st[i] for i, nid in enumerate(csr.ids)})
    assert emulate_cp(t, st[t.rank_of_pos], fi[t.rank_of_pos])[0] == want[0]


@pytest.mark.parametrize("seed", range(4))
def test_engine_tables_packing(seed):
    """succ entries, counter slots and packed initial counters encode the CSR exactly."""
    g = W.random_dag(150, 0.04, seed=seed, num_devices=3)
    h = host_csr(g)
    t = Tables(len(h["ids"]), len(h["devices"]), h["succ_off"], h["succ_idx"], h["indeg"], h["device"])
    indeg, off, idx, dev = h["indeg"], h["succ_off"], h["succ_idx"], h["device"]
    pos, rank = t.pos, t.rank_of_pos

    def field(word, shift, width):
        return (int(t.cnt_init[word]) >> shift) & ((1 << width) - 1)

    for p in range(t.n):  # engine tables are numbered by level position
        v = int(rank[p])
        m = int(t.meta[p])
        b, d = m & 0xFFFFFF, m >> 24
        assert d == off[v + 1] - off[v]
        got = []
        for j in range(b, b + d):
            e = int(t.succ[j])
            if t.succ_packed:
                mp, dv, single = e & 0x1FFF, (e >> 13) & 15, (e >> 17) & 1
                width, shift, word = (4 if (e >> 18) & 1 else 2), (e >> 19) & 31, e >> 24
            else:
                mp, dv, single = e & 0xFFFF, (e >> 16) & 31, (e >> 21) & 1
                code = int(t.cidx[mp])
                width, shift, word = 2 << (code & 3), (code >> 2) & 31, code >> 7
            mr = int(rank[mp])
            assert dv == dev[mr] and single == (indeg[mr] == 1)
            if indeg[mr] >= 2:
                assert field(word, shift, width) == indeg[mr] and indeg[mr] < (1 << width)
            got.append(mr)
        assert got == list(idx[off[v]:off[v + 1]])
    # every multi-input node owns a distinct field
    codes = [int(t.cidx[p]) for p in range(t.n) if indeg[int(rank[p])] >= 2]
    assert len(set(codes)) == len(codes)
    assert [int(rank[p]) for p in t.eng_sources] == [v for v in range(t.n) if indeg[v] == 0]
    assert (pos[rank] == np.arange(t.n)).all()


def test_engine_tables_wide_counters_unpacked():
    """In-degrees beyond 15 need 8-bit counter fields: the unpacked format with cidx codes."""
    from paper_2002_06790_b200.model import DeviceSpec, OpNode, make_graph

    nodes = [OpNode(f"s{i:02d}", "Op", f"gpu{i % 3}") for i in range(20)]
    nodes.append(OpNode("sink", "Op", "gpu0", inputs=tuple((f"s{i:02d}", 0) for i in range(20))))
    nodes += [OpNode(f"t{i}", "Op", "gpu1", inputs=(("sink", 0), ("s00", 0))) for i in range(3)]
    g = make_graph(nodes, [DeviceSpec(f"gpu{i}", "Compute") for i in range(3)])
    h = host_csr(g)
    t = Tables(len(h["ids"]), len(h["devices"]), h["succ_off"], h["succ_idx"], h["indeg"], h["device"])
    assert t.fused_ok and not t.succ_packed and t.counter_bits == 8
    for p in range(t.n):
        v = int(t.rank_of_pos[p])
        if h["indeg"][v] >= 2:
            code = int(t.cidx[p])
            width, shift, word = 2 << (code & 3), (code >> 2) & 31, code >> 7
            assert (int(t.cnt_init[word]) >> shift) & ((1 << width) - 1) == h["indeg"][v]


def test_dense_class_exceeds_critical_path_smem():
    """The class of tests/test_gpu_fuzz.py::test_dense_class_beyond_critical_path_smem passes
    the engine's table limits (fused_ok) while its level-order critical-path tables exceed
    one CTA's shared memory (the layout of csrc/fused.cu cp_shape), so that GPU test runs
    the capacity check's fallback."""
    import warnings

    from oracle import dfsim_oracle as O
    from oracle import native_oracle as NO
    from paper_2002_06790_b200 import workloads as W
    from paper_2002_06790_b200.model import CollectiveConfig, StrategyConfig
    from paper_2002_06790_b200.prepare import Tables

    g = W.random_dag(295, 0.14186208467922018, seed=50280, num_devices=4)
    cfg = StrategyConfig(replicas=7, device_map=tuple(f"gpu{k}" for k in range(7)),
                         collective=CollectiveConfig("RingAnalytic", "PCIeSwitch"), gradient_markers=("node_02*",),
                         hardware="hwA")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        gx = O.expand(g, cfg)[0]
    c = NO.Csr(gx)
    idx = np.asarray(c.idx)
    t = Tables(c.n, c.n_dev, np.asarray(c.off), idx, np.asarray(c.indeg), np.asarray(c.dev))
    assert t.fused_ok
    table = (c.n * 8 + len(idx) * 4 + (t.n_groups + 1) * 2 + (t.n_chunks + 1) * 4 + 15) // 16 * 16
    per_warp = 2 * (t.slot_region + 2 * t.stage_doubles) * 8
    assert table + per_warp > 227 * 1024 - 64
