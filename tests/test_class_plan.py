"""CPU: the host C++ class planners (csrc/levels.cpp: dfsim_level_order, dfsim_cp_levels_plan)
equal, array for array, the numpy formulation they replaced (restated here as the checker)
on random DAGs, the headline ResNet-50 DP8 class and C4's PS / AR classes."""

from __future__ import annotations

import types
import warnings

import numpy as np
import pytest

from oracle import dfsim_oracle as O
from paper_2002_06790_b200 import prepare
from paper_2002_06790_b200 import workloads as W
from paper_2002_06790_b200.lowering import host_csr


def np_level_order(n: int, succ_off: np.ndarray, succ_idx: np.ndarray, indeg: np.ndarray):
    """Kahn waves with numpy: returns (order, level_of_rank, level_offsets) or None on a cycle."""
    left = indeg.astype(np.int64).copy()
    frontier = np.nonzero(left == 0)[0]
    order, offsets = [], [0]
    level = np.full(n, -1, dtype=np.int64)
    lv = 0
    while frontier.size:
        frontier = np.sort(frontier)
        order.append(frontier)
        level[frontier] = lv
        offsets.append(offsets[-1] + frontier.size)
        starts, ends = succ_off[frontier], succ_off[frontier + 1]
        cnt = ends - starts
        if cnt.sum() == 0:
            break
        eidx = np.repeat(ends - cnt.cumsum(), cnt) + np.arange(cnt.sum())
        targets = succ_idx[eidx]
        np.subtract.at(left, targets, 1)
        cand = np.unique(targets)
        frontier = cand[left[cand] == 0]
        lv += 1
    order = np.concatenate(order) if order else np.zeros(0, np.int64)
    if order.size != n:
        return None
    return order, level, np.asarray(offsets, dtype=np.int64)


def np_cp_plan(group, chunk, N, idx, indeg, outdeg, order, pos, loff):
    self = types.SimpleNamespace(group=group, chunk=chunk)
    goff = [0]
    for lv in range(loff.size - 1):
        a, b = int(loff[lv]), int(loff[lv + 1])
        for p in range(a, b, self.group):
            goff.append(min(b, p + self.group))
    goff = np.asarray(goff, np.int64)
    coff, start = [0], 0
    for gi in range(1, goff.size):
        if goff[gi] - goff[start] > self.chunk:
            coff.append(gi - 1)
            start = gi - 1
    if coff[-1] != goff.size - 1:
        coff.append(goff.size - 1)
    coff = np.asarray(coff, np.int64)
    n_groups, n_chunks = goff.size - 1, coff.size - 1
    group_of_pos = np.repeat(np.arange(n_groups), np.diff(goff))
    chunk_of_pos = np.repeat(np.arange(n_chunks), np.diff(coff))[group_of_pos]
    step_of_pos = (n_groups - 1) - group_of_pos                  # reverse processing order
    src_of_edge = np.repeat(np.arange(N), outdeg)
    pu, pv = pos[src_of_edge], pos[idx]                          # reader u, written value v
    near = chunk_of_pos[pu] >= chunk_of_pos[pv] - 1
    far = ~near
    last_near = np.full(N, -1, np.int64)
    np.maximum.at(last_near, pv[near], step_of_pos[pu[near]])
    slot_of_pos = np.full(N, 0xFFFF, np.int64)
    free, nslots, release = [], 0, {}
    for g in range(n_groups - 1, -1, -1):
        step = (n_groups - 1) - g
        free.extend(release.pop(step - 1, ()))
        for p in range(int(goff[g]), int(goff[g + 1])):
            if last_near[p] < 0:
                continue
            if free:
                sl = free.pop()
            else:
                sl, nslots = nslots, nslots + 1
            slot_of_pos[p] = sl
            release.setdefault(int(last_near[p]), []).append(sl)
    spill_flag = np.zeros(N, bool)
    spill_flag[pv[far]] = True
    spill_of_pos = np.full(N, 0xFFFF, np.int64)
    spill_of_pos[spill_flag] = np.arange(int(spill_flag.sum()))
    far_chunk, far_k = chunk_of_pos[pu[far]], spill_of_pos[pv[far]]
    pairs = np.unique(np.stack([far_chunk, far_k], 1), axis=0) if far.any() else np.zeros((0, 2), np.int64)
    soff = np.zeros(n_chunks + 1, np.int64)
    if len(pairs):
        np.add.at(soff, pairs[:, 0] + 1, 1)
    soff = np.cumsum(soff)
    bufidx = {(c_, k_): i_ - int(soff[c_]) for i_, (c_, k_) in enumerate(pairs.tolist())}
    ent = np.where(near, slot_of_pos[pv], 0)
    if far.any():
        ent[far] = [0x8000 | bufidx[(c_, k_)] for c_, k_ in zip(far_chunk.tolist(), far_k.tolist())]
    cp_succ = ent[np.argsort(pu, kind="stable")]               # CSR by reading position
    cp_off = np.zeros(N + 1, np.int64)
    cp_off[1:] = np.cumsum(outdeg[order])
    src_flag = (indeg[order] == 0).astype(np.int64)
    self.cp_meta = (cp_off[:-1] & 0xFFFF) | (np.minimum(outdeg[order], 255) << 16) | (src_flag << 24)
    self.cp_slot, self.cp_spill, self.cp_succ = slot_of_pos, spill_of_pos, cp_succ
    has_slot = slot_of_pos != 0xFFFF
    self.pinfo = ((np.where(has_slot, slot_of_pos, 0) & 0x7FFF) | (has_slot.astype(np.int64) << 15)
                  | ((np.where(spill_flag, spill_of_pos, 0) & 0x7FFF) << 16) | (spill_flag.astype(np.int64) << 31))
    self.group_off, self.chunk_off, self.spill_off = goff, coff, soff
    self.spill_list = pairs[:, 1] if len(pairs) else np.zeros(0, np.int64)
    self.n_groups, self.n_chunks = n_groups, n_chunks
    self.n_slots, self.n_long = nslots, int(spill_flag.sum())
    self.max_spill_reads = int(np.diff(soff).max(initial=0))
    # per-candidate shared region (doubles): [slots | stage 0 | stage 1], stage = start K | finish K | spill R;
    # successor entries become absolute indices into it (the reader's chunk parity picks the stage)
    self.slot_region = (max(nslots, 1) + 1) // 2 * 2
    self.stage_doubles = (2 * self.chunk + self.max_spill_reads + 1) // 2 * 2
    reader_chunk = chunk_of_pos[pu]
    absent = np.where(near, slot_of_pos[pv], 0)
    if far.any():
        absent[far] = [self.slot_region + (c_ & 1) * self.stage_doubles + 2 * self.chunk + bufidx[(c_, k_)]
                       for c_, k_ in zip(far_chunk.tolist(), far_k.tolist())]
    del reader_chunk
    self.cp_succ_abs = absent[np.argsort(pu, kind="stable")]
    return self


def _graphs():
    rng = np.random.default_rng(7)
    for seed in range(6):
        yield f"rand{seed}", W.random_dag(int(rng.integers(5, 300)), float(rng.uniform(0.02, 0.3)), seed=seed, num_devices=int(rng.integers(1, 9)))
    import bench
    from paper_2002_06790_b200.ps import expand_parameter_server

    graphs, db, configs, _ = bench.build_workload(0, 64, "resnet50-dp8")
    yield "resnet50-dp8", O.expand(graphs[0], configs[0])[0]
    graphs, db, configs, graph_of = bench.build_workload(0, 2048, "bert-large-ps-ar")
    seen = set()
    for cfg, gi in zip(configs, graph_of):
        key = (cfg.sync, cfg.replicas)
        if key in seen:
            continue
        seen.add(key)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            gx = (expand_parameter_server(graphs[gi], cfg, db, cfg.ps_device).graph if cfg.sync == "parameter_server"
                  else O.expand(graphs[gi], cfg)[0])
        yield f"bert-{key}", gx


@pytest.mark.parametrize("name, g", list(_graphs()))
def test_planners_equal_numpy(name, g):
    c = host_csr(g)
    n = len(c["ids"])
    off, idx, indeg = (np.asarray(c[k], np.int64) for k in ("succ_off", "succ_idx", "indeg"))
    want = np_level_order(n, off, idx, indeg)
    got = prepare.level_order(n, off, idx, indeg)
    assert (want is None) == (got is None)
    if want is None:
        return
    for a, b in zip(want, got):
        assert np.array_equal(a, b), name
    order, _, loff = want
    pos = np.empty(n, np.int64)
    pos[order] = np.arange(n)
    outdeg = np.diff(off)
    ref = np_cp_plan(prepare.GROUP, prepare.CHUNK, n, idx, indeg, outdeg, order, pos, loff)
    t = prepare.Tables(n, 1, off, idx, indeg, np.zeros(n, np.int64), levels=False)
    t._critical_path(n, idx, indeg, outdeg, order, pos, loff)
    for k in ("cp_meta", "cp_slot", "cp_spill", "cp_succ", "cp_succ_abs", "pinfo", "group_off", "chunk_off",
              "spill_off", "spill_list"):
        assert np.array_equal(np.asarray(getattr(ref, k), np.int64), np.asarray(getattr(t, k), np.int64)), (name, k)
    for k in ("n_groups", "n_chunks", "n_slots", "n_long", "max_spill_reads", "slot_region", "stage_doubles"):
        assert getattr(ref, k) == getattr(t, k), (name, k)


def test_level_order_cycle():
    off = np.array([0, 1, 2, 2]); idx = np.array([1, 0]); indeg = np.array([1, 1, 0])
    assert prepare.level_order(3, off, idx, indeg) is None
