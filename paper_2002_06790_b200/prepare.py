"""Per-topology-class tables for the fused engine (K3 v2) and the level-order
critical path (K4 v2).  Host numpy, once per class.

* level order: Kahn waves (level = longest edge count from a source); the
  output position of a node is its index in this order, so the critical-path
  pass reads each schedule row contiguously, level by level, backwards.
* engine tables: ``meta[v]`` = successor begin (24 bits) | out-degree (8 bits,
  255 = read succ_off), ``succ[j]`` = consumer rank | device << 16 | single-input
  << 21 (a consumer with exactly one input reference needs no counter),
  ``cidx[v]`` = counter slot of multi-input nodes, packed initial counters.
* critical-path tables: for each position its suffix slot and its successors'
  slots.  Slots are allocated by interval colouring over the reverse level
  order: a node's suffix lives from its own level until its last predecessor's
  level (graph.py:463-469 reads suffix only through successor lists).
"""

from __future__ import annotations

import numpy as np

from . import native


def level_order(n: int, succ_off: np.ndarray, succ_idx: np.ndarray, indeg: np.ndarray):
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
        idx = np.repeat(ends - cnt.cumsum(), cnt) + np.arange(cnt.sum())
        targets = succ_idx[idx]
        np.subtract.at(left, targets, 1)
        cand = np.unique(targets)
        frontier = cand[left[cand] == 0]
        lv += 1
    order = np.concatenate(order) if order else np.zeros(0, np.int64)
    if order.size != n:
        return None
    return order, level, np.asarray(offsets, dtype=np.int64)


class ClassTables:
    """Device-resident engine + critical-path tables of one topology class."""

    GROUP = 32        # positions processed together (one per lane)
    CHUNK = 64        # positions prefetched per cp.async batch
    QCAP = 32         # per-device FIFO ring capacity of the fused engine

    def __init__(self, lg, host=None):
        self.ctx = lg.ctx
        if host is None:
            host = dict(succ_off=lg.t_succ_off[: lg.n + 1].cpu().numpy(),
                        succ_idx=lg.t_succ_idx[: lg.n_edges].cpu().numpy(),
                        indeg=lg.t_indeg[: lg.n].cpu().numpy(), device=lg.t_dev[: lg.n].cpu().numpy(),
                        sources=lg.t_sources[: lg.n_sources].cpu().numpy())
        N, D = lg.n, lg.n_devices
        off = np.asarray(host["succ_off"], np.int64)
        idx = np.asarray(host["succ_idx"], np.int64)
        indeg = np.asarray(host["indeg"], np.int64)
        dev = np.asarray(host["device"], np.int64)
        self.n, self.n_devices, self.n_edges = N, D, int(off[-1]) if N else 0
        lo = level_order(N, off, idx, indeg)
        self.acyclic = lo is not None
        outdeg = np.diff(off)
        self.fused_ok = (self.acyclic and 0 < N <= 65535 and D <= 32 and self.n_edges < (1 << 24)
                         and indeg.max(initial=0) <= 65534)
        if not self.acyclic:
            self.fused_ok = False
            return
        order, level, loff = lo
        pos = np.empty(N, np.int64)
        pos[order] = np.arange(N)
        self.pos, self.rank_of_pos, self.level_off = pos, order, loff
        # ---- engine tables (rank space)
        single = indeg == 1
        multi = np.nonzero(indeg >= 2)[0]
        cidx = np.zeros(N, np.int64)
        cidx[multi] = np.arange(multi.size)
        bits = 8 if indeg.max(initial=0) < 255 else 16
        per = 32 // bits
        words = max(1, -(-multi.size // per))
        init = np.zeros(words * per, np.uint64)
        init[: multi.size] = indeg[multi]
        init = init.reshape(words, per)
        packed = np.zeros(words, np.uint64)
        for i in range(per):
            packed |= init[:, i] << np.uint64(i * bits)
        meta = (off[:-1] & 0xFFFFFF) | (np.minimum(outdeg, 255) << 24)
        succ = idx | (dev[idx] << 16) | (single[idx].astype(np.int64) << 21)
        self.counter_bits, self.counter_words = bits, words
        # ---- critical-path tables (position space)
        n_lv = loff.size - 1
        pred_last = np.full(N, -1, np.int64)   # last reading level in reverse order (by rank)
        rlevel = (n_lv - 1) - level            # processing index of each node's level
        src_of_edge = np.repeat(np.arange(N), outdeg)
        np.maximum.at(pred_last, idx, rlevel[src_of_edge])
        release = np.where(pred_last >= 0, pred_last, rlevel)  # sources: only read by the final max
        slot = np.empty(N, np.int64)
        free, nslots = [], 0
        # interval colouring: process reverse levels, free slots released before this level
        by_release = {}
        for r in range(n_lv):
            lv = n_lv - 1 - r
            for s in by_release.pop(r - 1, ()):
                free.append(s)
            nodes = order[loff[lv]:loff[lv + 1]]
            for v in nodes.tolist():
                if free:
                    s = free.pop()
                else:
                    s, nslots = nslots, nslots + 1
                slot[v] = s
                by_release.setdefault(int(release[v]), []).append(s)
        self.n_slots = nslots
        self.fused_ok = self.fused_ok and nslots < 65536 and self.n_edges < 65536 and outdeg.max(initial=0) < 256
        cp_off = np.zeros(N + 1, np.int64)
        cp_off[1:] = np.cumsum(outdeg[order])
        cp_succ = slot[idx[np.concatenate([np.arange(off[v], off[v + 1]) for v in order.tolist()])
                       if self.n_edges else np.zeros(0, np.int64)]]
        # groups: <= GROUP positions inside one level; chunks: consecutive groups <= CHUNK positions
        goff = [0]
        for lv in range(n_lv):
            a, b = int(loff[lv]), int(loff[lv + 1])
            for p in range(a, b, self.GROUP):
                goff.append(min(b, p + self.GROUP))
        goff = np.asarray(goff, np.int64)
        coff = [0]
        start = 0
        for gi in range(1, goff.size):
            if goff[gi] - goff[start] > self.CHUNK:
                coff.append(gi - 1)
                start = gi - 1
        if coff[-1] != goff.size - 1:
            coff.append(goff.size - 1)
        coff = np.asarray(coff, np.int64)
        self.n_groups, self.n_chunks = goff.size - 1, coff.size - 1
        src_flag = (indeg[order] == 0).astype(np.int64)
        cp_meta = (cp_off[:-1] & 0xFFFF) | (np.minimum(outdeg[order], 255) << 16) | (src_flag << 24)
        T = lambda a, dt: _t(a, dt, self.ctx.device)  # noqa: E731
        self.t = dict(meta=T(meta, np.uint32), succ_off=lg.t_succ_off, succ=T(succ, np.uint32),
                      cidx=T(cidx, np.uint16), cnt_init=T(packed, np.uint32), pos=T(pos, np.uint16 if N <= 65535 else np.int32),
                      pos32=T(pos, np.int32),
                      sources=lg.t_sources, rank_of_pos=T(order, np.int32), cp_slot=T(slot[order], np.uint16 if nslots < 65536 else np.int32),
                      cp_meta=T(cp_meta, np.uint32), cp_succ=T(cp_succ, np.uint16 if nslots < 65536 else np.int32),
                      group_off=T(goff, np.int32), chunk_off=T(coff, np.int32))
        t = self.t
        p = native.ptr
        self.sim_struct = native.SimTables(N, D, self.n_edges, p(t["meta"]), p(t["succ_off"]), p(t["succ"]),
                                           p(t["cidx"]), p(t["cnt_init"]), words, bits, p(t["pos"]), p(t["sources"]),
                                           lg.n_sources, self.QCAP, p(lg.t_dev))
        self.cp_struct = native.CpTables(N, self.n_slots, self.n_edges, p(t["rank_of_pos"]), p(t["cp_meta"]),
                                         p(t["cp_slot"]), p(t["cp_succ"]), self.n_groups, p(t["group_off"]),
                                         self.n_chunks, p(t["chunk_off"]), self.CHUNK)

    def output_to_rank(self, arr_by_pos: np.ndarray) -> np.ndarray:
        """Schedule row(s) stored by position -> node-rank order."""
        return arr_by_pos[..., self.pos]


def _t(a, dt, device):
    import torch

    arr = np.ascontiguousarray(np.asarray(a).astype(dt, copy=False))
    if arr.size == 0:
        arr = np.zeros(1, dt)
    if arr.dtype == np.uint64:
        arr = arr.view(np.int64)
    if arr.dtype == np.uint32:
        arr = arr.view(np.int32)
    if arr.dtype == np.uint16:
        arr = arr.view(np.int16)
    return torch.from_numpy(arr).to(f"cuda:{device}")
