"""Per-topology-class tables for the fused engine (K3 v2) and the level-order
critical path (K4 v2).  Host numpy, once per class.

* level order: Kahn waves (level = longest edge count from a source); the
  output column of a node is its index in this order, so the critical-path
  pass reads each schedule row contiguously, level by level, backwards.
* engine tables: ``meta[v]`` = successor begin (24 bits) | out-degree (8 bits, < 255), ``succ[j]`` = consumer rank | device << 16 | single-input
  << 21 (a consumer with exactly one input reference needs no counter),
  ``cidx[v]`` = counter slot of multi-input nodes, packed 4/8/16-bit initial counters.
* critical-path tables: the reverse pass processes groups (<= GROUP positions of
  one level) inside prefetch chunks (<= CHUNK positions).  A suffix value read
  in its own chunk or the next one lives in a shared-memory slot (interval
  colouring over processing steps); one read two or more chunks later is also
  written to an L2-resident spill row and prefetched with the reader's chunk.
  ``cp_succ[j]`` names a slot, or (bit 15) an index into the chunk's spill list;
  ``pinfo[p]`` says where position p's own value goes (slot and/or spill row).
"""

from __future__ import annotations

import os

import numpy as np

from . import native
from .lowering import upload

GROUP = 16        # positions processed together (one per lane of a half-warp)
CHUNK = int(os.environ.get("DFSIM_CP_CHUNK", 32))  # positions prefetched per cp.async batch
QCAP = 16         # per-device FIFO ring capacity of the fused engine (overflow -> exact engine)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def level_order(n: int, succ_off: np.ndarray, succ_idx: np.ndarray, indeg: np.ndarray):
    """Kahn waves (dfsim_level_order, host C++): (order, level_of_rank, level_offsets) as int64
    arrays, or None on a cycle."""
    lib = native.load_library()
    off, idx, deg = _i32(succ_off), _i32(succ_idx if len(succ_idx) else np.zeros(1)), _i32(indeg)
    order, level, loff = (np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32),
                          np.zeros(n + 1, np.int32))
    pp = lambda a: a.ctypes.data_as(native.P)  # noqa: E731
    nl = lib.dfsim_level_order(n, pp(off), pp(idx), pp(deg), pp(order), pp(level), pp(loff))
    if nl == -2:
        raise ValueError("level_order: bad graph arrays")
    if nl < 0:
        return None
    return order[:n].astype(np.int64), level[:n].astype(np.int64), loff[: nl + 1].astype(np.int64)


class Tables:
    """Host arrays + statistics of one class (see module docstring)."""

    def __init__(self, N: int, D: int, succ_off, succ_idx, indeg, device, group: int = GROUP,
                 chunk: int = CHUNK, levels: bool = True):
        off = np.asarray(succ_off, np.int64)
        idx = np.asarray(succ_idx, np.int64)
        indeg = np.asarray(indeg, np.int64)
        dev = np.asarray(device, np.int64)
        self.n, self.n_devices, self.n_edges = N, D, int(off[-1]) if N else 0
        self.group, self.chunk = group, chunk
        outdeg = np.diff(off)
        lo = level_order(N, off, idx, indeg)
        self.acyclic = lo is not None
        self.fused_ok = False
        if not self.acyclic or N == 0:
            return
        order, level, loff = lo
        pos = np.empty(N, np.int64)
        pos[order] = np.arange(N)
        self.pos, self.rank_of_pos, self.level_off = pos, order, loff
        self._engine(N, off, idx, indeg, dev, outdeg)
        self._cp_args = (N, idx, indeg, outdeg, order, pos, loff)
        self.levels_built = False
        # engine limits; the critical path adds its own (K4 v3 planner or K4 v2 tables below)
        self.fused_ok = (N <= 65535 and D <= 32 and self.n_edges < 65536 and outdeg.max(initial=0) < 255
                         and self.counter_words <= 512 and indeg.max(initial=0) <= 65534)
        if levels:
            self.fused_ok = self.fused_ok and self.build_levels()

    def build_levels(self) -> bool:
        """K4 v2 tables (only needed when K4 v3's plan is unavailable); True when they fit."""
        if not self.levels_built:
            self._critical_path(*self._cp_args)
            self.levels_built = True
        return (self.n_slots < 0x7FFF and self.max_spill_reads < 0x7FFF and self.n_long < 0x7FFF
                and self.slot_region + 2 * self.stage_doubles < 65536 and len(self.spill_list) < 65536)

    def _engine(self, N, off, idx, indeg, dev, outdeg):
        """K3 v2 tables with nodes numbered by level position p (pos[rank]); ranks survive only
        as ``rank[p]`` for the FIFO tie-break sort, override lookups and the source order."""
        order, pos = self.rank_of_pos, self.pos
        single = indeg == 1
        # dependency counters of multi-input nodes, each as narrow as its in-degree allows
        # (2, 4, 8 or 16 bits); every width class starts on a fresh 32-bit word so no field
        # straddles a word.  code = word << 7 | shift << 2 | log2(width) - 1
        deg_p = indeg[order]
        multi_p = np.nonzero(deg_p >= 2)[0]
        wcode = np.select([deg_p <= 3, deg_p <= 15, deg_p <= 255], [0, 1, 2], 3)
        code = np.zeros(N, np.int64)
        words, init_words = 0, []
        for wc in range(4):
            sel = multi_p[wcode[multi_p] == wc]
            if sel.size == 0:
                continue
            width = 2 << wc
            per = 32 // width
            k = np.arange(sel.size)
            word, shift = words + k // per, (k % per) * width
            code[sel] = (word << 7) | (shift << 2) | wc
            fill = np.zeros(-(-sel.size // per) * per, np.uint64)
            fill[: sel.size] = deg_p[sel]
            fill = fill.reshape(-1, per)
            packed_w = np.zeros(fill.shape[0], np.uint64)
            for i in range(per):
                packed_w |= fill[:, i] << np.uint64(i * width)
            init_words.append(packed_w)
            words += fill.shape[0]
        packed = np.concatenate(init_words) if init_words else np.zeros(1, np.uint64)
        self.counter_bits = int(2 << int(wcode[multi_p].max())) if multi_p.size else 2
        self.counter_words = max(1, words)
        # successor CSR by position: the successors of the node at position p, in its rank-CSR order
        outdeg_p = outdeg[order]
        off_p = np.zeros(N + 1, np.int64)
        np.cumsum(outdeg_p, out=off_p[1:])
        take = np.arange(int(off_p[-1]), dtype=np.int64) + np.repeat(off[order] - off_p[:-1], outdeg_p)
        cons = idx[take]                                         # consumer ranks
        cpos = pos[cons]
        self.succ_off_pos, self.succ_pos = off_p, cpos           # successor positions by position
        self.meta = (off_p[:-1] & 0xFFFFFF) | (np.minimum(outdeg_p, 255) << 24)
        # packed entry: consumer position 13 | device 4 | single 1 | wide 1 | shift 5 | word 8
        self.succ_packed = (N <= 8192 and int(dev.max(initial=0)) < 16 and self.counter_bits <= 4
                            and self.counter_words <= 256)
        if self.succ_packed:
            cc = code[cpos]
            self.succ = (cpos | (dev[cons] << 13) | (single[cons].astype(np.int64) << 17) | ((cc & 3) << 18)
                         | (((cc >> 2) & 31) << 19) | ((cc >> 7) << 24))
        else:  # consumer position 16 | device 5 | single 1; the counter code comes from cidx[]
            self.succ = cpos | (dev[cons] << 16) | (single[cons].astype(np.int64) << 21)
        self.cidx, self.cnt_init = code, packed
        self.indeg_pos = deg_p
        self.eng_sources = pos[np.nonzero(indeg == 0)[0]]        # ascending ranks, as positions

    def _critical_path(self, N, idx, indeg, outdeg, order, pos, loff):
        """K4 v2 tables (dfsim_cp_levels_plan, host C++; layout in the module docstring)."""
        lib = native.load_library()
        E = int(outdeg.sum())
        off = np.zeros(N + 1, np.int32)
        np.cumsum(outdeg, out=off[1:])
        z = lambda k, dt=np.int32: np.zeros(max(k, 1), dt)  # noqa: E731
        goff, coff, soff = z(N + 1), z(N + 1), z(N + 1)
        slot, spill, meta, pinfo = z(N), z(N), z(N, np.uint32), z(N, np.uint32)
        slist, succ, succ_abs, info = z(E), z(E), z(E), z(8)
        pp = lambda a: a.ctypes.data_as(native.P)  # noqa: E731
        rc = lib.dfsim_cp_levels_plan(N, pp(off), pp(_i32(idx) if E else z(1)), pp(_i32(indeg)), pp(_i32(order)),
                                      pp(_i32(loff)), len(loff) - 1, self.group, self.chunk, pp(goff), pp(coff),
                                      pp(slot), pp(spill), pp(soff), pp(slist), pp(succ), pp(succ_abs), pp(meta),
                                      pp(pinfo), pp(info))
        if rc != 0:
            raise ValueError(f"dfsim_cp_levels_plan failed ({rc})")
        ng, nc, nslots, n_long, max_reads, nl, region, stage = (int(x) for x in info)
        self.cp_meta, self.cp_slot, self.cp_spill = meta[:N].astype(np.int64), slot[:N], spill[:N]
        self.cp_succ, self.cp_succ_abs, self.pinfo = succ[:E], succ_abs[:E], pinfo[:N].astype(np.int64)
        self.group_off, self.chunk_off, self.spill_off = goff[: ng + 1], coff[: nc + 1], soff[: nc + 1]
        self.spill_list = slist[:nl]
        self.n_groups, self.n_chunks = ng, nc
        self.n_slots, self.n_long, self.max_spill_reads = nslots, n_long, max_reads
        self.slot_region, self.stage_doubles = region, stage


LANE_K = 8  # positions per K4 v3 chunk (its register window)
LANE_RMAX = int(os.environ.get("DFSIM_CP_LANE_RMAX", 8))  # spill values per chunk (planner minimum)
LANE_STAGES = 0  # K4 v3 launch variant: register windows (the planner models 2 smem stages)


LANE_NEAR = int(os.environ.get("DFSIM_CP_LANE_NEAR", 12))  # chunks a value may wait in a slot (C2: 8 -> 12, CP 1.290 -> 1.280 ms; 14 drops a warp)
LANE_MIN_SIMS = int(os.environ.get("DFSIM_CP_LANES_MIN", 16384))  # candidates a class needs for K4 v3


def lane_plan(t: Tables, K: int = LANE_K, rmax_min: int = LANE_RMAX, stages: int = LANE_STAGES,
              near: int = LANE_NEAR):
    """K4 v3 tables of a class (dfsim_cp_lanes_plan, host C++): dict of numpy arrays + sizes,
    or None when a field overflows (the class then keeps K4 v2)."""
    import ctypes

    lib = native.load_library()
    N, E = t.n, t.n_edges
    off = np.ascontiguousarray(t.succ_off_pos, np.int32)
    sp = np.ascontiguousarray(t.succ_pos if E else np.zeros(1), np.int32)
    src = np.ascontiguousarray(t.indeg_pos == 0, np.uint8)
    blocks = np.zeros(4 * (2 * N + E // 8 + 2), np.uint32)
    boff = np.zeros(N + 1, np.int32)
    bounds = np.zeros(N + 1, np.int32)
    soff = np.zeros(N + 1, np.int32)
    slist = np.zeros(max(E, 1), np.uint16)
    info = np.zeros(6, np.int32)
    pp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    if stages == 0:
        K = 8  # the register variant's window size
    rc = lib.dfsim_cp_lanes_plan(N, pp(off), pp(sp), pp(src), K, rmax_min, stages or 2, near, pp(blocks), pp(boff),
                                 pp(bounds), pp(soff), pp(slist), pp(info))
    if rc != 0:
        return None
    nq, ns, rmax, n_long, nl, bmax = (int(x) for x in info)
    return dict(K=K, stages=stages, smem_stages=stages or 2, n_chunks=nq, n_slots=ns, rmax=rmax, n_long=n_long, n_spill_list=nl,
                block_max=bmax, blocks=blocks[: 4 * int(boff[nq])], block_off=boff[: nq + 1], bounds=bounds[: nq + 1],
                spill_off=soff[: nq + 1], spill_list=slist[:nl])


class ClassTables(Tables):
    """Tables uploaded to the device, with the C-ABI structs of K3 v2 and K4 v2."""

    GROUP, CHUNK, QCAP = GROUP, CHUNK, QCAP

    def __init__(self, lg, host=None, n_sims: int | None = None):
        self.ctx = lg.ctx
        if host is None:
            host = dict(succ_off=lg.t_succ_off[: lg.n + 1].cpu().numpy(),
                        succ_idx=lg.t_succ_idx[: lg.n_edges].cpu().numpy(),
                        indeg=lg.t_indeg[: lg.n].cpu().numpy(), device=lg.t_dev[: lg.n].cpu().numpy())
        super().__init__(lg.n, lg.n_devices, host["succ_off"], host["succ_idx"], host["indeg"], host["device"],
                         self.GROUP, self.CHUNK, levels=False)
        self.lane = self.cp_struct = None
        if not self.fused_ok:
            return
        d = self.ctx.device
        p = native.ptr
        tabs = dict(meta=(self.meta, np.uint32), succ=(self.succ, np.uint32), cidx=(self.cidx, np.uint16),
                    cnt_init=(self.cnt_init, np.uint32), rank16=(self.rank_of_pos, np.uint16),
                    eng_sources=(self.eng_sources, np.int32), pos32=(self.pos, np.int32),
                    rank_of_pos=(self.rank_of_pos, np.int32))
        # K4 v3 (lane per candidate) when its plan fits, else K4 v2 (level groups).
        # K4 v3 walks all N positions one after another per warp, so its latency is N steps: it
        # pays off once a class has enough candidates to keep every SM busy meanwhile
        # (measured on C2, 65,536: 1.99 ms vs 2.31 ms for K4 v2; C3 / C4 classes of ~200-900
        # candidates are faster on K4 v2's level groups)
        enough = n_sims is None or n_sims >= LANE_MIN_SIMS
        plan = lane_plan(self) if os.environ.get("DFSIM_CP_KERNEL", "lanes") == "lanes" and enough else None
        if plan is not None:
            tabs.update(l_blocks=(plan["blocks"], np.uint32), l_boff=(plan["block_off"], np.int32),
                        l_bounds=(plan["bounds"], np.int32), l_soff=(plan["spill_off"], np.int32),
                        l_slist=(plan["spill_list"], np.uint16))
        levels_ok = plan is not None or self.build_levels()
        if plan is None and levels_ok:
            tabs.update(cp_slot=(self.cp_slot, np.uint16), cp_spill=(self.cp_spill, np.uint16),
                        cp_meta=(self.cp_meta, np.uint32), cp_succ=(self.cp_succ_abs, np.uint16),
                        group_off=(self.group_off, np.int32), chunk_off=(self.chunk_off, np.int32),
                        spill_off=(self.spill_off, np.int32), spill_list=(self.spill_list, np.uint16),
                        pinfo=(self.pinfo, np.uint32))
        self.t = t = upload(tabs, d)  # one host-to-device copy for the class's tables
        self.sim_struct = native.SimTables(lg.n, lg.n_devices, self.n_edges, p(t["meta"]), p(lg.t_succ_off),
                                           p(t["succ"]), p(t["cidx"]), p(t["cnt_init"]), self.counter_words,
                                           self.counter_bits, p(t["rank16"]), p(t["eng_sources"]), lg.n_sources,
                                           self.QCAP,
                                           p(lg.t_dev), int(self.succ_packed))
        if plan is not None:
            st = native.CpLaneTables(lg.n, plan["n_chunks"], plan["K"], plan["n_slots"], plan["rmax"],
                                     plan["n_long"], plan["n_spill_list"], plan["block_max"], p(t["l_blocks"]),
                                     p(t["l_boff"]), p(t["l_bounds"]), p(t["l_soff"]), p(t["l_slist"]),
                                     p(t["rank_of_pos"]))
            if self.ctx.lib.dfsim_critical_path_lanes_capacity(native.ctypes.byref(st), plan["stages"]) > 0:
                self.lane, self.lane_struct = plan, st
        if self.lane is None:
            if not levels_ok or "cp_meta" not in t:
                if not self.build_levels():
                    self.fused_ok = False
                    return
                t.update(upload(dict(
                    cp_slot=(self.cp_slot, np.uint16), cp_spill=(self.cp_spill, np.uint16),
                    cp_meta=(self.cp_meta, np.uint32), cp_succ=(self.cp_succ_abs, np.uint16),
                    group_off=(self.group_off, np.int32), chunk_off=(self.chunk_off, np.int32),
                    spill_off=(self.spill_off, np.int32), spill_list=(self.spill_list, np.uint16),
                    pinfo=(self.pinfo, np.uint32)), d))
            self.cp_struct = native.CpTables(lg.n, self.n_slots, self.n_edges, p(t["rank_of_pos"]), p(t["cp_meta"]),
                                             p(t["cp_slot"]), p(t["cp_succ"]), self.n_groups, p(t["group_off"]),
                                             self.n_chunks, p(t["chunk_off"]), self.CHUNK, self.n_long,
                                             p(t["cp_spill"]), p(t["spill_off"]), p(t["spill_list"]),
                                             self.max_spill_reads, p(t["pinfo"]), self.slot_region,
                                             self.stage_doubles)

    def critical_path(self, n_sims: int, sched, cp_len, cp_src, cand_of_slot, slots=None):
        """K4 over the fused engine's tiled schedules: v3 (lane per candidate) when planned, else
        v2; slot k holds candidate ``cand_of_slot[k]`` (device int64: the engine's order).
        ``slots``: only these schedule slots (K4 v3's register variant takes a slot list)."""
        c = native.ptr(cand_of_slot) if cand_of_slot is not None else native.P(0)
        if self.lane is not None and slots is not None and len(slots) and self.lane["stages"] == 0:
            import torch

            sl = torch.as_tensor(sorted(set(int(x) for x in slots)), dtype=torch.int64,
                                 device=f"cuda:{self.ctx.device}")
            self.ctx.call("dfsim_critical_path_lanes_ex", native.ctypes.byref(self.lane_struct), 0, sl.numel(),
                          native.ptr(sl), c, 0, native.ptr(sched), native.ptr(cp_len), native.ptr(cp_src))
            return
        if self.lane is not None:
            self.ctx.call("dfsim_critical_path_lanes", native.ctypes.byref(self.lane_struct), self.lane["stages"],
                          n_sims, c, native.ptr(sched), native.ptr(cp_len), native.ptr(cp_src))
        else:
            self.ctx.call("dfsim_critical_path_levels", native.ctypes.byref(self.cp_struct), n_sims, c,
                          native.ptr(sched), native.ptr(cp_len), native.ptr(cp_src))

    def output_to_rank(self, arr_by_pos: np.ndarray) -> np.ndarray:
        """Schedule row(s) stored by position -> node-rank order."""
        return arr_by_pos[..., self.pos]
