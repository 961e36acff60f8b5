// K2a + K3 v2 + K4 v2: the fused per-candidate hot path.
//
// K2a dfsim_resolve_variants: estimate_all's fallback chain (costmodel.py:282-331)
//     evaluated once per (variant = hardware tag x collective algorithm, node) with
//     op_gap 0; the sign bit of the stored value marks "add op_gap" (Compute nodes
//     resolved from an exact record or a fitted model, costmodel.py:305-320).
// K3 v2 dfsim_simulate_fused: engine.py:96-146 per candidate with durations
//     formed on the fly: dur = override (302-304) | base + op_gap | base.
//     One CTA per SM holds the class graph and the staged duration row of the
//     variant it is working on in shared memory; each warp simulates one candidate
//     (lane d = device rank d) from ~3 KB of shared state: compact 8/16-bit
//     dependency counters for multi-input nodes and one 32-entry FIFO ring per
//     device.  A ring overflow aborts the candidate and flags it for the exact
//     engine (dfsim_simulate_batch_ex), so results never depend on the ring size.
// K4 v2 dfsim_critical_path_levels: graph.py:446-474 on finish-start, warp per
//     candidate, reverse level order; suffix values live in statically allocated
//     shared-memory slots, schedule rows (stored by level position) are prefetched
//     with cp.async one chunk ahead.
#include <cuda_runtime.h>

#include "group.cuh"
#include "internal.cuh"

namespace {

// ------------------------------------------------------------------ K3 v2

struct FusedArgs {
    dfsim_sim_tables g;
    dfsim_fused_strategies st;
    double *sched, *makespan, *busy;  // sched[s][pos] = (start, finish) pairs
    int32_t *n_placed, *flags;
    int32_t *chunk_counter;
    int32_t wpb;
    int32_t smem_graph;  // bytes of the CTA-shared part
    int32_t smem_warp;   // bytes per candidate group
    int32_t tail_bytes;  // FIFO tails at the start of each group's state
};

// Decrement the counter field (width mask at bit `shift` of cnt[word]); true when it reaches zero.
__device__ __forceinline__ bool counter_dec(unsigned *cnt, unsigned word, unsigned shift, unsigned mask,
                                            unsigned n_words) {
    DFSIM_CHECK(word < n_words && shift < 32u, 2);
    const unsigned old = atomicSub(cnt + word, 1u << shift);
    return ((old >> shift) & mask) == 1u;
}

// Read-only CTA tables through 32-bit shared-window addresses computed once: with generic
// pointers the compiler re-derives each table's base (S2R SR_CgaCtaId + LEA) inside the loop.
__device__ __forceinline__ unsigned smem_addr(const void *p) {
    unsigned r;  // opaque to the compiler, so the value stays in a register instead of being re-derived
    asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t lds_u32(unsigned a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_u16(unsigned a) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

constexpr int kWide = 4;  // out-degree above which a finished node's successors are spread over the group

// Successor entry formats: kPacked: consumer (13 bits) | device << 13 (4) | single << 17 | wide << 18 |
// shift << 19 | word << 24; otherwise consumer (16) | device << 16 | single << 21 with the counter
// code (word << 7 | shift << 2 | log2(width) - 1) in cidx[] in smem.
// kBaseG: the variant's duration row is read from global memory (L1/L2: all candidates of a
// chunk share it) instead of being staged in smem -- for classes whose smem tables would
// otherwise leave room for only a few candidates per CTA.
template <int kGS, bool kPacked, bool kBaseG, bool kTiled>
__global__ void __launch_bounds__(1024, 1) k_simulate_fused(FusedArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int kPerWarp = 32 / kGS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int ll, grp;  // opaque copies: otherwise lane % 10 and lane / 10 are re-derived at every use
    asm volatile("mov.u32 %0, %1;" : "=r"(ll) : "r"(lane % kGS));
    asm volatile("mov.u32 %0, %1;" : "=r"(grp) : "r"(lane / kGS));
    const int gid = warp * kPerWarp + grp;  // candidate slot of this lane group inside a chunk
    const bool in_group = grp < kPerWarp;   // kGS = 10: lanes 30-31 belong to no candidate
    const int N = a.g.n_nodes, D = a.g.n_devices;
    const int E = static_cast<int>(a.g.n_edges);
    const int QCAP = a.g.qcap;
    const int QSTRIDE = QCAP + 2;  // u16 entries: 17-word stride keeps the 16 lanes' rings on distinct banks
    const unsigned QMASK = static_cast<unsigned>(QCAP - 1);
    const unsigned n_cw = static_cast<unsigned>(a.g.n_counter_words);  // checked builds only
    (void)n_cw;

    // CTA-shared tables
    uint32_t *s_meta = reinterpret_cast<uint32_t *>(smem);
    uint32_t *s_succ = s_meta + N;
    uint16_t *s_rank = reinterpret_cast<uint16_t *>(s_succ + E);  // nodes are numbered by position; rank only for tie-breaks
    uint16_t *s_cidx = s_rank + N;                                // counter codes (unpacked format only)
    double *s_base = reinterpret_cast<double *>(
        smem + ((static_cast<size_t>(N) * (kPacked ? 6 : 8) + static_cast<size_t>(E) * 4 + 15) / 16) * 16);
    // idle lanes (kGS = 10) alias their warp's first group for reads; they never write
    unsigned char *gbase = smem + a.smem_graph + static_cast<size_t>(in_group ? gid : warp * kPerWarp) * a.smem_warp;
    int32_t *tails = reinterpret_cast<int32_t *>(gbase);
    unsigned *cnt = reinterpret_cast<unsigned *>(gbase + a.tail_bytes);
    uint16_t *q = reinterpret_cast<uint16_t *>(gbase + a.tail_bytes + a.g.n_counter_words * 4);
    __shared__ int s_chunk;
    const unsigned a_meta = smem_addr(s_meta), a_succ = smem_addr(s_succ), a_cidx = smem_addr(s_cidx);
    const unsigned a_rank = smem_addr(s_rank), a_base = smem_addr(s_base);

    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        s_meta[i] = __ldg(a.g.meta + i);
        if (!kPacked) s_cidx[i] = __ldg(a.g.cidx + i);
        s_rank[i] = __ldg(a.g.rank + i);
    }
    for (int i = threadIdx.x; i < E; i += blockDim.x) s_succ[i] = __ldg(a.g.succ + i);
    int staged = -1;
    const double *g_row = a.st.base;

    for (;;) {
        if (threadIdx.x == 0) s_chunk = atomicAdd(a.chunk_counter, 1);
        __syncthreads();
        const int c = s_chunk;
        if (c >= a.st.n_chunks) break;
        const int var = __ldg(a.st.chunk_variant + c);
        if (var != staged) {
            const double *row = a.st.base + static_cast<int64_t>(var) * N;
            g_row = row;
            if (!kBaseG) {
                for (int i = threadIdx.x; i < N; i += blockDim.x) s_base[i] = __ldg(row + s_rank[i]);
                __syncthreads();
            }
            staged = var;
        }
        const bool active = in_group && gid < __ldg(a.st.chunk_count + c);
        if (__any_sync(DFSIM_FULL_MASK, active)) {
            const int64_t s = active ? __ldg(a.st.order + __ldg(a.st.chunk_first + c) + gid) : 0;
            const double gap = active ? __ldg(a.st.op_gap + s) : 0.0;
            const int ovs = (active && a.st.override_set) ? __ldg(a.st.override_set + s) : -1;
            // tiled schedule (dfsim_b200.h): slot k = the candidate's position in the engine's
            // order (candidates of one chunk are neighbours), pair ((k / 32) N + v) 32 + k % 32;
            // row layout: pair s N + v
            const int64_t k_slot = active ? static_cast<int64_t>(__ldg(a.st.chunk_first + c)) + gid : 0;
            double2 *out = reinterpret_cast<double2 *>(a.sched) + (kTiled ? (k_slot >> 5) * N * 32 + (k_slot & 31) : s * N);
            constexpr int ostride = kTiled ? 32 : 1;
            asm volatile("mov.b64 %0, %0;" : "+l"(out));  // keep the row base in a register (no per-pop s * N)
            if (active) {
                for (int w = ll; w < a.g.n_counter_words; w += kGS) cnt[w] = __ldg(a.g.cnt_init + w);
                if (ll < D) tails[ll] = 0;
            }
            unsigned head = 0;
            bool flag = false;
            __syncwarp();
            for (int b = 0; b < a.g.n_sources; b += kGS) {  // sources in rank order (engine.py:111-114)
                const int i = b + ll;
                const bool has = active && i < a.g.n_sources;
                const int v = has ? __ldg(a.g.sources + i) : 0;
                DFSIM_CHECK(v >= 0 && v < N, 3);
                const int dv = has ? __ldg(a.g.device + s_rank[v]) : 0;
                DFSIM_CHECK(dv >= 0 && dv < D, 1);
                const unsigned peers = __match_any_sync(DFSIM_FULL_MASK, has ? dv + 32 * grp : 1024 + lane);
                const int base = has ? tails[dv] : 0;
                __syncwarp();
                if (has) {
                    const int p = base + __popc(peers & lanemask_lt());
                    q[dv * QSTRIDE + (p & QMASK)] = static_cast<uint16_t>(v);
                    if ((peers & lanemask_lt()) == 0) tails[dv] = base + __popc(peers);
                }
                __syncwarp();
            }
            flag = group_any<kGS>(active && ll < D && static_cast<unsigned>(tails[ll]) - head > static_cast<unsigned>(QCAP), grp);

            bool running = false, ovf = false;
            const bool owner = active && !flag && ll < D;  // this lane drives device ll of a live candidate
            int run_v = 0;
            double run_f = 0.0, busy_sum = 0.0, span = 0.0, now = 0.0;
            auto start_idle = [&]() {
                const int t = owner ? tails[ll] : 0;
                if (owner && !running && !ovf && static_cast<int>(head) < t) {
                    // a busy device only gains entries until its next pop, so checking the
                    // occupancy before every pop catches every ring overflow; the device then
                    // stops for good (no overwritten entry is ever read, so the flagged candidate
                    // cannot corrupt its counters or loop) and the candidate is re-run exactly
                    ovf = static_cast<unsigned>(t) - head > static_cast<unsigned>(QCAP);
                    if (ovf) return;
                    const int v = q[ll * QSTRIDE + (head & QMASK)];
                    DFSIM_CHECK(v < N, 3);
                    head++;
                    const double b = kBaseG ? __ldg(g_row + lds_u16(a_rank + 2u * v)) : lds_f64(a_base + 8u * v);
                    double dur = signbit(b) ? __dadd_rn(-b, gap) : b;
                    const int vr = ovs >= 0 ? static_cast<int>(lds_u16(a_rank + 2u * v)) : 0;
                    if (ovs >= 0 && (!a.st.ov_any || ((__ldg(a.st.ov_any + (vr >> 5)) >> (vr & 31)) & 1u))) {
                        // override tables are by rank; nodes in no set skip the search
                        int lo = __ldg(a.st.ov_off + ovs), hi = __ldg(a.st.ov_off + ovs + 1);
                        const int end = hi;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (__ldg(a.st.ov_node + mid) < vr) lo = mid + 1; else hi = mid;
                        }
                        if (lo < end && __ldg(a.st.ov_node + lo) == vr) dur = __ldg(a.st.ov_val + lo);
                    }
                    const double f = __dadd_rn(now, dur);
                    out[ostride * v] = make_double2(now, f);
                    running = true;
                    run_v = v;
                    run_f = f;
                    busy_sum = __dadd_rn(busy_sum, __dsub_rn(f, now));
                    span = f;  // a device's finishes never decrease (dur >= 0 here): its last one is its max
                }
            };
            start_idle();
            while (__any_sync(DFSIM_FULL_MASK, running)) {
                now = group_min_nonneg<kGS>(running ? run_f : __longlong_as_double(0x7ff0000000000000LL), grp);
                const bool done = running && run_f == now;
                const int seg_lo = ll < D ? tails[ll] : 0;
                __syncwarp();
                // successors of the finished nodes (engine.py:136-142); a node with a wide
                // fan-out (e.g. an AllReduce feeding every replica) is spread over the group
                int j0 = 0, deg = 0;
                if (done) {
                    running = false;
                    DFSIM_CHECK(run_v >= 0 && run_v < N, 0);
                    const uint32_t meta = lds_u32(a_meta + 4u * run_v);
                    j0 = static_cast<int>(meta & 0xffffffu);
                    deg = static_cast<int>(meta >> 24);  // < 255 in the fused engine (prepare.Tables)
                    DFSIM_CHECK(j0 + deg <= E, 0);
                }
                auto relax = [&](int j) {
                    const uint32_t e = lds_u32(a_succ + 4u * j);
                    int m, dv;
                    bool ready;
                    if constexpr (kPacked) {
                        m = static_cast<int>(e & 0x1fffu);
                        dv = static_cast<int>((e >> 13) & 15u);
                        ready = ((e >> 17) & 1u) || counter_dec(cnt, e >> 24, (e >> 19) & 31u, (e >> 18) & 1u ? 15u : 3u, n_cw);
                    } else {
                        m = static_cast<int>(e & 0xffffu);
                        dv = static_cast<int>((e >> 16) & 31u);
                        if ((e >> 21) & 1u) {
                            ready = true;
                        } else {
                            const unsigned code = lds_u16(a_cidx + 2u * m);
                            ready = counter_dec(cnt, code >> 7, (code >> 2) & 31u, (1u << (2u << (code & 3u))) - 1u, n_cw);
                        }
                    }
                    DFSIM_CHECK(m >= 0 && m < N && dv >= 0 && dv < D, 1);
                    if (ready) {
                        const int p = atomicAdd(tails + dv, 1);
                        q[dv * QSTRIDE + (p & QMASK)] = static_cast<uint16_t>(m);
                    }
                };
                const bool wide = deg > kWide;
                if (!wide)
                    for (int j = j0; j < j0 + deg; j++) relax(j);
                const unsigned wm = __ballot_sync(DFSIM_FULL_MASK, wide);
                if (wm) {
                    unsigned mine = in_group ? group_bits<kGS>(wm, grp) : 0u;  // uniform in the group
                    while (__any_sync(DFSIM_FULL_MASK, mine != 0)) {
                        const bool have = mine != 0;
                        const int src = (have ? __ffs(mine) - 1 : 0) + grp * kGS;
                        if (have) mine &= mine - 1;
                        const int wj0 = __shfl_sync(DFSIM_FULL_MASK, j0, src);
                        const int wdeg = __shfl_sync(DFSIM_FULL_MASK, deg, src);
                        if (have)
                            for (int j = wj0 + ll; j < wj0 + wdeg; j += kGS) relax(j);
                    }
                }
                __syncwarp();
                const int seg_hi = ll < D ? tails[ll] : 0;
                // a ring overflow corrupts only this candidate; it keeps running (every
                // iteration consumes a finish event, so it terminates) and is re-run exactly
                // enqueue(sorted(newly_ready)): sort each device's new ring segment by rank
                if (in_group && seg_hi - seg_lo > 1) {  // idle lanes alias group 0: never write
                    uint16_t *qd = q + ll * QSTRIDE;
                    for (int i = seg_lo + 1; i < seg_hi; i++) {
                        const uint16_t x = qd[i & QMASK];
                        const unsigned xr = lds_u16(a_rank + 2u * x);
                        int j = i - 1;
                        while (j >= seg_lo && lds_u16(a_rank + 2u * qd[j & QMASK]) > xr) {
                            qd[(j + 1) & QMASK] = qd[j & QMASK];
                            j--;
                        }
                        qd[(j + 1) & QMASK] = x;
                    }
                }
                __syncwarp();
                start_idle();
            }
            // evaluated by every lane: a short-circuit here would leave the groups of a warp at
            // different warp-wide votes (a deadlock when only some groups are flagged)
            const bool any_ovf = group_any<kGS>(ovf, grp);
            flag = flag || any_ovf;
            const double ms = group_max_nonneg<kGS>(span, grp);
            const unsigned total = group_add_u32<kGS>(ll < D ? head : 0u, grp);  // every pop starts a node
            if (active && ll == 0) {
                a.makespan[s] = ms;
                a.n_placed[s] = flag ? -1 : static_cast<int>(total);
                a.flags[s] = flag ? 1 : 0;
            }
            if (active && a.busy && ll < D) a.busy[s * D + ll] = busy_sum;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K4 v2

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

struct CpLevelArgs {
    dfsim_cp_tables t;
    int64_t S;
    const int64_t *cand;  // optional: candidate of each schedule slot (outputs go to cp_len[cand[slot]])
    const double *sched;  // [S][N] (start, finish) pairs by level position
    double *cp_len;
    int32_t *cp_src;
    double *spill;        // [grid * wpb * 2][n_long] rows, one per resident candidate slot
    int32_t wpb;
    int32_t table_bytes;  // CTA-shared tables
};

__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

// Two candidates per warp: lanes 0-15 and 16-31 each walk the same class-wide
// reverse level order for their own candidate (identical control flow, different
// data).  Shared tables (by level position): pinfo[p] = slot | has-slot << 15 |
// spill index << 16 | spill << 31; pmeta[p] = successor begin | count << 16 |
// source << 24; succ[E] = index of the successor's value in the candidate's shared
// region [slots | stage 0 | stage 1] (a slot, or a value prefetched with the
// reader's chunk); group_off[G+1] (<= 16 positions of one level each), chunk
// offsets and the per-chunk spill lists.
__global__ void __launch_bounds__(1024, 1) k_critical_path_levels(CpLevelArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ll = lane & 15, half = lane >> 4;
    const int N = a.t.n_nodes, K = a.t.chunk_positions, G = a.t.n_groups, E = a.t.n_edges;
    const int NC = a.t.n_chunks, SD = a.t.stage_doubles, SR = a.t.slot_region;
    const int NS = __ldg(a.t.spill_off + NC);
    uint2 *s_pm = reinterpret_cast<uint2 *>(smem);  // per position: (cp_meta, pinfo)
    const unsigned a_pm = smem_addr(s_pm);
    uint16_t *s_succ = reinterpret_cast<uint16_t *>(s_pm + N);
    uint16_t *s_goff = s_succ + E;
    uint16_t *s_coff = s_goff + (G + 1);
    uint16_t *s_soff = s_coff + (NC + 1);
    uint16_t *s_slist = s_soff + (NC + 1);
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_pm[i] = make_uint2(__ldg(a.t.cp_meta + i), __ldg(a.t.pinfo + i));
    for (int i = threadIdx.x; i < E; i += blockDim.x) s_succ[i] = __ldg(a.t.cp_succ_slot + i);
    for (int i = threadIdx.x; i <= G; i += blockDim.x) s_goff[i] = static_cast<uint16_t>(__ldg(a.t.group_off + i));
    for (int i = threadIdx.x; i <= NC; i += blockDim.x) {
        s_coff[i] = static_cast<uint16_t>(__ldg(a.t.chunk_off + i));
        s_soff[i] = static_cast<uint16_t>(__ldg(a.t.spill_off + i));
    }
    for (int i = threadIdx.x; i < NS; i += blockDim.x) s_slist[i] = __ldg(a.t.spill_list + i);
    __syncthreads();
    const int gid = warp * 2 + half;  // candidate slot of this half-warp in the CTA
    double *region = reinterpret_cast<double *>(smem + a.table_bytes) + static_cast<size_t>(gid) * (SR + 2 * SD);
    double *spill_row = a.spill + (static_cast<int64_t>(blockIdx.x) * a.wpb * 2 + gid) * a.t.n_long;
    asm volatile("mov.b64 %0, %0;" : "+l"(spill_row));
    const int64_t per_iter = static_cast<int64_t>(gridDim.x) * a.wpb * 2;

    for (int64_t base = static_cast<int64_t>(blockIdx.x) * a.wpb * 2 + warp * 2; base < a.S; base += per_iter) {
        const int64_t s = base + half;
        const bool live = s < a.S;
        const int64_t sr = live ? s : base;  // the idle half shadows its partner's reads
        const double *row = a.sched + 2 * sr * N;  // row layout (classes on K4 v2)
        asm volatile("mov.b64 %0, %0;" : "+l"(row));  // keep row bases in registers (no 64-bit re-derivation)
        auto prefetch = [&](int c) {
            const int p0 = s_goff[s_coff[c]], p1 = s_goff[s_coff[c + 1]];
            double *bs = region + SR + (c & 1) * SD;
            for (int p = p0 + ll; p < p1; p += 16) cp_async16(bs + 2 * (p - p0), row + 2 * p);
            const int r0 = s_soff[c], r1 = s_soff[c + 1];
            for (int r = r0 + ll; r < r1; r += 16) {
                DFSIM_CHECK(s_slist[r] < a.t.n_long && 2 * K + (r - r0) < SD, 11);
                cp_async8(bs + 2 * K + (r - r0), spill_row + s_slist[r]);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        double len = 0.0;
        int src = 0x7fffffff;
        if (NC > 0) prefetch(NC - 1);
        for (int c = NC - 1; c >= 0; c--) {
            // chunk c-1 may read spill values written up to chunk c+1: all complete (and
            // ordered by the __syncwarp that ended chunk c+1) before this prefetch is issued
            if (c > 0) {
                prefetch(c - 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncwarp();
            const double2 *bs = reinterpret_cast<const double2 *>(region + SR + (c & 1) * SD);
            const int g0 = s_coff[c], g1 = s_coff[c + 1];
            const int p0 = s_goff[g0];
            int q1 = s_goff[g1];  // groups are contiguous: group gi ends where gi+1 began
            for (int gi = g1 - 1; gi >= g0; gi--) {
                const int q0 = s_goff[gi];
                const int p = q0 + ll;
                if (p < q1) {
                    uint2 pm;
                    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(pm.x), "=r"(pm.y) : "r"(a_pm + 8u * p));
                    const uint32_t m = pm.x, info = pm.y;
                    const int j0 = static_cast<int>(m & 0xffffu), j1 = j0 + static_cast<int>((m >> 16) & 0xffu);
                    double best = 0.0;  // max(0.0, .) (graph.py:465-468)
                    DFSIM_CHECK(j1 <= E, 10);
                    for (int j = j0; j < j1; j++) {
                        DFSIM_CHECK(s_succ[j] < SR + 2 * SD, 10);
                        const double x = region[s_succ[j]];
                        best = x > best ? x : best;
                    }
                    const double2 sf = bs[p - p0];
                    const double sv = __dadd_rn(__dsub_rn(sf.y, sf.x), best);  // finish - start (reporting.py:128)
                    DFSIM_CHECK(!(info & 0x8000u) || (info & 0x7fffu) < static_cast<unsigned>(SR), 11);
                    DFSIM_CHECK(!(info >> 31) || ((info >> 16) & 0x7fffu) < static_cast<unsigned>(a.t.n_long), 11);
                    if (info & 0x8000u) region[info & 0x7fffu] = sv;
                    if (live && (info >> 31)) spill_row[(info >> 16) & 0x7fffu] = sv;
                    if ((m >> 24) & 1u) {
                        const int r = __ldg(a.t.rank_of_pos + p);
                        if (src == 0x7fffffff || sv > len || (sv == len && r < src)) {
                            len = sv;
                            src = r;
                        }
                    }
                }
                q1 = q0;
                __syncwarp();
            }
        }
        // max over sources, then the min id achieving it (graph.py:471-474), per half-warp
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const double ol = __shfl_xor_sync(DFSIM_FULL_MASK, len, o);
            const int os = __shfl_xor_sync(DFSIM_FULL_MASK, src, o);
            if (os != 0x7fffffff && (src == 0x7fffffff || ol > len || (ol == len && os < src))) {
                len = ol;
                src = os;
            }
        }
        if (live && ll == 0) {
            const int64_t cand = a.cand ? __ldg(a.cand + s) : s;  // s is the schedule slot
            a.cp_len[cand] = src == 0x7fffffff ? 0.0 : len;
            if (a.cp_src) a.cp_src[cand] = src == 0x7fffffff ? -1 : src;
        }
        __syncwarp();
    }
}

}  // namespace

namespace {
struct FusedShape {
    size_t graph_bytes, warp_bytes, smem;
    int gs, per_warp, wpb;
    bool fits, base_global;
};

// Duration rows stay in smem unless that leaves fewer than this many candidates per CTA
constexpr int kBaseGlobalBelow = 32;

FusedShape fused_shape_with(const dfsim_sim_tables *g, bool base_global) {
    FusedShape f;
    const size_t N = (size_t)g->n_nodes;
    f.base_global = base_global;
    f.graph_bytes = (N * (g->succ_packed ? 6 : 8) + (size_t)g->n_edges * 4 + 15) / 16 * 16 + (base_global ? 0 : N * 8);
    const size_t tail_bytes = g->n_devices <= 16 ? 64 : 128;  // 4-byte tail per device, padded
    f.warp_bytes = (tail_bytes + (size_t)g->n_counter_words * 4 + (size_t)g->n_devices * (g->qcap + 2) * 2 + 15) / 16 * 16;
    f.gs = g->n_devices <= 10 ? 10 : (g->n_devices <= 16 ? 16 : 32);

    // the candidate groups of one warp start on spread-out banks: 16 banks apart for two
    // groups (stride == 64 mod 128 bytes), 11 banks apart for three (== 44 mod 128)
    f.warp_bytes = (f.warp_bytes + 127) / 128 * 128 + (f.gs == 10 ? 44 : 64);
    const size_t budget = 227 * 1024 - 64;
    f.per_warp = 32 / f.gs;
    f.wpb = 32;
    while (f.wpb > 1 && f.graph_bytes + (size_t)f.wpb * f.per_warp * f.warp_bytes > budget) f.wpb--;
    f.smem = f.graph_bytes + (size_t)f.wpb * f.per_warp * f.warp_bytes;
    f.fits = f.smem <= budget;
    return f;
}

FusedShape fused_shape(const dfsim_sim_tables *g) {
    const FusedShape f = fused_shape_with(g, false);
    if (f.fits && f.wpb * f.per_warp >= kBaseGlobalBelow) return f;
    const FusedShape h = fused_shape_with(g, true);
    return h.fits && (!f.fits || h.wpb * h.per_warp > f.wpb * f.per_warp) ? h : f;
}
}  // namespace

extern "C" int32_t dfsim_fused_capacity(const dfsim_sim_tables *g) {
    if (!g || g->n_nodes <= 0) return 0;
    const FusedShape f = fused_shape(g);
    return f.fits ? f.wpb * f.per_warp : 0;
}

extern "C" int32_t dfsim_fused_chunk(const dfsim_sim_tables *g, int64_t n_sims, int32_t num_sms) {
    const int32_t cap = dfsim_fused_capacity(g);
    if (cap <= 0 || n_sims <= 0 || num_sms <= 0) return cap;
    const FusedShape f = fused_shape(g);
    const int64_t pw = f.per_warp;
    auto warps = [&](int64_t c) { return (c + pw - 1) / pw * pw; };
    // enough chunks to cover every SM, each holding at least as many candidate bytes as its
    // CTA's copy of the class tables (smaller chunks would trade candidates for table copies)
    const int64_t spread = warps((n_sims + num_sms - 1) / num_sms);
    const int64_t least = warps((int64_t)((f.graph_bytes + f.warp_bytes - 1) / f.warp_bytes));
    int64_t c = spread > least ? spread : least;
    return c < cap ? static_cast<int32_t>(c) : cap;
}

extern "C" int dfsim_simulate_fused(dfsim_ctx *ctx, const dfsim_sim_tables *g, const dfsim_fused_strategies *st,
                                    double *sched, double *makespan, double *busy, int32_t *n_placed,
                                    int32_t *flags) {
    if (!ctx || !g || !st) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, sched && makespan && n_placed && flags, "outputs are required");
    DFSIM_ARG_CHECK(ctx, (reinterpret_cast<uintptr_t>(sched) & 15) == 0, "sched must be 16-byte aligned");
    DFSIM_ARG_CHECK(ctx, g->n_nodes > 0 && g->n_nodes <= 65535 && g->n_devices <= 32, "fused engine limits");
    DFSIM_ARG_CHECK(ctx, g->qcap >= 2 && (g->qcap & (g->qcap - 1)) == 0, "qcap must be a power of two");
    DFSIM_ARG_CHECK(ctx, g->n_counter_words >= 1 && g->n_counter_words <= 512, "1..512 counter words");
    DFSIM_ARG_CHECK(ctx, !g->succ_packed || (g->n_nodes <= 8192 && g->n_devices <= 16 && g->counter_bits <= 4 &&
                                             g->n_counter_words <= 256), "packed successor format limits");
    if (st->n_sims <= 0 || st->n_chunks <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const FusedShape f = fused_shape(g);
    DFSIM_ARG_CHECK(ctx, f.fits, "class tables do not fit in shared memory");
    const size_t graph_bytes = f.graph_bytes, warp_bytes = f.warp_bytes;
    const int gs = f.gs;
    DFSIM_ARG_CHECK(ctx, st->max_chunk >= 0 && st->max_chunk <= f.wpb * f.per_warp, "max_chunk exceeds the capacity");
    // CTAs hold max_chunk candidates: a class cut into small chunks runs as many small CTAs
    // (several per SM) instead of a few full ones
    const int wpb = st->max_chunk > 0 ? (st->max_chunk + f.per_warp - 1) / f.per_warp : f.wpb;
    FusedArgs a;
    a.g = *g;
    a.st = *st;
    a.sched = sched; a.makespan = makespan; a.busy = busy; a.n_placed = n_placed; a.flags = flags;
    a.wpb = wpb;
    a.smem_graph = (int)graph_bytes;
    a.smem_warp = (int)warp_bytes;
    a.tail_bytes = g->n_devices <= 16 ? 64 : 128;
    void *p = nullptr;
    int rc = dfsim_scratch(ctx, 256, &p);
    if (rc) return rc;
    a.chunk_counter = static_cast<int32_t *>(p);
    DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(a.chunk_counter, 0, sizeof(int32_t), ctx->stream));
    const size_t smem = graph_bytes + (size_t)wpb * f.per_warp * warp_bytes;
    const int threads = wpb * 32;
#define DFSIM_LAUNCH_FUSED_T(GS, PK, BG, TL)                                                                   \
    do {                                                                                                       \
        DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_simulate_fused<GS, PK, BG, TL>,                             \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));     \
        int occ = 1;                                                                                           \
        DFSIM_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_simulate_fused<GS, PK, BG, TL>, \
                                                                          threads, smem));                    \
        const int64_t slots = (int64_t)ctx->num_sms * (occ > 0 ? occ : 1);                                    \
        const int grid = (int)(slots < st->n_chunks ? slots : st->n_chunks);                                   \
        k_simulate_fused<GS, PK, BG, TL><<<grid, threads, smem, ctx->stream>>>(a);                            \
    } while (0)
#define DFSIM_LAUNCH_FUSED_B(GS, PK, BG)                                                                       \
    do {                                                                                                       \
        if (st->sched_tiled) DFSIM_LAUNCH_FUSED_T(GS, PK, BG, true); else DFSIM_LAUNCH_FUSED_T(GS, PK, BG, false); \
    } while (0)
#define DFSIM_LAUNCH_FUSED_P(GS, PK)                                                                           \
    do {                                                                                                       \
        if (f.base_global) DFSIM_LAUNCH_FUSED_B(GS, PK, true); else DFSIM_LAUNCH_FUSED_B(GS, PK, false);       \
    } while (0)
#define DFSIM_LAUNCH_FUSED(GS)                                                                                 \
    do {                                                                                                       \
        if (g->succ_packed) DFSIM_LAUNCH_FUSED_P(GS, true); else DFSIM_LAUNCH_FUSED_P(GS, false);              \
    } while (0)
    if (gs == 10) DFSIM_LAUNCH_FUSED(10); else if (gs == 16) DFSIM_LAUNCH_FUSED(16); else DFSIM_LAUNCH_FUSED(32);
#undef DFSIM_LAUNCH_FUSED
#undef DFSIM_LAUNCH_FUSED_P
#undef DFSIM_LAUNCH_FUSED_B
#undef DFSIM_LAUNCH_FUSED_T
    return dfsim_after_launch(ctx, "k_simulate_fused");
}

namespace {
// shared-memory layout of k_critical_path_levels: class tables once per CTA, then one
// region pair (slots + two prefetch stages) per two candidates (a warp)
struct CpShape {
    size_t table_bytes, per_warp;
    int wpb;  // warps that fit (0: not even one)
};

CpShape cp_shape(const dfsim_cp_tables *t) {
    CpShape c;
    c.table_bytes = ((size_t)t->n_nodes * 8 + (size_t)t->n_edges * 2 + (size_t)(t->n_groups + 1) * 2 +
                     (size_t)(t->n_chunks + 1) * 4 + (size_t)t->n_edges * 2 + 15) / 16 * 16;
    // layout: (cp_meta, pinfo) pairs 8N | succ 2E | group_off 2(G+1) | chunk/spill offsets 4(NC+1) | spill list <= 2E
    c.per_warp = 2 * ((size_t)t->slot_region + 2 * (size_t)t->stage_doubles) * 8;  // two candidates
    const size_t budget = 227 * 1024 - 64;
    c.wpb = 32;
    while (c.wpb > 0 && c.table_bytes + c.wpb * c.per_warp > budget) c.wpb--;
    return c;
}
}  // namespace

extern "C" int32_t dfsim_critical_path_levels_capacity(const dfsim_cp_tables *t) {
    return t ? 2 * cp_shape(t).wpb : 0;
}

extern "C" int dfsim_critical_path_levels(dfsim_ctx *ctx, const dfsim_cp_tables *t, int64_t n_sims,
                                          const int64_t *cand_of_slot, const double *sched, double *cp_len,
                                          int32_t *cp_src) {
    if (!ctx || !t) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, sched && cp_len, "sched and cp_len are required");
    DFSIM_ARG_CHECK(ctx, (reinterpret_cast<uintptr_t>(sched) & 15) == 0, "sched must be 16-byte aligned");
    DFSIM_ARG_CHECK(ctx, t->chunk_positions >= 16, "chunk_positions >= 16");
    DFSIM_ARG_CHECK(ctx, t->n_nodes <= 65535 && t->n_edges <= 65535 && t->n_slots < 0x7fff &&
                         t->max_spill_reads < 0x7fff && t->slot_region + 2 * t->stage_doubles < 65536,
                    "level tables use 16-bit ids");
    DFSIM_ARG_CHECK(ctx, t->stage_doubles >= 2 * t->chunk_positions + t->max_spill_reads && t->slot_region >= t->n_slots,
                    "inconsistent critical-path region layout");
    if (n_sims <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const CpShape shape = cp_shape(t);
    const size_t table_bytes = shape.table_bytes, per_warp = shape.per_warp;
    int wpb = shape.wpb;
    DFSIM_ARG_CHECK(ctx, wpb >= 1, "critical-path tables do not fit in shared memory (dfsim_critical_path_levels_capacity)");
    // a small batch is spread over every SM (fewer warps per CTA, several CTAs per SM), but
    // never so thin that the per-CTA table copy outweighs the candidates' regions
    const int64_t spread = (n_sims + 2 * (int64_t)ctx->num_sms - 1) / (2 * (int64_t)ctx->num_sms);
    const int64_t least = (int64_t)((table_bytes + per_warp - 1) / per_warp);
    const int64_t thin = spread > least ? spread : least;
    if (thin < wpb) wpb = thin < 1 ? 1 : (int)thin;
    const size_t smem = table_bytes + wpb * per_warp;
    DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_critical_path_levels, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 1;
    const int threads = wpb * 32;
    DFSIM_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_critical_path_levels, threads, smem));
    const int64_t want = (n_sims + 2 * wpb - 1) / (2 * wpb);
    const int64_t slots = (int64_t)ctx->num_sms * (occ > 0 ? occ : 1);
    const int grid = (int)(want < slots ? want : slots);
    void *p = nullptr;
    int rc = dfsim_scratch(ctx, (size_t)grid * wpb * 2 * (size_t)(t->n_long > 0 ? t->n_long : 1) * 8, &p);
    if (rc) return rc;
    CpLevelArgs a;
    a.t = *t;
    a.S = n_sims;
    a.cand = cand_of_slot;
    a.sched = sched; a.cp_len = cp_len; a.cp_src = cp_src;
    a.spill = static_cast<double *>(p);
    a.wpb = wpb;
    a.table_bytes = (int)table_bytes;
    k_critical_path_levels<<<grid, threads, smem, ctx->stream>>>(a);
    return dfsim_after_launch(ctx, "k_critical_path_levels");
}
