// K4 v3 dfsim_critical_path_lanes: graph.py:446-474 on finish - start (reporting.py:128)
// with one candidate per LANE.
//
// The critical-path DP does not branch on data: every candidate of a topology class walks
// the same reverse topological order with the same reads.  So a warp takes 32 candidates
// and walks the class's level positions from the last to the first, one node per step,
// all lanes in lock-step: the node's table record and successor list are warp-uniform
// (one broadcast read for 32 candidates) and only the values differ per lane.  Per node and
// lane: one 16-byte (start, finish) read, one 8-byte read per successor, one max, two adds.
//
// Storage of suffix values (A4: suffix[v] = (finish - start)[v] + max(0, max succ suffix)):
//  * read within the writer's prefetch chunk or the next one -> a shared-memory slot
//    (interval colouring by the host planner, a few dozen slots);
//  * read later (forward activations read by their backward consumers ~half a graph
//    later) -> the warp's spill row [n_long][32] in global memory (one coalesced 256-byte
//    store per value), prefetched into a shared stage together with the reading chunk.
// Schedule pairs are prefetched with cp.async one chunk ahead: each candidate's chunk is a
// contiguous 256-byte run of its row (positions are level order), so the copies coalesce.
//
// Exactness: the same single max and add per node as graph.py:463-469 (any reverse
// topological order gives identical bits, A4); source = smallest rank among the maxima.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace {

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    unsigned r;
    asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void cpa16(unsigned dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cpa8(unsigned dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ double lds_d(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_d(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ double2 lds_d2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds_u2(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_h(unsigned a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_i(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

constexpr unsigned kHasSlot = 1u << 12, kSource = 1u << 13, kHasSpill = 1u << 14;

struct LaneArgs {
    dfsim_cp_lane_tables t;
    int64_t S;
    const double *sched;  // [S][N] (start, finish) pairs by level position
    double *cp_len;
    int32_t *cp_src;
    double *spill;        // [grid * wpb][n_long][32]
    int32_t wpb;
    int32_t table_bytes;
    int32_t region_bytes;
};

template <int K>
__global__ void __launch_bounds__(1024, 1) k_critical_path_lanes(LaneArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int kStride = K * 16 + 16;  // bytes per candidate in a pair stage (padded: conflict-free LDS.128)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int N = a.t.n_nodes, E = a.t.n_edges, NQ = a.t.n_chunks, NS = a.t.n_slots, RM = a.t.rmax;
    const int NL = a.t.n_spill_list;
    // CTA tables: rec[N] (uint2) | succ[E] (u16) | bounds[NQ+1] | spill_off[NQ+1] | spill_list[NL] (u16)
    uint2 *s_rec = reinterpret_cast<uint2 *>(smem);
    uint16_t *s_succ = reinterpret_cast<uint16_t *>(s_rec + N);
    int32_t *s_bounds = reinterpret_cast<int32_t *>(smem + ((static_cast<size_t>(N) * 8 + static_cast<size_t>(E) * 2 + 15) / 16) * 16);
    int32_t *s_soff = s_bounds + (NQ + 1);
    uint16_t *s_slist = reinterpret_cast<uint16_t *>(s_soff + (NQ + 1));
    for (int i = threadIdx.x; i < N; i += blockDim.x)
        s_rec[i] = make_uint2(__ldg(a.t.rec + 2 * i), __ldg(a.t.rec + 2 * i + 1));
    for (int i = threadIdx.x; i < E; i += blockDim.x) s_succ[i] = __ldg(a.t.succ + i);
    for (int i = threadIdx.x; i <= NQ; i += blockDim.x) {
        s_bounds[i] = __ldg(a.t.bounds + i);
        s_soff[i] = __ldg(a.t.spill_off + i);
    }
    for (int i = threadIdx.x; i < NL; i += blockDim.x) s_slist[i] = __ldg(a.t.spill_list + i);
    __syncthreads();

    const unsigned a_rec = smem_u32(s_rec), a_succ = smem_u32(s_succ), a_bounds = smem_u32(s_bounds);
    const unsigned a_soff = smem_u32(s_soff), a_slist = smem_u32(s_slist);
    unsigned char *region = smem + a.table_bytes + static_cast<size_t>(warp) * a.region_bytes;
    const unsigned a_region = smem_u32(region);                  // rows of 256 B: slots | spill stage 0 | 1
    const unsigned a_lane = a_region + 8u * lane;                // this lane's column in every row
    const unsigned a_pairs = a_region + static_cast<unsigned>(NS + 2 * RM) * 256u;  // two pair stages
    const int64_t slot_warp = static_cast<int64_t>(blockIdx.x) * a.wpb + warp;
    double *spill_warp = a.spill + slot_warp * static_cast<int64_t>(a.t.n_long) * 32 + lane;
    asm volatile("mov.b64 %0, %0;" : "+l"(spill_warp));
    const int64_t step = static_cast<int64_t>(gridDim.x) * a.wpb * 32;

    for (int64_t wbase = slot_warp * 32; wbase < a.S; wbase += step) {
        const bool live = wbase + lane < a.S;
        const int n_live = static_cast<int>(a.S - wbase < 32 ? a.S - wbase : 32);
        const double *rows = a.sched + 2 * wbase * N;
        asm volatile("mov.b64 %0, %0;" : "+l"(rows));

        auto prefetch = [&](int q) {
            const int hi = lds_i(a_bounds + 4u * q);
            const int wlo = hi > K ? hi - K : 0;
            const unsigned st = a_pairs + static_cast<unsigned>(q & 1) * (32u * kStride);
#pragma unroll
            for (int k = lane; k < 32 * K; k += 32) {  // candidate c = k / K, pair i = k % K: coalesced runs
                const int c = k / K, i = k % K;
                if (c < n_live && wlo + i < N)
                    cpa16(st + static_cast<unsigned>(c * kStride + i * 16), rows + 2 * (static_cast<int64_t>(c) * N + wlo + i));
            }
            const int r0 = lds_i(a_soff + 4u * q), r1 = lds_i(a_soff + 4u * (q + 1));
            const unsigned ss = a_lane + static_cast<unsigned>(NS + (q & 1) * RM) * 256u;
            if (live)
                for (int r = r0; r < r1; r++) cpa8(ss + static_cast<unsigned>(r - r0) * 256u, spill_warp + 32 * static_cast<int64_t>(lds_h(a_slist + 2u * r)));
            asm volatile("cp.async.commit_group;\n" ::);
        };

        double len = 0.0;
        int src = 0x7fffffff;
        if (NQ > 0) prefetch(0);
        for (int q = 0; q < NQ; q++) {
            if (q + 1 < NQ) {
                prefetch(q + 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncwarp();
            const int hi = lds_i(a_bounds + 4u * q), lo = lds_i(a_bounds + 4u * (q + 1));
            const int wlo = hi > K ? hi - K : 0;
            const unsigned pst = a_pairs + static_cast<unsigned>(q & 1) * (32u * kStride) + static_cast<unsigned>(lane * kStride) - 16u * wlo;
            for (int p = hi - 1; p >= lo; p--) {
                const uint2 r = lds_u2(a_rec + 8u * p);
                const int j0 = static_cast<int>(r.x & 0xffffffu), j1 = j0 + static_cast<int>(r.x >> 24);
                double best = 0.0;  // max(0.0, .) (graph.py:465-468)
                for (int j = j0; j < j1; j++) {
                    const double x = lds_d(a_lane + 256u * lds_h(a_succ + 2u * j));
                    best = x > best ? x : best;
                }
                const double2 sf = lds_d2(pst + 16u * p);
                const double sv = __dadd_rn(__dsub_rn(sf.y, sf.x), best);  // finish - start (reporting.py:128)
                if (r.y & kHasSlot) sts_d(a_lane + 256u * (r.y & 0xfffu), sv);
                if ((r.y & kHasSpill) && live) spill_warp[32 * static_cast<int64_t>(r.y >> 15)] = sv;
                if (r.y & kSource) {
                    const int rk = __ldg(a.t.rank_of_pos + p);
                    if (src == 0x7fffffff || sv > len || (sv == len && rk < src)) {
                        len = sv;
                        src = rk;
                    }
                }
            }
            __syncwarp();
        }
        if (live) {
            a.cp_len[wbase + lane] = src == 0x7fffffff ? 0.0 : len;
            if (a.cp_src) a.cp_src[wbase + lane] = src == 0x7fffffff ? -1 : src;
        }
    }
}

struct LaneShape {
    size_t table_bytes, region_bytes;
    int wpb;
};

LaneShape lane_shape(const dfsim_cp_lane_tables *t) {
    const int spill_list_len = t->n_spill_list;
    LaneShape s;
    const size_t K = static_cast<size_t>(t->chunk_positions);
    s.table_bytes = ((static_cast<size_t>(t->n_nodes) * 8 + static_cast<size_t>(t->n_edges) * 2 + 15) / 16) * 16 +
                    ((static_cast<size_t>(t->n_chunks + 1) * 8 + static_cast<size_t>(spill_list_len) * 2 + 15) / 16) * 16;
    s.region_bytes = static_cast<size_t>(t->n_slots + 2 * t->rmax) * 256 + 2 * 32 * (K * 16 + 16);
    const size_t budget = 227 * 1024 - 64;
    s.wpb = 32;
    while (s.wpb > 0 && s.table_bytes + s.wpb * s.region_bytes > budget) s.wpb--;
    return s;
}

}  // namespace

extern "C" int dfsim_cp_lanes_plan(int32_t n, const int32_t *succ_off, const int32_t *succ_pos, const uint8_t *is_source,
                                   int32_t K, int32_t rmax_min, uint32_t *rec, uint16_t *succ_loc, int32_t *bounds,
                                   int32_t *spill_off, uint16_t *spill_list, int32_t *info) {
    if (n < 0 || !succ_off || !info || K < 1 || K > 16 || rmax_min < 1) return DFSIM_BAD_ARGUMENT;
    const int64_t E = n ? succ_off[n] : 0;
    if (E >= (1 << 24)) return DFSIM_BAD_ARGUMENT;
    std::vector<int32_t> chunk_of(n, -1), stamp(n, -1), far_idx(E, -1);
    std::vector<uint8_t> is_long(n, 0);
    std::vector<int32_t> slist;  // spill positions per chunk, concatenated
    int32_t rmax = rmax_min, q = 0, p = n - 1;
    bounds[0] = n;
    spill_off[0] = 0;
    while (p >= 0) {
        const int32_t hi = p + 1, first = static_cast<int32_t>(slist.size());
        while (p >= 0 && hi - p <= K) {
            if (succ_off[p + 1] - succ_off[p] >= 255) return DFSIM_BAD_ARGUMENT;
            int32_t fresh = 0;  // distinct far successors not yet in this chunk's list
            for (int64_t j = succ_off[p]; j < succ_off[p + 1]; j++) {
                const int32_t v = succ_pos[j];
                if (v <= p || v >= n) return DFSIM_BAD_ARGUMENT;  // not a level order
                if (q - chunk_of[v] >= 2 && stamp[v] != q) {
                    stamp[v] = q;  // provisional: undone below if p moves to the next chunk
                    fresh++;
                }
            }
            const int32_t have = static_cast<int32_t>(slist.size()) - first;
            if (have + fresh > rmax && p < hi - 1) {  // chunk full: p starts the next one
                for (int64_t j = succ_off[p]; j < succ_off[p + 1]; j++) {
                    const int32_t v = succ_pos[j];
                    if (stamp[v] == q && std::find(slist.begin() + first, slist.end(), v) == slist.end()) stamp[v] = -1;
                }
                break;
            }
            if (have + fresh > rmax) rmax = have + fresh;  // one node alone: widen the stage
            for (int64_t j = succ_off[p]; j < succ_off[p + 1]; j++) {
                const int32_t v = succ_pos[j];
                if (q - chunk_of[v] >= 2) {
                    auto it = std::find(slist.begin() + first, slist.end(), v);
                    if (it == slist.end()) {
                        slist.push_back(v);
                        it = slist.end() - 1;
                    }
                    far_idx[j] = static_cast<int32_t>(it - (slist.begin() + first));
                    is_long[v] = 1;
                }
            }
            chunk_of[p] = q;
            p--;
        }
        bounds[q + 1] = p + 1;
        spill_off[q + 1] = static_cast<int32_t>(slist.size());
        q++;
    }
    const int32_t NQ = q;
    // spill indices in write order (descending positions: the warp's stores run forward)
    std::vector<int32_t> spill_of(n, -1);
    int32_t n_long = 0;
    for (int32_t v = n - 1; v >= 0; v--)
        if (is_long[v]) spill_of[v] = n_long++;
    if (n_long > 65536 || n_long >= (1 << 17)) return DFSIM_BAD_ARGUMENT;
    for (size_t i = 0; i < slist.size(); i++) spill_list[i] = static_cast<uint16_t>(spill_of[slist[i]]);
    // slots: values read near (same or next chunk) are live from their write step to the last near
    // read; greedy interval colouring in processing order (step t = n - 1 - position)
    std::vector<int32_t> last_near(n, -1);
    for (int32_t u = 0; u < n; u++)
        for (int64_t j = succ_off[u]; j < succ_off[u + 1]; j++)
            if (far_idx[j] < 0) last_near[succ_pos[j]] = std::max(last_near[succ_pos[j]], n - 1 - u);
    std::vector<int32_t> slot_of(n, -1), free_slots;
    std::vector<std::vector<int32_t>> release(n);
    int32_t n_slots = 0;
    for (int32_t v = n - 1; v >= 0; v--) {
        const int32_t t = n - 1 - v;
        for (int32_t s : release[t]) free_slots.push_back(s);  // last read at this step: reusable now
        if (last_near[v] < 0) continue;
        int32_t s;
        if (!free_slots.empty()) {
            s = free_slots.back();
            free_slots.pop_back();
        } else {
            s = n_slots++;
        }
        slot_of[v] = s;
        release[last_near[v]].push_back(s);
    }
    if (n_slots >= 4096) return DFSIM_BAD_ARGUMENT;
    const int32_t NS = std::max(n_slots, 1);
    for (int32_t u = 0; u < n; u++) {
        const int32_t cnt = succ_off[u + 1] - succ_off[u];
        rec[2 * u] = static_cast<uint32_t>(succ_off[u]) | (static_cast<uint32_t>(cnt) << 24);
        uint32_t y = 0;
        if (slot_of[u] >= 0) y |= static_cast<uint32_t>(slot_of[u]) | kHasSlot;
        if (is_source && is_source[u]) y |= kSource;
        if (spill_of[u] >= 0) y |= kHasSpill | (static_cast<uint32_t>(spill_of[u]) << 15);
        rec[2 * u + 1] = y;
        for (int64_t j = succ_off[u]; j < succ_off[u + 1]; j++) {
            const int32_t row = far_idx[j] >= 0 ? NS + (chunk_of[u] & 1) * rmax + far_idx[j] : slot_of[succ_pos[j]];
            if (row < 0 || row >= 65536) return DFSIM_BAD_ARGUMENT;
            succ_loc[j] = static_cast<uint16_t>(row);
        }
    }
    info[0] = NQ;
    info[1] = NS;
    info[2] = rmax;
    info[3] = n_long;
    info[4] = static_cast<int32_t>(slist.size());
    return DFSIM_OK;
}

extern "C" int32_t dfsim_critical_path_lanes_capacity(const dfsim_cp_lane_tables *t) {
    if (!t || t->n_chunks <= 0) return 0;
    return lane_shape(t).wpb;
}

extern "C" int dfsim_critical_path_lanes(dfsim_ctx *ctx, const dfsim_cp_lane_tables *t, int64_t n_sims,
                                         const double *sched, double *cp_len, int32_t *cp_src) {
    if (!ctx || !t) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, sched && cp_len, "sched and cp_len are required");
    DFSIM_ARG_CHECK(ctx, (reinterpret_cast<uintptr_t>(sched) & 15) == 0, "sched must be 16-byte aligned");
    DFSIM_ARG_CHECK(ctx, t->chunk_positions == 8 || t->chunk_positions == 16, "chunk_positions must be 8 or 16");
    DFSIM_ARG_CHECK(ctx, t->n_nodes > 0 && t->n_chunks > 0 && t->n_slots >= 1 && t->n_slots < 4096 && t->rmax >= 1 &&
                         t->n_spill_list >= 0 && t->n_edges < (1 << 24),
                    "inconsistent lane tables");
    if (n_sims <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const LaneShape shape = lane_shape(t);
    DFSIM_ARG_CHECK(ctx, shape.wpb >= 1, "lane tables do not fit in shared memory");
    // as many warps as the batch needs, spread over the SMs
    const int64_t warps = (n_sims + 31) / 32;
    int wpb = shape.wpb;
    const int64_t per_sm = (warps + ctx->num_sms - 1) / ctx->num_sms;
    if (per_sm < wpb) wpb = static_cast<int>(per_sm < 1 ? 1 : per_sm);
    const size_t smem = shape.table_bytes + static_cast<size_t>(wpb) * shape.region_bytes;
    const int grid = static_cast<int>(std::min<int64_t>((warps + wpb - 1) / wpb, ctx->num_sms));
    void *p = nullptr;
    int rc = dfsim_scratch(ctx, static_cast<size_t>(grid) * wpb * std::max(t->n_long, 1) * 32 * 8, &p);
    if (rc) return rc;
    LaneArgs a;
    a.t = *t;
    a.S = n_sims;
    a.sched = sched;
    a.cp_len = cp_len;
    a.cp_src = cp_src;
    a.spill = static_cast<double *>(p);
    a.wpb = wpb;
    a.table_bytes = static_cast<int32_t>(shape.table_bytes);
    a.region_bytes = static_cast<int32_t>(shape.region_bytes);
    auto launch = [&](auto kern) -> int {
        DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<grid, wpb * 32, smem, ctx->stream>>>(a);
        return dfsim_after_launch(ctx, "k_critical_path_lanes");
    };
    return t->chunk_positions == 16 ? launch(k_critical_path_lanes<16>) : launch(k_critical_path_lanes<8>);
}
