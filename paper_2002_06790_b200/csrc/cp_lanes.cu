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
//  * read within the next NST - 1 prefetch chunks of its writer's -> a shared-memory slot
//    (interval colouring by the host planner, a few dozen slots);
//  * read later (forward activations read by their backward consumers ~half a graph
//    later) -> the warp's spill row [n_long][32] in global memory (one coalesced 256-byte
//    store per value), prefetched into a shared stage together with the reading chunk.
// Schedule pairs, the chunk's node records (first four successor rows inline) and its spill
// values are prefetched with cp.async NST - 1 chunks ahead (NST = 2 or 3 stages): each
// candidate's chunk is a contiguous run of its row (positions are level order), so the
// copies coalesce, and no class table occupies shared memory beyond a few offsets.
//
// Exactness: the same single max and add per node as graph.py:463-469 (any reverse
// topological order gives identical bits, A4); source = smallest rank among the maxima.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
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
__device__ __forceinline__ uint4 lds_u4(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_i(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

constexpr unsigned kHasSlot = 1u << 12, kSource = 1u << 13, kHasSpill = 1u << 14;

// a_lane + 256 * (16-bit row field lo / hi of w): one byte permute moves the field to bytes 1-2
__device__ __forceinline__ unsigned row_lo(unsigned a_lane, unsigned w) { return a_lane + __byte_perm(w, 0u, 0x4104); }
__device__ __forceinline__ unsigned row_hi(unsigned a_lane, unsigned w) { return a_lane + __byte_perm(w, 0u, 0x4324); }

struct LaneArgs {
    dfsim_cp_lane_tables t;
    int64_t S;
    const double *sched;  // [S][N] (start, finish) pairs by level position
    double *cp_len;
    int32_t *cp_src;
    double *spill;        // [grid * wpb][n_long][32]
    int32_t *task_counter; // groups of 32 candidates handed out dynamically (SMs finish together)
    const int64_t *slots;  // optional: lane i of task t takes schedule slot slots[32 t + i]
    const int64_t *cand;   // optional: candidate of each schedule slot (outputs go to cp_len[cand[slot]])
    int32_t wpb;
    int32_t table_bytes;  // CTA tables: bounds | spill_off | block_off | spill_list
    int32_t region_bytes; // per warp: rows [slots | spill stages | zero row] | block stages
};

// Register-staged variant (K = 8): each lane loads its own candidate's 8 (start, finish)
// pairs of the next chunk straight into registers, one chunk ahead, so the pair stages need no
// shared memory and twice as many warps fit an SM.  Schedules are tiled by 32 candidates
// (position-major inside a tile, see dfsim_b200.h): position p of a warp's 32 candidates is one
// contiguous 512-byte run, so each of the 8 loads per chunk is a fully coalesced LDG.128.  Node
// records and spill values use two shared-memory stages as above.
__device__ __forceinline__ void ldg_pair(double (&d)[2], const double *p) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(d[0]), "=d"(d[1]) : "l"(p));
}

// 14 warps per CTA (one CTA per SM): what shared memory holds for C2 anyway
constexpr int kRegWarps = 14;

template <int K>
__global__ void __launch_bounds__(kRegWarps * 32, 1) k_critical_path_lanes_reg(LaneArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NST = 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int N = a.t.n_nodes, NQ = a.t.n_chunks, NS = a.t.n_slots, RM = a.t.rmax, BM = a.t.block_max;
    const int NL = a.t.n_spill_list;
    int32_t *s_bounds = reinterpret_cast<int32_t *>(smem);
    int32_t *s_soff = s_bounds + (NQ + 1);
    int32_t *s_boff = s_soff + (NQ + 1);
    uint16_t *s_slist = reinterpret_cast<uint16_t *>(s_boff + (NQ + 1));
    for (int i = threadIdx.x; i <= NQ; i += blockDim.x) {
        s_bounds[i] = __ldg(a.t.bounds + i);
        s_soff[i] = __ldg(a.t.spill_off + i);
        s_boff[i] = __ldg(a.t.block_off + i);
    }
    for (int i = threadIdx.x; i < NL; i += blockDim.x) s_slist[i] = __ldg(a.t.spill_list + i);
    __syncthreads();

    const unsigned a_bounds = smem_u32(s_bounds), a_soff = smem_u32(s_soff), a_boff = smem_u32(s_boff);
    const unsigned a_slist = smem_u32(s_slist);
    unsigned char *region = smem + a.table_bytes + static_cast<size_t>(warp) * a.region_bytes;
    const unsigned a_region = smem_u32(region);
    const unsigned a_lane = a_region + 8u * lane;
    const unsigned a_zero = a_region + static_cast<unsigned>(NS + NST * RM) * 256u;  // row of 0.0 (never written)
    const unsigned a_blocks = a_zero + 256u;
    sts_d(a_zero + 8u * lane, 0.0);
    __syncwarp();
    const int64_t slot_warp = static_cast<int64_t>(blockIdx.x) * a.wpb + warp;
    double *spill_warp = a.spill + slot_warp * static_cast<int64_t>(a.t.n_long) * 32 + lane;
    asm volatile("mov.b64 %0, %0;" : "+l"(spill_warp));
    const int64_t n_tasks = (a.S + 31) / 32;
    for (;;) {
        int task = 0;
        if (lane == 0) task = atomicAdd(a.task_counter, 1);
        task = __shfl_sync(DFSIM_FULL_MASK, task, 0);
        if (task >= n_tasks) break;
        const int64_t k = static_cast<int64_t>(task) * 32 + lane;
        const bool live = k < a.S;
        const int64_t kk = live ? k : a.S - 1;  // idle lanes shadow the last candidate's row
        const int64_t slot = a.slots ? __ldg(a.slots + kk) : kk;
        const int64_t s = a.cand ? __ldg(a.cand + slot) : slot;  // the candidate (outputs)
        // slot k, position p: pair ((k / 32) N + p) 32 + k % 32
        const double *col = a.sched + 2 * ((slot >> 5) * static_cast<int64_t>(N) * 32 + (slot & 31));
        asm volatile("mov.b64 %0, %0;" : "+l"(col));

        auto prefetch_smem = [&](int q) {  // node records + spill values of chunk q
            const unsigned stg = static_cast<unsigned>(q & 1);
            const int b0 = lds_i(a_boff + 4u * q), b1 = lds_i(a_boff + 4u * (q + 1));
            const unsigned bs = a_blocks + stg * static_cast<unsigned>(BM) * 16u;
            DFSIM_CHECK(b1 - b0 <= BM, 8);
            for (int b = b0 + lane; b < b1; b += 32) cpa16(bs + 16u * static_cast<unsigned>(b - b0), a.t.blocks + 4 * static_cast<int64_t>(b));
            const int r0 = lds_i(a_soff + 4u * q), r1 = lds_i(a_soff + 4u * (q + 1));
            const unsigned ss = a_lane + static_cast<unsigned>(NS + static_cast<int>(stg) * RM) * 256u;
            for (int r = r0; r < r1; r += 32) {  // spill ids loaded by the lanes together, then broadcast
                const int my = r + lane < r1 ? static_cast<int>(lds_h(a_slist + 2u * (r + lane))) : 0;
                const int nr = r1 - r < 32 ? r1 - r : 32;
                for (int k = 0; k < nr; k++) {
                    const int id = __shfl_sync(DFSIM_FULL_MASK, my, k);
                    DFSIM_CHECK(id < a.t.n_long && r - r0 + k < RM, 7);
                    if (live) cpa8(ss + static_cast<unsigned>(r - r0 + k) * 256u, spill_warp + 32 * static_cast<int64_t>(id));
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        // window of chunk q: positions hi - K .. hi - 1 at register index p - (hi - K); positions
        // below 0 (the first chunk) are never read and load position 0 instead
        auto load_window = [&](int q, double (&w)[K][2]) {
            const int hi = lds_i(a_bounds + 4u * q);
#pragma unroll
            for (int i = 0; i < K; i++) {
                const int p = hi - K + i;
                ldg_pair(w[i], col + 64 * static_cast<int64_t>(p >= 0 ? p : 0));
            }
        };

        double wa[K][2], wb[K][2];
        double len = 0.0;
        int src = 0x7fffffff;
        prefetch_smem(0);
        load_window(0, wa);
        auto process = [&](int q, double (&w)[K][2], double (&wn)[K][2]) {
            if (q + 1 < NQ) {
                load_window(q + 1, wn);  // first: the window registers are claimed before any temporaries
                prefetch_smem(q + 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncwarp();
            const unsigned stg = static_cast<unsigned>(q & 1);
            const int hi = lds_i(a_bounds + 4u * q), lo = lds_i(a_bounds + 4u * (q + 1));
            const unsigned blk = a_blocks + stg * static_cast<unsigned>(BM) * 16u;
#pragma unroll
            for (int t = 0; t < K; t++) {
                if (t < hi - lo) {
                    const int p = hi - 1 - t;
                    DFSIM_CHECK(t < BM && p >= 0 && p < N, 8);
                    const uint4 r = lds_u4(blk + 16u * t);
                    const unsigned deg = r.y & 0xffu;
                    DFSIM_CHECK((r.z & 0xffffu) <= static_cast<unsigned>(NS + NST * RM) &&
                                    (r.z >> 16) <= static_cast<unsigned>(NS + NST * RM) &&
                                    (r.w & 0xffffu) <= static_cast<unsigned>(NS + NST * RM) &&
                                    (r.w >> 16) <= static_cast<unsigned>(NS + NST * RM),
                                6);  // row NS + NST * RM: the zero row
                    DFSIM_CHECK(!(r.x & kHasSlot) || (r.x & 0xfffu) < static_cast<unsigned>(NS), 5);
                    DFSIM_CHECK(!(r.x & kHasSpill) || (r.x >> 15) < static_cast<unsigned>(a.t.n_long), 7);
                    const double x0 = lds_d(row_lo(a_lane, r.z)), x1 = lds_d(row_hi(a_lane, r.z));
                    const double x2 = lds_d(row_lo(a_lane, r.w)), x3 = lds_d(row_hi(a_lane, r.w));
                    const double st = w[K - 1 - t][0], fi = w[K - 1 - t][1];  // position hi - 1 - t
                    const double m01 = x1 > x0 ? x1 : x0, m23 = x3 > x2 ? x3 : x2;
                    double best = m23 > m01 ? m23 : m01;
                    if (deg > 4) {
                        const unsigned ex = blk + 2u * (r.y >> 8);
#pragma unroll 1
                        for (unsigned j = 4; j < deg; j++) {  // rare (wide fan-outs): kept compact
                            DFSIM_CHECK((r.y >> 8) + (j - 4) < 8u * static_cast<unsigned>(BM), 8);
                            DFSIM_CHECK(lds_h(ex + 2u * (j - 4)) < static_cast<unsigned>(NS + NST * RM), 6);
                            const double x = lds_d(a_lane + 256u * lds_h(ex + 2u * (j - 4)));
                            best = x > best ? x : best;
                        }
                    }
                    const double sv = __dadd_rn(__dsub_rn(fi, st), best);  // finish - start (reporting.py:128)
                    if (r.x & kHasSlot) sts_d(a_lane + 256u * (r.x & 0xfffu), sv);
                    if (r.x & kHasSpill) spill_warp[32 * static_cast<int64_t>(r.x >> 15)] = sv;
                    if (r.x & kSource) {
                        const int rk = __ldg(a.t.rank_of_pos + p);
                        if (src == 0x7fffffff || sv > len || (sv == len && rk < src)) {
                            len = sv;
                            src = rk;
                        }
                    }
                }
            }
            __syncwarp();
        };
        for (int q = 0; q < NQ; q += 2) {  // two chunks per iteration: the window registers swap roles
            process(q, wa, wb);
            if (q + 1 < NQ) process(q + 1, wb, wa);
        }
        if (live) {
            a.cp_len[s] = src == 0x7fffffff ? 0.0 : len;
            if (a.cp_src) a.cp_src[s] = src == 0x7fffffff ? -1 : src;
        }
        __syncwarp();
    }
}

struct LaneShape {
    size_t table_bytes, region_bytes;
    int wpb;
};

// stages 2 / 3: pairs staged in shared memory; stages 0: pairs in registers (K = 8), two
// shared-memory stages for records and spill values
LaneShape lane_shape(const dfsim_cp_lane_tables *t, int /*stages: 0*/) {
    LaneShape s;
    const size_t nst = 2;  // shared-memory stages of node records and spill values
    s.table_bytes = ((static_cast<size_t>(t->n_chunks + 1) * 12 + static_cast<size_t>(t->n_spill_list) * 2 + 15) / 16) * 16;
    s.region_bytes = static_cast<size_t>(t->n_slots + nst * t->rmax + 1) * 256 +  // + the zero row
                     nst * static_cast<size_t>(t->block_max) * 16;
    const size_t budget = 227 * 1024 - 64;
    s.wpb = kRegWarps;
    while (s.wpb > 0 && s.table_bytes + s.wpb * s.region_bytes > budget) s.wpb--;
    return s;
}

}  // namespace

extern "C" int dfsim_cp_lanes_plan(int32_t n, const int32_t *succ_off, const int32_t *succ_pos, const uint8_t *is_source,
                                   int32_t K, int32_t rmax_min, int32_t stages, int32_t near_chunks, uint32_t *blocks,
                                   int32_t *block_off, int32_t *bounds, int32_t *spill_off, uint16_t *spill_list,
                                   int32_t *info) {
    if (n < 0 || !succ_off || !info || K < 1 || K > 16 || rmax_min < 1 || stages < 2 || stages > 4)
        return DFSIM_BAD_ARGUMENT;
    // a value read at most near_chunks - 1 chunks after its writer's stays in a slot; later reads go
    // through a spill row, whose prefetch (stages - 1 chunks ahead) must follow the write
    const int32_t far_at = near_chunks > stages ? near_chunks : stages;
    const int64_t E = n ? succ_off[n] : 0;
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
                if (q - chunk_of[v] >= far_at && stamp[v] != q) {
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
                if (q - chunk_of[v] >= far_at) {
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
    if (n_long >= (1 << 17) || n_long > 65536) return DFSIM_BAD_ARGUMENT;
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
    if (NS + stages * rmax + 1 > 65535) return DFSIM_BAD_ARGUMENT;
    // chunk blocks: records in processing order, then the rows of successors 5.., padded to 16 B
    int64_t unit = 0;  // 16-byte units written
    int32_t block_max = 1;
    for (int32_t c = 0; c < NQ; c++) {
        block_off[c] = static_cast<int32_t>(unit);
        const int32_t hi = bounds[c], lo = bounds[c + 1];
        uint32_t extra = static_cast<uint32_t>(hi - lo) * 8u;  // u16 index of the first extra row
        std::vector<uint16_t> ext;
        for (int32_t u = hi - 1; u >= lo; u--) {
            uint32_t *r = blocks + 4 * unit++;
            const int32_t deg = succ_off[u + 1] - succ_off[u];
            uint32_t x = 0;
            if (slot_of[u] >= 0) x |= static_cast<uint32_t>(slot_of[u]) | kHasSlot;
            if (is_source && is_source[u]) x |= kSource;
            if (spill_of[u] >= 0) x |= kHasSpill | (static_cast<uint32_t>(spill_of[u]) << 15);
            // unused fields name the warp's zero row (after the slots and spill stages): the kernels
            // load all four without branching, and max(0.0, .) comes for free (graph.py:465-468)
            const uint16_t zr = static_cast<uint16_t>(NS + stages * rmax);
            uint16_t row[4] = {zr, zr, zr, zr};
            for (int32_t k = 0; k < deg; k++) {
                const int64_t j = succ_off[u] + k;
                const int32_t rv = far_idx[j] >= 0 ? NS + (chunk_of[u] % stages) * rmax + far_idx[j] : slot_of[succ_pos[j]];
                if (rv < 0 || rv >= 65536) return DFSIM_BAD_ARGUMENT;
                if (k < 4) row[k] = static_cast<uint16_t>(rv); else ext.push_back(static_cast<uint16_t>(rv));
            }
            const uint32_t off = deg > 4 ? extra + static_cast<uint32_t>(ext.size()) - static_cast<uint32_t>(deg - 4) : 0u;
            if (off >= (1u << 24)) return DFSIM_BAD_ARGUMENT;
            r[0] = x;
            r[1] = static_cast<uint32_t>(deg) | (off << 8);
            r[2] = row[0] | (static_cast<uint32_t>(row[1]) << 16);
            r[3] = row[2] | (static_cast<uint32_t>(row[3]) << 16);
        }
        const size_t eu = (ext.size() + 7) / 8;  // extra rows, 8 per 16-byte unit
        uint16_t *eb = reinterpret_cast<uint16_t *>(blocks + 4 * unit);
        for (size_t i = 0; i < eu * 8; i++) eb[i] = i < ext.size() ? ext[i] : 0;
        unit += static_cast<int64_t>(eu);
        block_max = std::max(block_max, static_cast<int32_t>(unit - block_off[c]));
        if (unit >= (int64_t(1) << 31)) return DFSIM_BAD_ARGUMENT;
    }
    block_off[NQ] = static_cast<int32_t>(unit);
    info[0] = NQ;
    info[1] = NS;
    info[2] = rmax;
    info[3] = n_long;
    info[4] = static_cast<int32_t>(slist.size());
    info[5] = block_max;
    return DFSIM_OK;
}

extern "C" int32_t dfsim_critical_path_lanes_capacity(const dfsim_cp_lane_tables *t, int32_t stages) {
    if (!t || t->n_chunks <= 0 || stages != 0 || t->chunk_positions != 8) return 0;
    return lane_shape(t, stages).wpb;
}

extern "C" int dfsim_critical_path_lanes(dfsim_ctx *ctx, const dfsim_cp_lane_tables *t, int32_t stages, int64_t n_sims,
                                         const int64_t *cand_of_slot, const double *sched, double *cp_len,
                                         int32_t *cp_src) {
    return dfsim_critical_path_lanes_ex(ctx, t, stages, n_sims, nullptr, cand_of_slot, 0, sched, cp_len, cp_src);
}

extern "C" int dfsim_critical_path_lanes_ex(dfsim_ctx *ctx, const dfsim_cp_lane_tables *t, int32_t stages,
                                            int64_t n_sims, const int64_t *slots, const int64_t *cand_of_slot,
                                            int32_t max_warps, const double *sched, double *cp_len, int32_t *cp_src) {
    if (!ctx || !t) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, sched && cp_len, "sched and cp_len are required");
    DFSIM_ARG_CHECK(ctx, (reinterpret_cast<uintptr_t>(sched) & 15) == 0, "sched must be 16-byte aligned");
    DFSIM_ARG_CHECK(ctx, stages == 0 && t->chunk_positions == 8, "stages 0 (register windows) with chunk_positions 8");
    DFSIM_ARG_CHECK(ctx, t->n_nodes > 0 && t->n_chunks > 0 && t->n_slots >= 1 && t->n_slots < 4096 && t->rmax >= 1 &&
                         t->n_spill_list >= 0 && t->block_max >= 1,
                    "inconsistent lane tables");
    if (n_sims <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const LaneShape shape = lane_shape(t, stages);
    DFSIM_ARG_CHECK(ctx, shape.wpb >= 1, "lane tables do not fit in shared memory");
    // as many warps as the batch needs, spread over the SMs
    const int64_t warps = (n_sims + 31) / 32;
    int wpb = shape.wpb;
    if (max_warps > 0 && max_warps < wpb) wpb = max_warps;  // leaves room for a co-resident kernel
    const int64_t per_sm = (warps + ctx->num_sms - 1) / ctx->num_sms;
    if (per_sm < wpb) wpb = static_cast<int>(per_sm < 1 ? 1 : per_sm);
    const size_t smem = shape.table_bytes + static_cast<size_t>(wpb) * shape.region_bytes;
    const int grid = static_cast<int>(std::min<int64_t>((warps + wpb - 1) / wpb, ctx->num_sms));
    void *p = nullptr;
    const size_t spill_bytes = static_cast<size_t>(grid) * wpb * std::max(t->n_long, 1) * 32 * 8;
    int rc = dfsim_scratch(ctx, spill_bytes + 256, &p);
    if (rc) return rc;
    int32_t *counter = reinterpret_cast<int32_t *>(static_cast<unsigned char *>(p) + spill_bytes);
    DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(counter, 0, sizeof(int32_t), ctx->stream));
    LaneArgs a;
    a.task_counter = counter;
    a.slots = slots;
    a.cand = cand_of_slot;
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
        const int rc = dfsim_after_launch(ctx, "k_critical_path_lanes");
        if (rc) {  // say what was asked for
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kern);
            ctx->last_error += " (grid " + std::to_string(grid) + ", block " + std::to_string(wpb * 32) + ", smem " +
                               std::to_string(smem) + ", registers " + std::to_string(fa.numRegs) + ", max threads " +
                               std::to_string(fa.maxThreadsPerBlock) + ")";
        }
        return rc;
    };
    return launch(k_critical_path_lanes_reg<8>);
}
