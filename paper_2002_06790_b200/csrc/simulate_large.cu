// K3 large: the exact event loop (engine.py:96-146) for graphs whose per-candidate
// state cannot live in shared memory (C5: 1M nodes), one warp per candidate.
//
// With a few hundred candidates per GPU each candidate is one long serial chain of
// event iterations (~N of them), so the design goal is the latency of one iteration,
// not bandwidth.  Against the exact-capacity engine (simulate.cu, global mode) it
// removes every dependent global round trip from the iteration:
//   * FIFO rings of node ids in shared memory (4 bytes an entry, so most of the SM's
//     256 KB stays L1 for the counter rows).  When a device starts a node it also loads
//     the duration of its next ring entry (whose place at the head is final), so the
//     next pop rarely waits on memory.  Ring occupancy is checked before every pop (a
//     device only gains entries until its next pop); an overflowed candidate is re-run
//     by the exact engine.
//   * A start loads the node's 32-byte successor record (range + the first kPre
//     successors with their devices, built once per launch).  At finish the relax step
//     loads the carried successors' counters together (longer lists fall back to direct
//     loads) and prefetches each newly ready node's duration into L2 for its pop.
//   * One finishing device per iteration (the common case) relaxes alone with plain
//     counter and ring-tail updates; ties between devices take the combining path.
//   * Dependency counters are plain byte/short loads and stores in a global row per
//     warp, L1-resident for the active frontier.  Lanes relaxing the same node in one
//     iteration are combined with __match_any_sync (the leader subtracts the group
//     size), so no atomics are needed: one warp owns the row.
// The iteration itself is the reference's: now = min finish (exact, via redux over the
// IEEE bits of non-negative doubles), every device finishing at `now` releases its
// successors, each device's newly ready nodes are appended in rank order, idle devices
// pop at `now` (start == now).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "internal.cuh"

int dfsim_simulate_exact_flagged(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                                 int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                                 int32_t *n_placed, const int32_t *redo);

namespace {

constexpr int kPre = 4;  // successors carried in a node's prefetch record

struct LargeArgs {
    int32_t N, D;
    const int32_t *succ_off, *succ_idx, *indeg, *device, *sources;
    int32_t n_sources;
    int64_t S;
    const double *dur;
    int64_t dur_stride;
    double *start, *finish, *makespan, *busy;
    int32_t *n_placed;
    int32_t *redo;             // [S] 1 when the candidate overflowed a ring
    const uint4 *srec;         // [N][2] successor record: {j0, deg, s0, s1}, {s2, s3, -, -}; s = m | dev << 27
    unsigned char *gcnt;       // counters, cnt_bytes per resident warp
    int64_t cnt_bytes;
    int32_t qcap;              // ring entries per device (power of two)
    int32_t warp_smem;         // bytes of shared state per warp
};

// One 32-byte record per node: its successor range and the first kPre successors with
// their devices, so a start issues one load and the finish needs no dependent loads.
__global__ void k_successor_records(int32_t N, const int32_t *succ_off, const int32_t *succ_idx,
                                    const int32_t *device, uint4 *srec) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
        const int32_t j0 = succ_off[v], deg = succ_off[v + 1] - j0;
        unsigned pk[kPre];
#pragma unroll
        for (int k = 0; k < kPre; k++) {
            pk[k] = 0;
            if (k < deg) {
                const int32_t m = succ_idx[j0 + k];
                pk[k] = static_cast<unsigned>(m) | (static_cast<unsigned>(device[m]) << 27);
            }
        }
        srec[2 * v] = make_uint4(static_cast<unsigned>(j0), static_cast<unsigned>(deg), pk[0], pk[1]);
        srec[2 * v + 1] = make_uint4(pk[2], pk[3], 0u, 0u);
    }
}

__device__ __forceinline__ double warp_min_nonneg(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned hi = __reduce_min_sync(DFSIM_FULL_MASK, static_cast<unsigned>(b >> 32));
    const unsigned lo = __reduce_min_sync(DFSIM_FULL_MASK, static_cast<unsigned>(b >> 32) == hi
                                                               ? static_cast<unsigned>(b) : 0xffffffffu);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo));
}

template <typename CT>
__global__ void __launch_bounds__(256) k_simulate_large(LargeArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int N = a.N, D = a.D, QC = a.qcap;
    const unsigned QM = static_cast<unsigned>(QC - 1);
    unsigned char *ws = smem + static_cast<size_t>(wib) * a.warp_smem;
    int32_t *tails = reinterpret_cast<int32_t *>(ws);                  // [32]
    int32_t *rnode = reinterpret_cast<int32_t *>(ws + 128);            // [D][QC]
    CT *cnt = reinterpret_cast<CT *>(a.gcnt + (static_cast<int64_t>(blockIdx.x) * wpb + wib) * a.cnt_bytes);
    asm volatile("mov.b64 %0, %0;" : "+l"(cnt));

    for (int64_t s = static_cast<int64_t>(blockIdx.x) * wpb + wib; s < a.S; s += static_cast<int64_t>(gridDim.x) * wpb) {
        const double *dur = a.dur + s * a.dur_stride;
        double *out_s = a.start ? a.start + s * N : nullptr;
        double *out_f = a.finish ? a.finish + s * N : nullptr;
        asm volatile("mov.b64 %0, %0;" : "+l"(dur));  // row bases stay in registers
        asm volatile("mov.b64 %0, %0;" : "+l"(out_s));
        asm volatile("mov.b64 %0, %0;" : "+l"(out_f));
        for (int v = lane; v < N; v += 32) cnt[v] = static_cast<CT>(__ldg(a.indeg + v));
        if (lane < D) tails[lane] = 0;
        __syncwarp();
        // sources in rank order (engine.py:111-114)
        for (int b = 0; b < a.n_sources; b += 32) {
            const int i = b + lane;
            const bool has = i < a.n_sources;
            const int v = has ? __ldg(a.sources + i) : 0;
            const int dv = has ? __ldg(a.device + v) : 32 + lane;
            const unsigned peers = __match_any_sync(DFSIM_FULL_MASK, dv);
            const int base = has ? tails[dv] : 0;
            __syncwarp();
            if (has) {
                const int p = base + __popc(peers & lanemask_lt());
                rnode[dv * QC + (p & QM)] = v;
                if ((peers & lanemask_lt()) == 0) tails[dv] = base + __popc(peers);
            }
            __syncwarp();
        }
        bool ovf = lane < D && tails[lane] > QC;

        unsigned head = 0;
        bool running = false;
        uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);  // successor record of the running node
        int nx_v = -1;      // the device's next ring entry, whose duration is already in flight
        double nx_d = 0.0;
        double run_f = 0.0, busy_sum = 0.0, span = 0.0, now = 0.0;
        int placed = 0;
        auto succ_of = [&](int k) -> unsigned { return k == 0 ? r0.z : (k == 1 ? r0.w : (k == 2 ? r1.x : r1.y)); };
        auto start_idle = [&]() {
            const int t = lane < D ? tails[lane] : 0;
            if (lane < D && !running && !ovf && static_cast<int>(head) < t) {
                ovf = static_cast<unsigned>(t) - head > static_cast<unsigned>(QC);
                if (ovf) return;  // stop the device: the candidate is re-run exactly
                const int v = rnode[lane * QC + static_cast<int>(head & QM)];
                // the duration was loaded when the previous node started, unless this entry
                // arrived (or was re-sorted to the head) since
                const double d0 = v == nx_v ? nx_d : __ldcg(dur + v);
                const double d = d0 >= 0.0 ? d0 : 0.0;  // failing rows (NaN / negative) still terminate
                const double f = __dadd_rn(now, d);
                head++;
                if (out_s) {
                    __stcs(out_s + v, now);
                    __stcs(out_f + v, f);
                }
                running = true;
                run_f = f;
                busy_sum = __dadd_rn(busy_sum, __dsub_rn(f, now));
                if (f > span) span = f;
                placed++;
                r0 = __ldg(a.srec + 2 * static_cast<int64_t>(v));
                r1 = __ldg(a.srec + 2 * static_cast<int64_t>(v) + 1);
                nx_v = -1;
                if (static_cast<int>(head) < t) {  // the device's next node: its duration and record now
                    nx_v = rnode[lane * QC + static_cast<int>(head & QM)];
                    nx_d = __ldcg(dur + nx_v);  // L2 only: L1 stays with the counters and records
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.srec + 2 * static_cast<int64_t>(nx_v)));
                }
            } else if (lane < D && running && nx_v < 0 && static_cast<int>(head) < t) {
                // an entry arrived while this device runs: its place at the head is final
                // (later arrivals sort behind it), so load its duration now
                nx_v = rnode[lane * QC + static_cast<int>(head & QM)];
                nx_d = __ldcg(dur + nx_v);
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.srec + 2 * static_cast<int64_t>(nx_v)));
            }
        };

        start_idle();
        while (__any_sync(DFSIM_FULL_MASK, running)) {
            now = warp_min_nonneg(running ? run_f : __longlong_as_double(0x7ff0000000000000LL));
            const bool done = running && run_f == now;
            const int seg_lo = lane < D ? tails[lane] : 0;
            const unsigned dm = __ballot_sync(DFSIM_FULL_MASK, done);
            if (done) running = false;
            if ((dm & (dm - 1)) == 0) {
                // one device finished (the common case): it alone updates counters and rings
                if (done) {
                    const int deg = static_cast<int>(r0.y);
                    // the carried successors' counters are loaded together (one latency, not
                    // deg); a repeated successor (duplicate edge) sees the earlier decrements
                    int cpre[kPre];
#pragma unroll
                    for (int k = 0; k < kPre; k++)
                        if (k < deg) cpre[k] = static_cast<int>(cnt[succ_of(k) & 0x7ffffffu]);
#pragma unroll
                    for (int k = 0; k < kPre; k++) {
                        if (k < deg) {
                            const unsigned e = succ_of(k);
                            const int m = static_cast<int>(e & 0x7ffffffu), dv = static_cast<int>(e >> 27);
                            DFSIM_CHECK(m < N && dv < D && cpre[k] >= 1, 12);  // a released node's counter was >= 1
                            int c = cpre[k];
#pragma unroll
                            for (int j = 0; j < k; j++) c -= (succ_of(j) & 0x7ffffffu) == static_cast<unsigned>(m);
                            cnt[m] = static_cast<CT>(c - 1);
                            if (c == 1) {
                                const int p = tails[dv];
                                tails[dv] = p + 1;
                                rnode[dv * QC + (p & QM)] = m;
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(dur + m));  // read at its pop
                            }
                        }
                    }
                    for (int k = kPre; k < deg; k++) {
                        const int m = __ldg(a.succ_idx + static_cast<int>(r0.x) + k);
                        DFSIM_CHECK(m >= 0 && m < N, 12);
                        const int dv = __ldg(a.device + m);
                        DFSIM_CHECK(dv >= 0 && dv < D, 12);
                        const int c = static_cast<int>(cnt[m]);
                        cnt[m] = static_cast<CT>(c - 1);
                        if (c == 1) {
                            const int p = tails[dv];
                            tails[dv] = p + 1;
                            rnode[dv * QC + (p & QM)] = m;
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(dur + m));  // read at its pop
                        }
                    }
                }
            } else {
                // several devices finished at `now`: relax in rounds, lanes releasing the same
                // node combined by __match_any_sync (the leader subtracts the group size)
                const int deg = done ? static_cast<int>(r0.y) : 0;
                const int rounds = __reduce_max_sync(DFSIM_FULL_MASK, static_cast<unsigned>(deg));
                for (int r = 0; r < rounds; r++) {
                    const bool act = r < deg;
                    const unsigned am = __ballot_sync(DFSIM_FULL_MASK, act);
                    if (act) {
                        unsigned e;
                        if (r < kPre) {
                            e = succ_of(r);
                        } else {
                            const int m = __ldg(a.succ_idx + static_cast<int>(r0.x) + r);
                            e = static_cast<unsigned>(m) | (static_cast<unsigned>(__ldg(a.device + m)) << 27);
                        }
                        const int m = static_cast<int>(e & 0x7ffffffu), dv = static_cast<int>(e >> 27);
                        DFSIM_CHECK(m < N && dv < D, 12);
                        const unsigned grp = __match_any_sync(am, m);
                        if ((grp & lanemask_lt()) == 0) {
                            const int k = __popc(grp);
                            const int c = static_cast<int>(cnt[m]);
                            cnt[m] = static_cast<CT>(c - k);
                            if (c == k) {
                                const int p = atomicAdd(tails + dv, 1);
                                rnode[dv * QC + (p & QM)] = m;
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(dur + m));  // read at its pop
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
            const int seg_hi = lane < D ? tails[lane] : 0;
            if (seg_hi - seg_lo > 1) {  // enqueue(sorted(newly_ready)) (engine.py:139-142)
                for (int i = seg_lo + 1; i < seg_hi; i++) {
                    const int xs = lane * QC + (i & QM);
                    const int x = rnode[xs];
                    int j = i - 1;
                    while (j >= seg_lo && rnode[lane * QC + (j & QM)] > x) {
                        rnode[lane * QC + ((j + 1) & QM)] = rnode[lane * QC + (j & QM)];
                        j--;
                    }
                    rnode[lane * QC + ((j + 1) & QM)] = x;
                }
            }
            __syncwarp();
            start_idle();
        }
        const bool bad = __any_sync(DFSIM_FULL_MASK, ovf);
        const double ms = warp_max_f64(span);
        const int total = warp_sum_i32(placed);
        if (lane == 0) {
            a.makespan[s] = ms;
            if (a.n_placed) a.n_placed[s] = total;
            a.redo[s] = bad ? 1 : 0;
        }
        if (a.busy && lane < D) a.busy[s * D + lane] = busy_sum;
        __syncwarp();
    }
}

}  // namespace

// Called by dfsim_simulate_batch_ex for graphs beyond the shared-memory engine with the
// plain [S][N] layout.  Returns DFSIM_OK after queueing the kernel and the exact re-run
// of any overflowed candidate (stream-ordered; no host synchronisation).
int dfsim_simulate_large(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                         int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                         int32_t *n_placed) {
    const int32_t N = g->n_nodes, D = g->n_devices;
    const int cbytes = g->max_indeg < 255 ? 1 : (g->max_indeg < 65535 ? 2 : 4);
    int wpb = static_cast<int>(std::min<int64_t>(8, std::max<int64_t>(1, (n_sims + ctx->num_sms - 1) / ctx->num_sms)));
    const int budget = 220 * 1024 / wpb;
    // small rings: the rest of the SM's 256 KB stays L1 for the counter rows' active frontier
    static const int kQcapMax = [] {  // ring entries per device; DFSIM_LARGE_QCAP overrides (power of two)
        const char *e = std::getenv("DFSIM_LARGE_QCAP");
        const int v = e ? std::atoi(e) : 0;
        return v >= 16 && (v & (v - 1)) == 0 ? v : 512;
    }();
    int qcap = kQcapMax;
    while (qcap > 16 && 128 + static_cast<int64_t>(std::max(D, 1)) * qcap * 4 > budget) qcap >>= 1;
    const int warp_smem = (128 + std::max(D, 1) * qcap * 4 + 15) / 16 * 16;
    const int64_t want = (n_sims + wpb - 1) / wpb;
    const int grid = static_cast<int>(std::min<int64_t>(want, ctx->num_sms));
    const int64_t cnt_bytes = (static_cast<int64_t>(N) * cbytes + 127) / 128 * 128;
    void *p = nullptr, *redo = nullptr;
    const size_t rec_off = static_cast<size_t>(grid) * wpb * cnt_bytes;
    int rc = dfsim_scratch(ctx, rec_off + 32 * static_cast<size_t>(std::max(N, 1)) + 256, &p);
    if (rc) return rc;
    uint4 *srec = reinterpret_cast<uint4 *>(static_cast<unsigned char *>(p) + (rec_off + 255) / 256 * 256);
    k_successor_records<<<std::max(1, std::min((N + 255) / 256, ctx->num_sms * 8)), 256, 0, ctx->stream>>>(
        N, g->succ_off, g->succ_idx, g->device, srec);
    rc = dfsim_after_launch(ctx, "k_successor_records");
    if (rc) return rc;
    rc = dfsim_aux(ctx, sizeof(int32_t) * n_sims, &redo);
    if (rc) return rc;
    LargeArgs a;
    a.N = N; a.D = D;
    a.succ_off = g->succ_off; a.succ_idx = g->succ_idx; a.indeg = g->indeg; a.device = g->device;
    a.sources = g->sources; a.n_sources = g->n_sources;
    a.S = n_sims; a.dur = dur; a.dur_stride = dur_stride;
    a.start = start; a.finish = finish; a.makespan = makespan; a.busy = busy; a.n_placed = n_placed;
    a.gcnt = static_cast<unsigned char *>(p);
    a.srec = srec;
    a.redo = static_cast<int32_t *>(redo);
    a.cnt_bytes = cnt_bytes;
    a.qcap = qcap;
    a.warp_smem = warp_smem;
    const size_t smem = static_cast<size_t>(wpb) * warp_smem;
    auto launch = [&](auto kern) -> int {
        DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 static_cast<int>((smem * 100 + 228 * 1024 - 1) / (228 * 1024))));
        kern<<<grid, wpb * 32, smem, ctx->stream>>>(a);
        return dfsim_after_launch(ctx, "k_simulate_large");
    };
    rc = cbytes == 1 ? launch(k_simulate_large<uint8_t>)
                     : (cbytes == 2 ? launch(k_simulate_large<uint16_t>) : launch(k_simulate_large<uint32_t>));
    if (rc) return rc;
    // exact re-run of ring overflows (flags in ctx->aux survive the exact engine's scratch growth)
    return dfsim_simulate_exact_flagged(ctx, g, n_sims, dur, dur_stride, start, finish, makespan, busy, n_placed,
                                        a.redo);
}
