// K3: batched event-driven list scheduling -- the reference's engine.simulate
// (pkg/src/dfsim/engine.py:96-146) and _finalize (69-93), one warp per strategy.
//
// Mapping: lane d owns device rank d (D <= 32; beyond that lane l owns l, l + 32, ...): its running node, its finish
// time, its FIFO head and its busy accumulator live in registers.  The per-strategy
// dependency counters (packed 8/16/32-bit, decremented with 32-bit shared-memory
// atomics) and the per-device FIFOs (one segment of queue_off[d]..queue_off[d+1]
// per device, exact capacity) live in shared memory, or in a global scratch slot
// per resident warp when N is too large for shared memory.
//
// One loop iteration == one pass of the reference's `while events` loop:
//   now   = min over running devices of finish           (warp min, exact)
//   done  = running && finish == now                     (exact ==, engine.py:131-134)
//   done lanes decrement their successors' counters; a counter reaching zero
//   appends the node to its device FIFO segment; each segment's new tail is then
//   sorted by node rank (== enqueue(sorted(newly_ready)), engine.py:111-114)
//   idle lanes pop their FIFO head: start = now, finish = now + dur (engine.py:116-125)
// start == max(device_free, ready) == now always holds, so it is
// written as `now`.  busy[d] accumulates finish-start in device execution order,
// which equals entry order for every non-zero term ("busy").
#include <cuda_runtime.h>

#include "internal.cuh"

namespace {

struct SimArgs {
    int32_t N, D;
    const int32_t *succ_off, *succ_idx, *indeg, *device, *sources, *queue_off;
    int32_t n_sources;
    int64_t S;
    const double *dur;
    int64_t dur_stride;
    double *start, *finish, *makespan, *busy;
    int32_t *n_placed;
    unsigned char *gscratch;  // global-mode state, per_warp bytes per resident warp
    int64_t per_warp;         // bytes of counters+queue per warp (global or shared)
    int32_t cnt_words;        // u32 words of packed counters
    const int32_t *pos;       // optional output column per node
    const int64_t *out_rows;  // optional output row per simulated row
    int32_t interleaved;      // start points at (start, finish) pairs; finish unused
    const int32_t *redo;      // optional: simulate only rows s with redo[s] != 0
};

template <int kBits>
struct Counter {
    static constexpr int kPer = 32 / kBits;
    static constexpr unsigned kMask = kBits == 32 ? 0xffffffffu : ((1u << kBits) - 1u);
    // Decrement counter v; true when it reaches zero.
    __device__ __forceinline__ static bool dec(unsigned *words, int v) {
        const int shift = (v % kPer) * kBits;
        unsigned old = atomicSub(words + v / kPer, 1u << shift);
        return ((old >> shift) & kMask) == 1u;
    }
    __device__ __forceinline__ static void init(unsigned *words, int nwords, const int32_t *indeg, int N, int lane) {
        for (int w = lane; w < nwords; w += 32) {
            unsigned word = 0;
#pragma unroll
            for (int i = 0; i < kPer; i++) {
                int v = w * kPer + i;
                if (v < N) word |= (static_cast<unsigned>(__ldg(indeg + v)) & kMask) << (i * kBits);
            }
            words[w] = word;
        }
    }
};

// Sort q[lo, hi) ascending (node ranks are distinct).  Short runs: the owning
// lane alone (insertion sort); long runs: whole-warp odd-even transposition.
template <typename QT>
__device__ __forceinline__ void insertion_sort(QT *q, int lo, int hi) {
    for (int i = lo + 1; i < hi; i++) {
        QT x = q[i];
        int j = i - 1;
        while (j >= lo && q[j] > x) { q[j + 1] = q[j]; j--; }
        q[j + 1] = x;
    }
}

template <typename QT>
__device__ void warp_sort(QT *q, int lo, int hi, int lane) {
    const int L = hi - lo;
    for (int r = 0; r < L; r++) {
        for (int i = lo + (r & 1) + 2 * lane; i + 1 < hi; i += 64) {
            QT a = q[i], b = q[i + 1];
            if (a > b) { q[i] = b; q[i + 1] = a; }
        }
        __syncwarp();
    }
}

constexpr int kShortRun = 24;

// kV devices per lane (device d = lane + 32 k): kV = 1 covers D <= 32, larger kV the
// wide device sets of big parameter-server or data-parallel expansions (D <= 32 kV).
template <int kBits, typename QT, bool kShared, int kV>
__global__ void __launch_bounds__(256) k_simulate(SimArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int N = a.N, D = a.D;

    int32_t *tails = reinterpret_cast<int32_t *>(smem) + wib * 32 * kV;  // per-warp FIFO tails
    unsigned char *state = kShared ? smem + wpb * 32 * kV * sizeof(int32_t) + wib * a.per_warp
                                   : a.gscratch + (static_cast<int64_t>(blockIdx.x) * wpb + wib) * a.per_warp;
    unsigned *cnt = reinterpret_cast<unsigned *>(state);
    QT *q = reinterpret_cast<QT *>(state + static_cast<int64_t>(a.cnt_words) * 4);
    int my_qoff[kV];
#pragma unroll
    for (int k = 0; k < kV; k++) my_qoff[k] = lane + 32 * k < D ? __ldg(a.queue_off + lane + 32 * k) : 0;

    for (int64_t s = static_cast<int64_t>(blockIdx.x) * wpb + wib; s < a.S; s += static_cast<int64_t>(gridDim.x) * wpb) {
        if (a.redo && !a.redo[s]) continue;
        const double *dur = a.dur + s * a.dur_stride;
        const int64_t row = a.out_rows ? a.out_rows[s] : s;
        // interleaved 1: (start, finish) pairs by row; 2: pairs in 32-candidate tiles (fused layout)
        double *out_start = !a.start ? nullptr
                            : a.interleaved == 2 ? a.start + 2 * ((row >> 5) * N * 32 + (row & 31))
                                                 : a.start + row * N * (a.interleaved ? 2 : 1);
        double *out_finish = a.interleaved ? (out_start ? out_start + 1 : nullptr) : (a.finish ? a.finish + row * N : nullptr);
        const int ostride = a.interleaved == 2 ? 64 : a.interleaved ? 2 : 1;

        Counter<kBits>::init(cnt, a.cnt_words, a.indeg, N, lane);
        int head[kV];
#pragma unroll
        for (int k = 0; k < kV; k++) {
            if (lane + 32 * k < D) tails[lane + 32 * k] = my_qoff[k];
            head[k] = my_qoff[k];
        }
        __syncwarp();

        // sources, already in rank order: append chunk by chunk (engine.py:111-114)
        for (int b = 0; b < a.n_sources; b += 32) {
            const int i = b + lane;
            const bool has = i < a.n_sources;
            const int v = has ? __ldg(a.sources + i) : 0;
            const int dv = has ? __ldg(a.device + v) : 32 * kV + lane;
            const unsigned peers = __match_any_sync(DFSIM_FULL_MASK, dv);
            const int base = has ? tails[dv] : 0;
            __syncwarp();
            if (has) {
                q[base + __popc(peers & lanemask_lt())] = static_cast<QT>(v);
                if ((peers & lanemask_lt()) == 0) tails[dv] = base + __popc(peers);
            }
            __syncwarp();
        }

        bool running[kV];
        int run_v[kV];
        double run_f[kV], busy_sum[kV];
        double span = 0.0, now = 0.0;
        int placed = 0;
#pragma unroll
        for (int k = 0; k < kV; k++) {
            running[k] = false;
            run_v[k] = 0;
            run_f[k] = 0.0;
            busy_sum[k] = 0.0;
        }

        // start_idle_devices (engine.py:116-125) at `now`
        auto start_idle = [&]() {
#pragma unroll
            for (int k = 0; k < kV; k++) {
                const int d = lane + 32 * k;
                if (d < D && !running[k] && head[k] < tails[d]) {
                    const int v = q[head[k]++];
                    // a failing row (estimate status >= 253: NaN / negative value) still terminates;
                    // its exception is raised from the estimate status, never from this schedule
                    const double dv = __ldg(dur + v);
                    const double f = __dadd_rn(now, dv >= 0.0 ? dv : 0.0);
                    if (out_start) {
                        const int col = (a.pos ? __ldg(a.pos + v) : v) * ostride;
                        out_start[col] = now;
                        out_finish[col] = f;
                    }
                    running[k] = true;
                    run_v[k] = v;
                    run_f[k] = f;
                    busy_sum[k] = __dadd_rn(busy_sum[k], __dsub_rn(f, now));
                    if (f > span) span = f;
                    placed++;
                }
            }
        };
        auto any_running = [&]() {
            bool r = false;
#pragma unroll
            for (int k = 0; k < kV; k++) r |= running[k];
            return r;
        };

        start_idle();
        while (__any_sync(DFSIM_FULL_MASK, any_running())) {
            double mine = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
            for (int k = 0; k < kV; k++)
                if (running[k] && run_f[k] < mine) mine = run_f[k];
            now = warp_min_f64(mine);
            int seg_lo[kV];
#pragma unroll
            for (int k = 0; k < kV; k++) seg_lo[k] = lane + 32 * k < D ? tails[lane + 32 * k] : 0;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kV; k++) {
                if (running[k] && run_f[k] == now) {
                    running[k] = false;
                    const int e1 = __ldg(a.succ_off + run_v[k] + 1);
                    for (int j = __ldg(a.succ_off + run_v[k]); j < e1; j++) {
                        const int m = __ldg(a.succ_idx + j);
                        if (Counter<kBits>::dec(cnt, m)) {
                            const int pos = atomicAdd(tails + __ldg(a.device + m), 1);
                            q[pos] = static_cast<QT>(m);
                        }
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kV; k++) {
                const int seg_hi = lane + 32 * k < D ? tails[lane + 32 * k] : 0;
                if (seg_hi - seg_lo[k] > 1 && seg_hi - seg_lo[k] <= kShortRun) insertion_sort(q, seg_lo[k], seg_hi);
                unsigned long_runs = __ballot_sync(DFSIM_FULL_MASK, seg_hi - seg_lo[k] > kShortRun);
                while (long_runs) {
                    const int d = __ffs(long_runs) - 1;
                    long_runs &= long_runs - 1;
                    const int lo = __shfl_sync(DFSIM_FULL_MASK, seg_lo[k], d);
                    const int hi = __shfl_sync(DFSIM_FULL_MASK, seg_hi, d);
                    warp_sort(q, lo, hi, lane);
                }
            }
            __syncwarp();
            start_idle();
        }

        const double ms = warp_max_f64(span);
        const int total = warp_sum_i32(placed);
        if (lane == 0) {
            a.makespan[row] = ms;
            if (a.n_placed) a.n_placed[row] = total;
        }
#pragma unroll
        for (int k = 0; k < kV; k++)
            if (a.busy && lane + 32 * k < D) a.busy[row * D + lane + 32 * k] = busy_sum[k];
        __syncwarp();
    }
}

template <int kBits, typename QT, int kV>
int launch_v(dfsim_ctx *ctx, SimArgs &a, bool shared_mode, int wpb, int grid, size_t smem) {
    if (shared_mode) {
        auto kern = k_simulate<kBits, QT, true, kV>;
        DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, wpb * 32, smem, ctx->stream>>>(a);
    } else {
        k_simulate<kBits, QT, false, kV><<<grid, wpb * 32, smem, ctx->stream>>>(a);
    }
    return dfsim_after_launch(ctx, "k_simulate");
}

constexpr int kWideV = 8;  // devices per lane of the wide-device instantiation (D <= 256)

template <int kBits, typename QT>
int launch_bits(dfsim_ctx *ctx, SimArgs &a, bool shared_mode, int wpb, int grid, size_t smem) {
    return a.D <= 32 ? launch_v<kBits, QT, 1>(ctx, a, shared_mode, wpb, grid, smem)
                     : launch_v<kBits, QT, kWideV>(ctx, a, shared_mode, wpb, grid, smem);
}

}  // namespace

int dfsim_simulate_large(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                         int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                         int32_t *n_placed);
static int simulate_exact(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                          int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                          int32_t *n_placed, const int32_t *pos, const int64_t *out_rows, int32_t interleaved,
                          const int32_t *redo, bool allow_large);

extern "C" int dfsim_simulate_batch(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                                    int64_t dur_stride, double *start, double *finish, double *makespan,
                                    double *busy, int32_t *n_placed) {
    return dfsim_simulate_batch_ex(ctx, g, n_sims, dur, dur_stride, start, finish, makespan, busy, n_placed, nullptr,
                                   nullptr, 0);
}

static int simulate_exact(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                          int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                          int32_t *n_placed, const int32_t *pos, const int64_t *out_rows, int32_t interleaved,
                          const int32_t *redo, bool allow_large) {
    if (!ctx || !g) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, g->n_nodes >= 0 && n_sims >= 0, "negative sizes");
    DFSIM_ARG_CHECK(ctx, g->n_devices >= 0 && g->n_devices <= 32 * kWideV, "the warp engine supports at most 256 devices");
    DFSIM_ARG_CHECK(ctx, makespan != nullptr, "makespan output is required");
    DFSIM_ARG_CHECK(ctx, interleaved || (start == nullptr) == (finish == nullptr), "start and finish go together");
    DFSIM_ARG_CHECK(ctx, dur_stride == 0 || dur_stride >= g->n_nodes, "dur_stride < n_nodes");
    if (n_sims == 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));

    const int32_t N = g->n_nodes;
    DFSIM_ARG_CHECK(ctx, g->max_indeg >= 0, "max_indeg must be set");
    const int bits = g->max_indeg < 255 ? 8 : (g->max_indeg < 65535 ? 16 : 32);

    SimArgs a;
    a.N = N; a.D = g->n_devices;
    a.succ_off = g->succ_off; a.succ_idx = g->succ_idx; a.indeg = g->indeg; a.device = g->device;
    a.sources = g->sources; a.queue_off = g->queue_off; a.n_sources = g->n_sources;
    a.S = n_sims; a.dur = dur; a.dur_stride = dur_stride;
    a.start = start; a.finish = finish; a.makespan = makespan; a.busy = busy; a.n_placed = n_placed;
    a.pos = pos; a.out_rows = out_rows; a.interleaved = interleaved; a.redo = redo;
    const int per = 32 / bits;
    a.cnt_words = (N + per - 1) / per;
    const bool q16 = N <= 65536;
    int64_t qbytes = (int64_t)N * (q16 ? 2 : 4);
    a.per_warp = ((int64_t)a.cnt_words * 4 + qbytes + 15) / 16 * 16;

    // shared mode if up to 8 warps x per_warp fits comfortably
    const int64_t kSmemBudget = 200 * 1024;
    int wpb = 8;
    bool shared_mode = true;
    const int64_t tail_bytes = g->n_devices <= 32 ? 128 : 128 * kWideV;  // per-warp FIFO tails
    while (wpb > 1 && wpb * (a.per_warp + tail_bytes) > kSmemBudget) wpb >>= 1;
    if (wpb * (a.per_warp + tail_bytes) > kSmemBudget) { shared_mode = false; wpb = 4; }
    if (!shared_mode && allow_large && !pos && !out_rows && !interleaved && N < (1 << 27) &&
        g->n_devices <= 32)  // K3 large
        return dfsim_simulate_large(ctx, g, n_sims, dur, dur_stride, start, finish, makespan, busy, n_placed);
    size_t smem = (size_t)wpb * tail_bytes + (shared_mode ? (size_t)wpb * a.per_warp : 0);

    int blocks_per_sm = 1;
    if (shared_mode) {
        blocks_per_sm = (int)(227 * 1024 / (smem + 1024));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        if (blocks_per_sm * wpb > 64) blocks_per_sm = 64 / wpb;
    } else {
        blocks_per_sm = 4;
    }
    int64_t want = (n_sims + wpb - 1) / wpb;
    int64_t cap = (int64_t)ctx->num_sms * blocks_per_sm;
    int grid = (int)(want < cap ? want : cap);
    a.gscratch = nullptr;
    if (!shared_mode) {
        void *p = nullptr;
        int rc = dfsim_scratch(ctx, (size_t)grid * wpb * a.per_warp, &p);
        if (rc) return rc;
        a.gscratch = static_cast<unsigned char *>(p);
    }
    if (bits == 8) return q16 ? launch_bits<8, uint16_t>(ctx, a, shared_mode, wpb, grid, smem)
                              : launch_bits<8, uint32_t>(ctx, a, shared_mode, wpb, grid, smem);
    if (bits == 16) return q16 ? launch_bits<16, uint16_t>(ctx, a, shared_mode, wpb, grid, smem)
                               : launch_bits<16, uint32_t>(ctx, a, shared_mode, wpb, grid, smem);
    return q16 ? launch_bits<32, uint16_t>(ctx, a, shared_mode, wpb, grid, smem)
               : launch_bits<32, uint32_t>(ctx, a, shared_mode, wpb, grid, smem);
}

extern "C" int dfsim_simulate_batch_ex(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                                       int64_t dur_stride, double *start, double *finish, double *makespan,
                                       double *busy, int32_t *n_placed, const int32_t *pos, const int64_t *out_rows,
                                       int32_t interleaved) {
    return simulate_exact(ctx, g, n_sims, dur, dur_stride, start, finish, makespan, busy, n_placed, pos, out_rows,
                          interleaved, nullptr, true);
}

// The exact-capacity engine over the rows flagged in redo (ring overflows of K3 large).
int dfsim_simulate_exact_flagged(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                                 int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                                 int32_t *n_placed, const int32_t *redo) {
    return simulate_exact(ctx, g, n_sims, dur, dur_stride, start, finish, makespan, busy, n_placed, nullptr, nullptr,
                          0, redo, false);
}
