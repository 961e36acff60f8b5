// K6: the schedule summary of reporting.summarize (reporting.py:117-162) for a batch
// of schedules already resident in HBM -- the next consumer of the engine's output.
//
// Every number the reference derives is an order-dependent floating-point fold over
// the schedule's entry order (engine.py:88: by start, device string, node id string),
// so the kernels first rebuild that order and then fold sequentially, exactly as the
// reference does, with the independent folds spread over threads:
//   1. entry order   -- stable segmented radix sort of start bits (starts are >= +0.0,
//                       so their IEEE bits order like unsigned integers) over the class's
//                       (device rank, node rank) order: ties fall back to device then id.
//   2. key groups    -- stable segmented radix sort of the entries by op key
//                       (`op_type or node_id`, reporting.py:132), keeping entry order
//                       inside each key; one thread folds each key's totals (133).
//   3. busy folds    -- compute_us / comm_us (142-148) and the union + two-pointer
//                       overlap sweep (92-114, 149) on two independent cursors over the
//                       entry stream (no interval buffers); one thread per fold.
// The host ranks the (few) key totals with the reference's own sorted()/sum().
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "internal.cuh"

namespace {

size_t align_up(size_t x) { return (x + 255) / 256 * 256; }

__global__ void k_sum_init(int64_t n_rows, int32_t n_keys, double *key_total, int32_t *key_first,
                           int64_t *seg_begin, int32_t N) {
    const int64_t nk = n_rows * n_keys;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nk;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        key_total[i] = 0.0;
        key_first[i] = -1;
    }
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= n_rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        seg_begin[r] = r * N;
}

// sort input 1: start bits of the class's (device, node) order
__global__ void k_entry_keys(int64_t n_rows, int32_t N, const int32_t *base_order, const double *start, int64_t ld,
                             unsigned long long *keys, int32_t *vals) {
    const int64_t total = n_rows * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N;
        const int32_t v = __ldg(base_order + (i - r * N));
        keys[i] = static_cast<unsigned long long>(__double_as_longlong(start[r * ld + v]));
        vals[i] = v;
    }
}

// sort input 2: op key of each entry, value = entry index
__global__ void k_group_keys(int64_t n_rows, int32_t N, const int32_t *key, const int32_t *entry_order,
                             uint32_t *keys, int32_t *vals) {
    const int64_t total = n_rows * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N;
        keys[i] = static_cast<uint32_t>(__ldg(key + entry_order[i]));
        vals[i] = static_cast<int32_t>(i - r * N);
    }
}

// One thread per key segment: totals[key] = totals.get(key, 0.0) + (finish - start)
// in entry order (reporting.py:131-133).  Loads run 8 entries ahead of the fold.
__global__ void k_key_totals(int64_t n_rows, int32_t N, int32_t n_keys, const uint32_t *gkey, const int32_t *gentry,
                             const int32_t *entry_order, const double *start, const double *finish, int64_t ld,
                             double *key_total, int32_t *key_first) {
    const int64_t total = n_rows * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / N;
        const int64_t j0 = i - r * N;
        const uint32_t k = gkey[i];
        if (j0 > 0 && gkey[i - 1] == k) continue;  // not the first entry of its key
        const int32_t *ord = entry_order + r * N;
        const double *st = start + r * ld, *fi = finish + r * ld;
        double sum = 0.0;
        int64_t j = i;
        const int64_t end = (r + 1) * N;
        for (;;) {
            double d[8];
            int n = 0;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const bool in = j + u < end && gkey[j + u] == k;
                if (in) {
                    const int32_t v = ord[gentry[j + u]];
                    d[u] = __dsub_rn(fi[v], st[v]);
                    n = u + 1;
                }
            }
            // n counts a prefix: keys are contiguous, so the first miss ends the segment
            for (int u = 0; u < n; u++) sum = __dadd_rn(sum, d[u]);
            j += n;
            if (n < 8) break;
        }
        key_total[r * n_keys + k] = sum;
        key_first[r * n_keys + k] = gentry[i];
    }
}

struct Cursor {  // walks the entries of one kind (compute or comm) in entry order
    int32_t i;
};

// next union component of the kind's intervals at or after cursor position (reporting.py:92-99)
__device__ __forceinline__ bool next_component(Cursor &c, int32_t N, const int32_t *ord, const uint8_t *comm,
                                               uint8_t want, const double *st, const double *fi, double &lo,
                                               double &hi) {
    int32_t i = c.i;
    while (i < N && __ldg(comm + ord[i]) != want) i++;
    if (i >= N) {
        c.i = N;
        return false;
    }
    int32_t v = ord[i++];
    lo = st[v];
    hi = fi[v];
    for (; i < N; i++) {
        v = ord[i];
        if (__ldg(comm + v) != want) continue;
        const double s = st[v];
        if (s <= hi) {
            const double f = fi[v];
            if (f > hi) hi = f;
        } else {
            break;
        }
    }
    c.i = i;
    return true;
}

// Per row, three independent folds: task 0 compute_us, task 1 comm_us (reporting.py:142-148),
// task 2 the overlap sweep (102-114) over the two kinds' union components.
__global__ void k_busy_folds(int64_t n_rows, int32_t N, const int32_t *entry_order, const uint8_t *comm,
                             const double *start, const double *finish, int64_t ld, double *sums) {
    const int64_t total = n_rows * 3;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int task = static_cast<int>(t / n_rows);
        const int64_t r = t - task * n_rows;
        const int32_t *ord = entry_order + r * N;
        const double *st = start + r * ld, *fi = finish + r * ld;
        double acc = 0.0;
        if (task < 2) {
            const uint8_t want = static_cast<uint8_t>(task);
            for (int32_t i = 0; i < N; i += 8) {
                double d[8];
                bool in[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    in[u] = false;
                    if (i + u < N) {
                        const int32_t v = ord[i + u];
                        if (__ldg(comm + v) == want) {
                            in[u] = true;
                            d[u] = __dsub_rn(fi[v], st[v]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; u++)
                    if (in[u]) acc = __dadd_rn(acc, d[u]);
            }
        } else {
            Cursor a{0}, b{0};
            double alo = 0, ahi = 0, blo = 0, bhi = 0;
            bool ha = next_component(a, N, ord, comm, 0, st, fi, alo, ahi);
            bool hb = next_component(b, N, ord, comm, 1, st, fi, blo, bhi);
            while (ha && hb) {
                const double lo = alo >= blo ? alo : blo;
                const double hi = ahi <= bhi ? ahi : bhi;
                if (hi > lo) acc = __dadd_rn(acc, __dsub_rn(hi, lo));
                if (ahi <= bhi)
                    ha = next_component(a, N, ord, comm, 0, st, fi, alo, ahi);
                else
                    hb = next_component(b, N, ord, comm, 1, st, fi, blo, bhi);
            }
        }
        sums[r * 3 + task] = acc;
    }
}

int grid_for(dfsim_ctx *ctx, int64_t n, int threads = 256) {
    const int64_t want = (n + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(ctx->num_sms) * 8;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

int bits_for(int64_t n) {
    int b = 1;
    while ((1ll << b) < n) b++;
    return b;
}

}  // namespace

extern "C" int dfsim_summarize(dfsim_ctx *ctx, const dfsim_summary_tables *t, int64_t n_rows, const double *start,
                               const double *finish, int64_t ld, int32_t *entry_order, int32_t order_given,
                               double *key_total, int32_t *key_first, double *sums) {
    if (!ctx || !t) return DFSIM_BAD_ARGUMENT;
    const int32_t N = t->n_nodes, K = t->n_keys;
    DFSIM_ARG_CHECK(ctx, N >= 0 && K >= 1 && n_rows >= 0 && ld >= N, "bad summary sizes");
    DFSIM_ARG_CHECK(ctx, n_rows == 0 || N == 0 || (start && finish && entry_order && t->key && t->comm),
                    "null summary input");
    DFSIM_ARG_CHECK(ctx, order_given || N == 0 || t->base_order, "entry order needs base_order");
    DFSIM_ARG_CHECK(ctx, key_total && key_first && sums, "null summary output");
    DFSIM_ARG_CHECK(ctx, n_rows * static_cast<int64_t>(N) < (1ll << 31), "summary batch too large");
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (n_rows == 0) return DFSIM_OK;
    const int64_t items = n_rows * N;
    const int nseg = static_cast<int>(n_rows);

    // scratch: keys/vals in+out for both sorts, segment offsets, cub temp
    size_t tmp1 = 0, tmp2 = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp1, (const unsigned long long *)nullptr,
                                             (unsigned long long *)nullptr, (const int32_t *)nullptr,
                                             (int32_t *)nullptr, (int)items, nseg, (const int64_t *)nullptr,
                                             (const int64_t *)nullptr, 0, 64);
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp2, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                             (const int32_t *)nullptr, (int32_t *)nullptr, (int)items, nseg,
                                             (const int64_t *)nullptr, (const int64_t *)nullptr, 0, bits_for(K));
    const size_t tmp = std::max(tmp1, tmp2);
    size_t o_k64 = 0;                                                  // u64 keys in
    size_t o_k64b = align_up(o_k64 + 8 * (size_t)items);               // u64 keys out
    size_t o_vin = align_up(o_k64b + 8 * (size_t)items);               // i32 vals in
    size_t o_gent = align_up(o_vin + 4 * (size_t)items);               // i32 grouped entry idx
    size_t o_seg = align_up(o_gent + 4 * (size_t)items);               // i64 [n_rows + 1]
    size_t o_tmp = align_up(o_seg + 8 * (size_t)(n_rows + 1));
    void *scratch = nullptr;
    int rc = dfsim_scratch(ctx, o_tmp + tmp + 256, &scratch);
    if (rc) return rc;
    char *sb = static_cast<char *>(scratch);
    auto *k64 = reinterpret_cast<unsigned long long *>(sb + o_k64);
    auto *k64b = reinterpret_cast<unsigned long long *>(sb + o_k64b);
    auto *vin = reinterpret_cast<int32_t *>(sb + o_vin);
    auto *gent = reinterpret_cast<int32_t *>(sb + o_gent);
    auto *seg = reinterpret_cast<int64_t *>(sb + o_seg);
    void *ctmp = sb + o_tmp;
    const int64_t *cseg = seg;
    // the u32 group keys reuse the u64 key buffers
    auto *g32 = reinterpret_cast<uint32_t *>(k64);
    auto *g32b = reinterpret_cast<uint32_t *>(k64b);

    k_sum_init<<<grid_for(ctx, std::max<int64_t>(n_rows * K, n_rows + 1)), 256, 0, ctx->stream>>>(
        n_rows, K, key_total, key_first, seg, N);
    rc = dfsim_after_launch(ctx, "k_sum_init");
    if (rc) return rc;
    if (N == 0) {
        DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(sums, 0, sizeof(double) * 3 * n_rows, ctx->stream));
        return DFSIM_OK;
    }
    if (!order_given) {
        k_entry_keys<<<grid_for(ctx, items), 256, 0, ctx->stream>>>(n_rows, N, t->base_order, start, ld, k64, vin);
        rc = dfsim_after_launch(ctx, "k_entry_keys");
        if (rc) return rc;
        size_t tb = tmp;
        DFSIM_CUDA_TRY(ctx, cub::DeviceSegmentedRadixSort::SortPairs(ctmp, tb, k64, k64b, vin, entry_order,
                                                                     (int)items, nseg, cseg, cseg + 1, 0, 64,
                                                                     ctx->stream));
        ctx->launches += 1;
    }
    k_group_keys<<<grid_for(ctx, items), 256, 0, ctx->stream>>>(n_rows, N, t->key, entry_order, g32, vin);
    rc = dfsim_after_launch(ctx, "k_group_keys");
    if (rc) return rc;
    {
        size_t tb = tmp;
        DFSIM_CUDA_TRY(ctx, cub::DeviceSegmentedRadixSort::SortPairs(ctmp, tb, g32, g32b, vin, gent, (int)items, nseg,
                                                                     cseg, cseg + 1, 0, bits_for(K), ctx->stream));
        ctx->launches += 1;
    }
    k_key_totals<<<grid_for(ctx, items), 256, 0, ctx->stream>>>(n_rows, N, K, g32b, gent, entry_order, start, finish,
                                                                ld, key_total, key_first);
    rc = dfsim_after_launch(ctx, "k_key_totals");
    if (rc) return rc;
    k_busy_folds<<<grid_for(ctx, n_rows * 3, 64), 64, 0, ctx->stream>>>(n_rows, N, entry_order, t->comm, start,
                                                                         finish, ld, sums);
    return dfsim_after_launch(ctx, "k_busy_folds");
}
