// K5: best-strategy selection.  The reference has no search; the
// closest behaviour is cmd_simulate's list of per-config makespans
// (cli.py:133-148).  "Best" is the first minimum: min over (makespan, index),
// i.e. Python's min(range(S), key=makespan.__getitem__).  Per GPU this reduces
// to one 16-byte record; across GPUs the records are all-gathered over NCCL and
// reduced again with dfsim_argmin_records.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace {

struct Rec {
    double v;
    long long i;
};

__device__ __forceinline__ bool rec_less(double va, long long ia, double vb, long long ib) {
    return va < vb || (va == vb && ia < ib);
}

__device__ __forceinline__ void warp_rec_min(double &v, long long &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(DFSIM_FULL_MASK, v, o);
        const long long oi = __shfl_xor_sync(DFSIM_FULL_MASK, i, o);
        if (rec_less(ov, oi, v, i)) { v = ov; i = oi; }
    }
}

template <bool kRecords>
__global__ void __launch_bounds__(1024) k_argmin(int64_t n, const double *values, int64_t base, const Rec *recs,
                                                 Rec *out) {
    __shared__ double sv[32];
    __shared__ long long si[32];
    double v = __longlong_as_double(0x7ff0000000000000LL);
    long long idx = 0x7fffffffffffffffLL;
    // block b reduces its slice [b * per, min(n, (b + 1) * per)) into out[b]
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * per, k1 = k0 + per < n ? k0 + per : n;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const double x = kRecords ? recs[k].v : values[k];
        const long long j = kRecords ? recs[k].i : base + k;
        if (rec_less(x, j, v, idx)) { v = x; idx = j; }
    }
    warp_rec_min(v, idx);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sv[w] = v; si[w] = idx; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        v = lane < nw ? sv[lane] : __longlong_as_double(0x7ff0000000000000LL);
        idx = lane < nw ? si[lane] : 0x7fffffffffffffffLL;
        warp_rec_min(v, idx);
        if (lane == 0) { out[blockIdx.x].v = v; out[blockIdx.x].i = idx; }
    }
}

}  // namespace

extern "C" int dfsim_argmin(dfsim_ctx *ctx, int64_t n, const double *values, int64_t index_base, void *out_record) {
    if (!ctx || !out_record || (n > 0 && !values)) return DFSIM_BAD_ARGUMENT;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (n <= 16384) {
        k_argmin<false><<<1, 1024, 0, ctx->stream>>>(n, values, index_base, nullptr, static_cast<Rec *>(out_record));
        return dfsim_after_launch(ctx, "k_argmin");
    }
    // two passes: one partial record per SM-sized slice, then the first minimum of the partials
    // (slices are in index order, so ties still resolve to the smallest index)
    const int blocks = ctx->num_sms;
    void *part = nullptr;
    int rc = dfsim_aux(ctx, sizeof(Rec) * blocks, &part);
    if (rc) return rc;
    k_argmin<false><<<blocks, 1024, 0, ctx->stream>>>(n, values, index_base, nullptr, static_cast<Rec *>(part));
    rc = dfsim_after_launch(ctx, "k_argmin");
    if (rc) return rc;
    k_argmin<true><<<1, 1024, 0, ctx->stream>>>(blocks, nullptr, 0, static_cast<const Rec *>(part),
                                                static_cast<Rec *>(out_record));
    return dfsim_after_launch(ctx, "k_argmin_records");
}

extern "C" int dfsim_argmin_records(dfsim_ctx *ctx, int64_t n, const void *records, void *out_record) {
    if (!ctx || !out_record || (n > 0 && !records)) return DFSIM_BAD_ARGUMENT;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    k_argmin<true><<<1, 1024, 0, ctx->stream>>>(n, nullptr, 0, static_cast<const Rec *>(records),
                                                static_cast<Rec *>(out_record));
    return dfsim_after_launch(ctx, "k_argmin_records");
}
