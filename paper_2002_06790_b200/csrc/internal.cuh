// Internal declarations shared by the sm_100a translation units of libdfsim_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <deque>
#include <mutex>
#include <string>

#include "dfsim_b200.h"

// Device scratch belongs to (context, stream): kernels of different topology classes may
// run concurrently on different streams of one context without sharing scratch.
struct dfsim_stream_scratch {
    cudaStream_t stream = nullptr;
    void *scratch = nullptr;  // per-warp engine state in global mode, CP suffix values, cub temp
    size_t scratch_bytes = 0;
    void *aux = nullptr;      // small per-call arrays that must survive a scratch reallocation
    size_t aux_bytes = 0;
};

struct dfsim_ctx {
    int32_t device = 0;
    cudaStream_t stream = nullptr;
    int32_t num_sms = 148;
    int64_t launches = 0;
    // deque: entries keep their address while other streams are added; guarded by mu (a
    // context may be shared by threads that serialise their calls, see dfsim_b200.h)
    std::deque<dfsim_stream_scratch> per_stream;
    std::mutex mu;
    // pinned host staging for small synchronous results
    void *host_small = nullptr;
    std::string last_error;
};

#define DFSIM_FULL_MASK 0xffffffffu

// Record a CUDA failure on ctx and return DFSIM_CUDA from the enclosing function.
#define DFSIM_CUDA_TRY(ctx, expr)                                                          \
    do {                                                                                   \
        cudaError_t err__ = (expr);                                                        \
        if (err__ != cudaSuccess) {                                                        \
            (ctx)->last_error = std::string(#expr) + ": " + cudaGetErrorString(err__);     \
            return DFSIM_CUDA;                                                             \
        }                                                                                  \
    } while (0)

#define DFSIM_ARG_CHECK(ctx, cond, msg)                                                    \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            (ctx)->last_error = (msg);                                                     \
            return DFSIM_BAD_ARGUMENT;                                                     \
        }                                                                                  \
    } while (0)

// After a kernel launch: count it and surface launch-configuration errors.
int dfsim_after_launch(dfsim_ctx *ctx, const char *what);
// Grow ctx->scratch to at least `bytes` (stream-ordered: synchronises the stream first).
int dfsim_scratch(dfsim_ctx *ctx, size_t bytes, void **out);
// Grow ctx->aux (same rules); independent of ctx->scratch.
int dfsim_aux(dfsim_ctx *ctx, size_t bytes, void **out);

// ------------------------------------------------------------------ device helpers

__device__ __forceinline__ double warp_min_f64(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(DFSIM_FULL_MASK, x, o));
    return x;
}

__device__ __forceinline__ double warp_max_f64(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(DFSIM_FULL_MASK, x, o));
    return x;
}

__device__ __forceinline__ int warp_sum_i32(int x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(DFSIM_FULL_MASK, x, o);
    return x;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
