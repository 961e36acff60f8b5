// Internal declarations shared by the sm_100a translation units of libdfsim_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
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
int dfsim_after_launch_base(dfsim_ctx *ctx, const char *what);

// Checked builds (libdfsim_b200_checked.so, -DDFSIM_CHECKED; the pool has no compute-sanitizer):
// DFSIM_CHECK(cond, bit) guards an index the kernels derive from table data.  A failed check
// sets `bit` in this translation unit's check word -- no trap, the launch completes -- and the
// launch's dfsim_after_launch synchronises, reads and clears the word and returns
// DFSIM_CHECK_FAILED.  In the product build both are no-ops.
#ifdef DFSIM_CHECKED
static __device__ unsigned int dfsim_check_word;
#define DFSIM_CHECK(cond, bit)                                                            \
    do {                                                                                  \
        if (!(cond)) atomicOr(&dfsim_check_word, 1u << (bit));                            \
    } while (0)
static inline int dfsim_after_launch(dfsim_ctx *ctx, const char *what) {
    int rc = dfsim_after_launch_base(ctx, what);
    if (rc) return rc;
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    unsigned v = 0;
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(&v, dfsim_check_word, sizeof v);
    if (e != cudaSuccess) {
        ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
        return DFSIM_CUDA;
    }
    if (v) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(dfsim_check_word, &z, sizeof z);
        char buf[32];
        snprintf(buf, sizeof buf, "0x%x", v);
        ctx->last_error = std::string(what) + ": device bounds check failed (bits " + buf + ")";
        return DFSIM_CHECK_FAILED;
    }
    return DFSIM_OK;
}
#else
#define DFSIM_CHECK(cond, bit) \
    do {                       \
    } while (0)
static inline int dfsim_after_launch(dfsim_ctx *ctx, const char *what) { return dfsim_after_launch_base(ctx, what); }
#endif
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
