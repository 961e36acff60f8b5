// Scalar cost formulas of the drop-in surface, evaluated on the device with the same
// arithmetic as K2 (estimate.cu): predict (costmodel.py:158-165) over a batch of feature
// vectors, and comm_time_us / transfer_time / allreduce_time (costmodel.py:168-223) over a
// batch of (bytes, participants, link) rows.  Round-to-nearest intrinsics, never FMA.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace {

constexpr double kMiB = 1048576.0;

// value = intercept + sum(c * f) with CPython 3.12's float sum (first term exact, Neumaier
// compensation added when nonzero and finite), then max(0.0, value)
__global__ void k_predict(int32_t k, const double *coef, double intercept, int64_t n, const double *feats, double *out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double *f = feats + i * k;
        double s = 0.0, comp = 0.0;
        for (int j = 0; j < k; j++) {
            const double x = __dmul_rn(__ldg(coef + j), __ldg(f + j));
            if (j == 0) {
                s = __dadd_rn(0.0, x);
            } else {
                const double t = __dadd_rn(s, x);
                comp = fabs(s) >= fabs(x) ? __dadd_rn(comp, __dadd_rn(__dsub_rn(s, t), x))
                                          : __dadd_rn(comp, __dadd_rn(__dsub_rn(x, t), s));
                s = t;
            }
        }
        if (comp != 0.0 && isfinite(comp)) s = __dadd_rn(s, comp);
        const double v = __dadd_rn(intercept, s);
        out[i] = v > 0.0 ? v : 0.0;
    }
}

// kind 0: comm_time_us = lat + (bytes / MiB) / thr * 1e6 (transfer_time, measured allreduce)
// kind 1: ring = ((2 (n-1) / n) * (bytes / MiB)) / thr * 1e6 + 2 (n-1) lat
__global__ void k_comm(int64_t n, const uint8_t *kind, const int64_t *bytes, const int32_t *parts, const double *thr,
                       const double *lat, double *out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double b = __ll2double_rn(bytes[i]);
        if (kind[i] == 0) {
            out[i] = __dadd_rn(lat[i], __dmul_rn(__ddiv_rn(__ddiv_rn(b, kMiB), thr[i]), 1e6));
        } else {
            const double nm1 = static_cast<double>(parts[i] - 1);
            const double ring = __ddiv_rn(__dmul_rn(2.0, nm1), static_cast<double>(parts[i]));
            const double bw = __dmul_rn(__ddiv_rn(__dmul_rn(ring, __ddiv_rn(b, kMiB)), thr[i]), 1e6);
            out[i] = __dadd_rn(bw, __dmul_rn(__dmul_rn(2.0, nm1), lat[i]));
        }
    }
}

int grid_for(dfsim_ctx *ctx, int64_t n) {
    const int64_t b = (n + 255) / 256;
    return static_cast<int>(b < ctx->num_sms * 4 ? (b > 0 ? b : 1) : ctx->num_sms * 4);
}

}  // namespace

extern "C" int dfsim_predict_batch(dfsim_ctx *ctx, int32_t k, const double *coef, double intercept, int64_t n,
                                   const double *feats, double *out) {
    if (!ctx || k < 0 || n < 0 || (n > 0 && (!out || (k > 0 && (!coef || !feats))))) return DFSIM_BAD_ARGUMENT;
    if (n == 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    k_predict<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(k, coef, intercept, n, feats, out);
    return dfsim_after_launch(ctx, "k_predict");
}

extern "C" int dfsim_comm_batch(dfsim_ctx *ctx, int64_t n, const uint8_t *kind, const int64_t *bytes,
                                const int32_t *participants, const double *thr, const double *lat, double *out) {
    if (!ctx || n < 0 || (n > 0 && (!kind || !bytes || !participants || !thr || !lat || !out))) return DFSIM_BAD_ARGUMENT;
    if (n == 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    k_comm<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, kind, bytes, participants, thr, lat, out);
    return dfsim_after_launch(ctx, "k_comm");
}
