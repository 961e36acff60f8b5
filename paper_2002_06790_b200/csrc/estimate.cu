// K2: batched profile gather -- the reference's estimate_all fallback chain
// (pkg/src/dfsim/costmodel.py:282-331) for every (strategy, node):
//   override (302-304) -> exact record + gap (305-311) -> fitted model + gap
//   (313-321, predict 158-165) -> communication formula (323-326, 347-376,
//   transfer_time 176-182, allreduce_time 185-223) -> unknown (327).
// Arithmetic is IEEE double in the reference's evaluation order with explicit
// round-to-nearest intrinsics (never contracted to FMA), and predict's sum is
// CPython 3.12's compensated float sum.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace {

constexpr double kMiB = 1048576.0;

__device__ __forceinline__ int find_u64(const uint64_t *keys, int n, uint64_t k) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(reinterpret_cast<const unsigned long long *>(keys) + mid) < k) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(reinterpret_cast<const unsigned long long *>(keys) + lo) == k ? lo : -1;
}

__device__ __forceinline__ int find_i32(const int32_t *keys, int lo, int hi, int32_t k) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(keys + mid) < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// comm_time_us (costmodel.py:168-173): latency + (bytes / MiB) / thr * 1e6
__device__ __forceinline__ double comm_time(double bytes, double thr, double lat) {
    return __dadd_rn(lat, __dmul_rn(__ddiv_rn(__ddiv_rn(bytes, kMiB), thr), 1e6));
}

// predict (costmodel.py:158-165) with CPython's float sum: 0 + first term, then
// Neumaier-compensated terms, compensation added if nonzero and finite; clamp.
// Returns false when the model does not cover the node's features (costmodel.py:318).
__device__ bool predict(const dfsim_profile_tables &t, int m, int sg, double *out) {
    const int m0 = __ldg(t.model_off + m), m1 = __ldg(t.model_off + m + 1);
    const int f0 = __ldg(t.sig_off + sg), f1 = __ldg(t.sig_off + sg + 1);
    double s = 0.0, comp = 0.0;
    int f = f0;
    for (int j = m0; j < m1; j++) {
        const int32_t name = __ldg(t.model_name + j);
        f = find_i32(t.sig_name, f, f1, name);  // names ascending on both sides
        if (f >= f1 || __ldg(t.sig_name + f) != name) return false;
        const double x = __dmul_rn(__ldg(t.model_coef + j), __ldg(t.sig_val + f));
        if (j == m0) {
            s = __dadd_rn(0.0, x);
        } else {
            const double tt = __dadd_rn(s, x);
            comp = fabs(s) >= fabs(x) ? __dadd_rn(comp, __dadd_rn(__dsub_rn(s, tt), x))
                                      : __dadd_rn(comp, __dadd_rn(__dsub_rn(x, tt), s));
            s = tt;
        }
    }
    if (comp != 0.0 && isfinite(comp)) s = __dadd_rn(s, comp);
    const double value = __dadd_rn(__ldg(t.model_icpt + m), s);
    *out = value > 0.0 ? value : 0.0;  // max(0.0, value); NaN -> 0.0 like Python's max
    return true;
}

// v: node rank; gv: graph variant (per-node feature / comm rows are [n_graph_variants][N])
__device__ __forceinline__ double estimate_one(const dfsim_profile_tables &t, int N, int v, int gv, int hw,
                                               double gap_s, int algo, int path, int ovs, uint8_t *src) {
    const int64_t vv = static_cast<int64_t>(gv) * N + v;
    if (ovs >= 0) {
        const int o0 = __ldg(t.ov_off + ovs), o1 = __ldg(t.ov_off + ovs + 1);
        const int p = find_i32(t.ov_node, o0, o1, v);
        if (p < o1 && __ldg(t.ov_node + p) == v) { *src = DFSIM_SRC_OVERRIDE; return __ldg(t.ov_val + p); }
    }
    const int kind = __ldg(t.kind + v);
    const double gap = kind == 0 ? gap_s : 0.0;
    const int op = __ldg(t.op + v), sg = __ldg(t.sig + vv);
    const uint64_t ekey = (static_cast<uint64_t>(hw) << 42) | (static_cast<uint64_t>(op) << 21) | static_cast<uint64_t>(sg);
    const int e = find_u64(t.exact_key, t.n_exact, ekey);
    if (e >= 0) { *src = DFSIM_SRC_EXACT; return __dadd_rn(__ldg(t.exact_mean + e), gap); }
    const int m = find_u64(t.model_key, t.n_models, (static_cast<uint64_t>(hw) << 21) | static_cast<uint64_t>(op));
    double pv;
    if (m >= 0 && predict(t, m, sg, &pv)) { *src = DFSIM_SRC_FITTED; return __dadd_rn(pv, gap); }
    if (kind != 0 && __ldg(t.comm_ok + vv)) {
        const long long b = __ldg(reinterpret_cast<const long long *>(t.comm_bytes) + vv);
        const double bd = __ll2double_rn(b);
        if (kind == 1) {  // Transfer over its Link device (transfer_time)
            if (b <= 0) { *src = DFSIM_SRC_BAD_BYTES; return 0.0; }
            *src = DFSIM_SRC_COMM;
            return comm_time(bd, __ldg(t.link_thr + vv), __ldg(t.link_lat + vv));
        }
        const int n = __ldg(t.group_size + vv);  // Collective (allreduce_time)
        if (b > 0 && n >= 2 && path >= 0 && path < t.n_paths) {
            if (algo == 0) {
                const int r = find_u64(t.nccl_key, t.n_nccl, (static_cast<uint64_t>(path) << 32) | static_cast<uint32_t>(n));
                if (r >= 0) { *src = DFSIM_SRC_COMM; return comm_time(bd, __ldg(t.nccl_thr + r), 0.0); }
            }
            if (__ldg(t.uni_ok + path)) {
                const double nm1 = static_cast<double>(n - 1);
                const double ring = __ddiv_rn(__dmul_rn(2.0, nm1), static_cast<double>(n));
                const double bw = __dmul_rn(__ddiv_rn(__dmul_rn(ring, __ddiv_rn(bd, kMiB)), __ldg(t.uni_thr + path)), 1e6);
                *src = DFSIM_SRC_COMM;
                return __dadd_rn(bw, __dmul_rn(__dmul_rn(2.0, nm1), __ldg(t.uni_lat + path)));
            }
        }
    }
    *src = DFSIM_SRC_UNKNOWN;
    return 0.0;
}

__global__ void __launch_bounds__(256) k_estimate(int32_t N, dfsim_profile_tables t, dfsim_strategies st,
                                                  double *dur, uint8_t *src_out, int32_t *bad) {
    const int64_t total = st.n_sims * static_cast<int64_t>(N);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = i / N;
        const int v = static_cast<int>(i - s * N);
        uint8_t src;
        double val = estimate_one(t, N, v, st.gvariant ? __ldg(st.gvariant + s) : 0, __ldg(st.hw + s),
                                  __ldg(st.op_gap + s), __ldg(st.algo + s), __ldg(st.path + s),
                                  st.override_set ? __ldg(st.override_set + s) : -1, &src);
        if (src < DFSIM_SRC_BAD_BYTES && !(val >= 0.0)) src = DFSIM_SRC_NEGATIVE;  // DurationEntry check
        dur[i] = val;
        if (src_out) src_out[i] = src;
        if (src >= DFSIM_SRC_BAD_BYTES && bad) atomicAdd(bad + s, 1);
    }
}

__global__ void __launch_bounds__(256) k_resolve_variants(int32_t N, dfsim_profile_tables t, int32_t V,
                                                          const int32_t *var_hw, const uint8_t *var_algo,
                                                          const int32_t *var_path, const int32_t *var_gv,
                                                          double *base, uint8_t *status) {
    const int64_t total = static_cast<int64_t>(V) * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int var = static_cast<int>(i / N);
        const int v = static_cast<int>(i - static_cast<int64_t>(var) * N);
        uint8_t src;
        double val = estimate_one(t, N, v, var_gv ? __ldg(var_gv + var) : 0, __ldg(var_hw + var), 0.0,
                                  __ldg(var_algo + var), __ldg(var_path + var), -1, &src);
        if (src < DFSIM_SRC_BAD_BYTES && !(val >= 0.0)) src = DFSIM_SRC_NEGATIVE;
        if (src >= DFSIM_SRC_BAD_BYTES) val = __longlong_as_double(0x7ff8000000000000LL);
        // record/model values get the candidate's op_gap on Compute nodes (costmodel.py:305)
        const bool add_gap = (src == DFSIM_SRC_EXACT || src == DFSIM_SRC_FITTED) && __ldg(t.kind + v) == 0;
        base[i] = add_gap ? -val : val;
        status[i] = src;
    }
}

// rows of (variant, override set) combinations: the variant's K2a row with the set's override
// values stamped in (costmodel.py:302-304 -- an override replaces the estimate, no op_gap), so
// the fused engine reads every duration from one row and never searches an override table
__global__ void __launch_bounds__(256) k_override_rows(int32_t N, int32_t C, const double *base, const int32_t *c_var,
                                                       const int32_t *c_set, const int32_t *ov_off,
                                                       const int32_t *ov_node, const double *ov_val, double *out) {
    const int64_t total = static_cast<int64_t>(C) * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i / N);
        const int r = static_cast<int>(i - static_cast<int64_t>(c) * N);
        double b = __ldg(base + static_cast<int64_t>(__ldg(c_var + c)) * N + r);
        const int s = __ldg(c_set + c);
        if (s >= 0) {
            int lo = __ldg(ov_off + s), hi = __ldg(ov_off + s + 1);
            const int end = hi;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(ov_node + mid) < r) lo = mid + 1; else hi = mid;
            }
            if (lo < end && __ldg(ov_node + lo) == r) b = __ldg(ov_val + lo);  // finite, >= 0: sign clear
        }
        out[i] = b;
    }
}

}  // namespace

extern "C" int dfsim_override_rows(dfsim_ctx *ctx, int32_t n_nodes, int32_t n_combos, const double *base,
                                   const int32_t *combo_variant, const int32_t *combo_set, const int32_t *ov_off,
                                   const int32_t *ov_node, const double *ov_val, double *out) {
    if (!ctx || !base || !combo_variant || !combo_set || !out) return DFSIM_BAD_ARGUMENT;
    if (n_nodes <= 0 || n_combos <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const int64_t total = (int64_t)n_combos * n_nodes;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)ctx->num_sms * 16) blocks = (int64_t)ctx->num_sms * 16;
    k_override_rows<<<(unsigned)blocks, 256, 0, ctx->stream>>>(n_nodes, n_combos, base, combo_variant, combo_set,
                                                              ov_off, ov_node, ov_val, out);
    return dfsim_after_launch(ctx, "k_override_rows");
}

extern "C" int dfsim_resolve_variants(dfsim_ctx *ctx, int32_t n_nodes, const dfsim_profile_tables *t, int32_t n_variants,
                                      const int32_t *var_hw, const uint8_t *var_algo, const int32_t *var_path,
                                      const int32_t *var_gv, double *base, uint8_t *status) {
    if (!ctx || !t || !base || !status) return DFSIM_BAD_ARGUMENT;
    if (n_nodes <= 0 || n_variants <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const int64_t total = (int64_t)n_variants * n_nodes;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)ctx->num_sms * 16) blocks = (int64_t)ctx->num_sms * 16;
    k_resolve_variants<<<(unsigned)blocks, 256, 0, ctx->stream>>>(n_nodes, *t, n_variants, var_hw, var_algo, var_path,
                                                                 var_gv, base, status);
    return dfsim_after_launch(ctx, "k_resolve_variants");
}

extern "C" int dfsim_estimate_batch(dfsim_ctx *ctx, int32_t n_nodes, const dfsim_profile_tables *t,
                                    const dfsim_strategies *st, double *dur, uint8_t *src, int32_t *bad) {
    if (!ctx || !t || !st || !dur) return DFSIM_BAD_ARGUMENT;
    if (st->n_sims <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (n_nodes <= 0) {  // an empty graph estimates fine: bad[s] = 0 (no unresolved node)
        if (bad) DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, sizeof(int32_t) * (size_t)st->n_sims, ctx->stream));
        return DFSIM_OK;
    }
    const int64_t total = st->n_sims * (int64_t)n_nodes;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)ctx->num_sms * 16;
    if (blocks > cap) blocks = cap;
    if (bad) DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, sizeof(int32_t) * (size_t)st->n_sims, ctx->stream));
    k_estimate<<<(unsigned)blocks, 256, 0, ctx->stream>>>(n_nodes, *t, *st, dur, src, bad);
    return dfsim_after_launch(ctx, "k_estimate");
}
