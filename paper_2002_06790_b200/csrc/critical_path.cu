// K4: critical path over finish-start durations, batched -- the reference's
// graph.critical_path (pkg/src/dfsim/graph.py:446-485) as summarize calls it
// (reporting.py:128,154) -- plus the topological order it walks (graph.py:424-443).
//
// suffix[v] = d[v] + max(0.0, max over successors suffix) is evaluated in ANY
// reverse topological order: each value is one exact max followed by one add, so
// the result is independent of the order.  One thread per strategy:
// every thread of a warp walks the same class-wide order, so control flow stays
// uniform and the per-node suffix values (layout [node][sim]) are coalesced.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace {

struct CpArgs {
    int32_t N;
    const int32_t *succ_off, *succ_idx, *indeg, *topo;
    int64_t S;       // sims in this chunk
    int64_t s0;      // first sim of the chunk
    const double *start, *finish;
    double *cp_len;
    int32_t *cp_path, *cp_path_len;
    double *suffix;  // [N][S] scratch
};

__global__ void __launch_bounds__(128) k_critical_path(CpArgs a) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.S) return;
    const int64_t s = a.s0 + i;
    const int32_t N = a.N;
    const double *st = a.start ? a.start + s * N : nullptr;  // NULL: `finish` holds durations
    const double *fi = a.finish + s * N;
    double *suf = a.suffix + i;
    const int64_t ld = a.S;

    double len = 0.0;
    int32_t src = -1;
    for (int32_t t = N - 1; t >= 0; t--) {
        const int32_t v = __ldg(a.topo + t);
        const double d = st ? __dsub_rn(fi[v], st[v]) : fi[v];  // finish - start (reporting.py:128)
        double best = 0.0;
        const int32_t e1 = __ldg(a.succ_off + v + 1);
        for (int32_t j = __ldg(a.succ_off + v); j < e1; j++) {
            const double x = suf[static_cast<int64_t>(__ldg(a.succ_idx + j)) * ld];
            if (x > best) best = x;
        }
        const double sv = __dadd_rn(d, best);
        suf[static_cast<int64_t>(v) * ld] = sv;
        if (__ldg(a.indeg + v) == 0 && (src < 0 || sv > len || (sv == len && v < src))) {
            len = sv;  // max over sources, then the min id achieving it (graph.py:471-474)
            src = v;
        }
    }
    a.cp_len[s] = len;
    if (!a.cp_path) return;
    int32_t *path = a.cp_path + s * N;
    int32_t k = 0;
    if (src >= 0) {
        int32_t v = src;
        path[k++] = v;
        for (;;) {  // greedy min-id walk (graph.py:479-484); successors are rank-sorted
            const int32_t j0 = __ldg(a.succ_off + v), j1 = __ldg(a.succ_off + v + 1);
            if (j0 == j1) break;
            double top = suf[static_cast<int64_t>(__ldg(a.succ_idx + j0)) * ld];
            for (int32_t j = j0 + 1; j < j1; j++) {
                const double x = suf[static_cast<int64_t>(__ldg(a.succ_idx + j)) * ld];
                if (x > top) top = x;
            }
            int32_t nxt = -1;
            for (int32_t j = j0; j < j1; j++) {
                const int32_t m = __ldg(a.succ_idx + j);
                if (suf[static_cast<int64_t>(m) * ld] == top) { nxt = m; break; }
            }
            v = nxt;
            path[k++] = v;
        }
    }
    a.cp_path_len[s] = k;
}

// Kahn's algorithm, level-synchronous, in one CTA (graph.py:424-443 semantics;
// the order inside a level is irrelevant to every consumer).
__global__ void __launch_bounds__(1024) k_topo(int32_t N, const int32_t *succ_off, const int32_t *succ_idx,
                                                const int32_t *indeg, int32_t *left, int32_t *order,
                                                int32_t *n_ordered) {
    __shared__ int32_t s_tail;
    if (threadIdx.x == 0) s_tail = 0;
    __syncthreads();
    for (int32_t v = threadIdx.x; v < N; v += blockDim.x) {
        const int32_t c = indeg[v];
        left[v] = c;
        if (c == 0) order[atomicAdd(&s_tail, 1)] = v;
    }
    __syncthreads();
    int32_t lo = 0, hi = s_tail;
    while (lo < hi) {
        __syncthreads();
        for (int32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const int32_t v = order[i];
            for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++) {
                const int32_t m = succ_idx[j];
                if (atomicSub(left + m, 1) == 1) order[atomicAdd(&s_tail, 1)] = m;
            }
        }
        __syncthreads();
        lo = hi;
        hi = s_tail;
    }
    if (threadIdx.x == 0) *n_ordered = s_tail;
}

}  // namespace

int dfsim_topo_launch(dfsim_ctx *ctx, int32_t N, const int32_t *succ_off, const int32_t *succ_idx,
                      const int32_t *indeg, int32_t *topo, int32_t *n_ordered_dev, int32_t *left_scratch) {
    k_topo<<<1, 1024, 0, ctx->stream>>>(N, succ_off, succ_idx, indeg, left_scratch, topo, n_ordered_dev);
    return dfsim_after_launch(ctx, "k_topo");
}

extern "C" int dfsim_topo_order(dfsim_ctx *ctx, const dfsim_graph *g, int32_t *topo, int32_t *n_ordered_host) {
    if (!ctx || !g || !topo || !n_ordered_host) return DFSIM_BAD_ARGUMENT;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (g->n_nodes == 0) { *n_ordered_host = 0; return DFSIM_OK; }
    void *p = nullptr;
    int rc = dfsim_scratch(ctx, sizeof(int32_t) * ((size_t)g->n_nodes + 1), &p);
    if (rc) return rc;
    int32_t *left = static_cast<int32_t *>(p);
    int32_t *cnt = left + g->n_nodes;
    rc = dfsim_topo_launch(ctx, g->n_nodes, g->succ_off, g->succ_idx, g->indeg, topo, cnt, left);
    if (rc) return rc;
    DFSIM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_small, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    DFSIM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    *n_ordered_host = *static_cast<int32_t *>(ctx->host_small);
    return DFSIM_OK;
}

extern "C" int dfsim_critical_path_batch(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *start,
                                         const double *finish, double *cp_len, int32_t *cp_path,
                                         int32_t *cp_path_len) {
    if (!ctx || !g) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, finish && cp_len, "finish (or durations) and cp_len are required");
    DFSIM_ARG_CHECK(ctx, g->topo != nullptr || g->n_nodes == 0, "graph topo order is required");
    DFSIM_ARG_CHECK(ctx, (cp_path == nullptr) == (cp_path_len == nullptr), "cp_path and cp_path_len go together");
    if (n_sims <= 0) return DFSIM_OK;
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    // chunk the batch so the [N][chunk] suffix scratch stays bounded (<= 8 GiB of HBM)
    const int64_t N = g->n_nodes > 0 ? g->n_nodes : 1;
    int64_t chunk = (int64_t)(8ll << 30) / (8 * N);
    chunk = chunk < 128 ? 128 : chunk / 128 * 128;
    if (chunk > n_sims) chunk = n_sims;
    void *p = nullptr;
    int rc = dfsim_scratch(ctx, (size_t)8 * N * chunk, &p);
    if (rc) return rc;
    for (int64_t s0 = 0; s0 < n_sims; s0 += chunk) {
        CpArgs a;
        a.N = g->n_nodes;
        a.succ_off = g->succ_off; a.succ_idx = g->succ_idx; a.indeg = g->indeg; a.topo = g->topo;
        a.S = n_sims - s0 < chunk ? n_sims - s0 : chunk;
        a.s0 = s0;
        a.start = start; a.finish = finish; a.cp_len = cp_len;
        a.cp_path = cp_path; a.cp_path_len = cp_path_len;
        a.suffix = static_cast<double *>(p);
        const int threads = 128;
        k_critical_path<<<(unsigned)((a.S + threads - 1) / threads), threads, 0, ctx->stream>>>(a);
        rc = dfsim_after_launch(ctx, "k_critical_path");
        if (rc) return rc;
    }
    return DFSIM_OK;
}
