// K1: data-parallel expansion emitted straight into CSR -- the reference's
// expand_data_parallel (pkg/src/dfsim/strategy.py:170-282) followed by
// DataflowGraph.successors()/in_degree() (graph.py:122-135).
//
// The host resolves strings once per topology class (ranks of "<id>@r<k>" and
// "allreduce_<gid>", device ranks); the device builds everything per edge:
//   clone (k, v) keeps v's refs within replica k (strategy.py:215); a ref to a
//   marked gradient becomes a ref to its collective when R > 1 (231-238); the
//   collective of gradient g consumes g@r0..g@r{R-1} (249).  PS mode (ps.py, new code):
//   g@r<k> -> push_<g>@r<k> -> aggregate_<g> -> pull_<g>@r<k>, and refs to g@r<k> read the pull.
// Edges are (producer rank << 32 | consumer rank) keys; one radix sort gives the
// rank-sorted successor lists with multiplicity, a histogram + scan gives offsets.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.cuh"

int dfsim_topo_launch(dfsim_ctx *ctx, int32_t N, const int32_t *succ_off, const int32_t *succ_idx,
                      const int32_t *indeg, int32_t *topo, int32_t *n_ordered_dev, int32_t *left_scratch);

namespace {

constexpr unsigned long long kDangling = ~0ull;

__global__ void k_expand_nodes(dfsim_base_graph b, dfsim_expand_plan p, int32_t *indeg, int32_t *device,
                               int32_t *dev_count) {
    const int64_t n_clone = static_cast<int64_t>(p.replicas) * b.n_base;
    const int64_t total = n_clone + static_cast<int64_t>(p.n_collectives) * (p.ps ? 2 * p.replicas + 1 : 1);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int32_t r, deg, dev;
        if (i < n_clone) {
            const int k = static_cast<int>(i / b.n_base);
            const int v = static_cast<int>(i - static_cast<int64_t>(k) * b.n_base);
            r = p.clone_rank[i];
            deg = b.in_off[v + 1] - b.in_off[v];
            dev = b.remap[v] ? p.map_dev[k] : b.base_dev[v];
        } else if (!p.ps) {
            r = p.coll_rank[i - n_clone];
            deg = p.replicas;
            dev = p.fabric_dev;
        } else {  // PS nodes of gradient g: R pushes, the aggregate, R pulls
            const int64_t j = i - n_clone, per = 2 * static_cast<int64_t>(p.replicas) + 1;
            const int g = static_cast<int>(j / per), m = static_cast<int>(j - g * per);
            if (m < p.replicas) {
                r = p.push_rank[static_cast<int64_t>(g) * p.replicas + m];
                deg = 1;
                dev = p.up_dev[m];
            } else if (m == p.replicas) {
                r = p.coll_rank[g];
                deg = p.replicas;
                dev = p.ps_dev;
            } else {
                const int k = m - p.replicas - 1;
                r = p.pull_rank[static_cast<int64_t>(g) * p.replicas + k];
                deg = 1;
                dev = p.down_dev[k];
            }
        }
        indeg[r] = deg;
        device[r] = dev;
        atomicAdd(dev_count + dev, 1);
    }
}

// keys: [R * n_refs] clone refs, then [G * R] collective inputs
__global__ void k_expand_edges(dfsim_base_graph b, dfsim_expand_plan p, int64_t n_refs, unsigned long long *keys) {
    const int64_t n_clone_refs = static_cast<int64_t>(p.replicas) * b.n_base;  // iterate (k, v) pairs
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_clone_refs;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int k = static_cast<int>(i / b.n_base);
        const int v = static_cast<int>(i - static_cast<int64_t>(k) * b.n_base);
        const unsigned long long cons = static_cast<uint32_t>(p.clone_rank[i]);
        for (int j = b.in_off[v]; j < b.in_off[v + 1]; j++) {
            const int32_t u = b.in_src[j];
            unsigned long long key = kDangling;
            if (u >= 0) {
                const int32_t g = p.replicas > 1 ? b.marked[u] : -1;
                const int32_t prod = g < 0 ? p.clone_rank[static_cast<int64_t>(k) * b.n_base + u]
                                           : (p.ps ? p.pull_rank[static_cast<int64_t>(g) * p.replicas + k] : p.coll_rank[g]);
                key = (static_cast<unsigned long long>(static_cast<uint32_t>(prod)) << 32) | cons;
            }
            keys[static_cast<int64_t>(k) * n_refs + j] = key;
        }
        // collective inputs: the gradient's clone in replica k feeds its collective; in PS mode
        // it feeds push(g, k), which feeds aggregate(g), which feeds pull(g, k)
        const int32_t g = p.replicas > 1 ? b.marked[v] : -1;
        auto key = [](int32_t prod, int32_t cons) {
            return (static_cast<unsigned long long>(static_cast<uint32_t>(prod)) << 32) | static_cast<uint32_t>(cons);
        };
        if (g >= 0 && !p.ps) {
            keys[static_cast<int64_t>(p.replicas) * n_refs + static_cast<int64_t>(g) * p.replicas + k] =
                key(p.clone_rank[i], p.coll_rank[g]);
        } else if (g >= 0) {
            const int64_t gk = static_cast<int64_t>(g) * p.replicas + k;
            unsigned long long *out = keys + static_cast<int64_t>(p.replicas) * n_refs + 3 * gk;
            out[0] = key(p.clone_rank[i], p.push_rank[gk]);
            out[1] = key(p.push_rank[gk], p.coll_rank[g]);
            out[2] = key(p.coll_rank[g], p.pull_rank[gk]);
        }
    }
}

__global__ void k_csr_fill(int64_t n_keys, const unsigned long long *keys, int32_t *succ_idx, int32_t *out_count,
                           unsigned long long *n_valid) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_keys;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long key = keys[i];
        if (key == kDangling) continue;
        succ_idx[i] = static_cast<int32_t>(key & 0xffffffffu);
        atomicAdd(out_count + static_cast<int32_t>(key >> 32), 1);
        atomicAdd(n_valid, 1ull);
    }
}

__global__ void k_sources_flags(int32_t N, const int32_t *indeg, uint8_t *flags) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) flags[v] = indeg[v] == 0;
}

__global__ void k_queue_off(int32_t D, const int32_t *dev_count, int32_t *queue_off) {
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int d = 0; d < D; d++) { queue_off[d] = acc; acc += dev_count[d]; }
        queue_off[D] = acc;
    }
}

// ---- K1 for small classes in ONE launch (one 1024-thread CTA): the clone / edge phases of
// the kernels above, then a block radix sort of 32-bit (producer << bits | consumer) keys,
// the successor histogram + scan, the source compaction and the queue offsets, all through
// shared memory.  The multi-kernel path (radix sort, scan, select: ~20 launches) costs more
// in launch latency than in work at these sizes (C2 N = 4,619; C3 / C4 classes <= 9,474
// nodes and 13,568 edges), and a multi-class step launches it once per class.
constexpr int kSmallT = 1024, kSmallIPT = 16, kSmallKeys = kSmallT * kSmallIPT, kSmallN = 16384, kSmallD = 256;
using SmallSort = cub::BlockRadixSort<uint32_t, kSmallT, kSmallIPT>;
using SmallScan = cub::BlockScan<int32_t, kSmallT>;
struct SmallSmem {
    union {
        typename SmallSort::TempStorage sort;
        typename SmallScan::TempStorage scan;
        uint32_t keys[kSmallKeys];
    } u;
    int32_t count[kSmallN + 1];
    int32_t dev_count[kSmallD + 1];
    int32_t n_valid;
};

__device__ __forceinline__ int32_t block_exclusive_scan(SmallSmem &s, int32_t x, int32_t &total) {
    int32_t out;
    SmallScan(s.u.scan).ExclusiveSum(x, out, total);
    __syncthreads();
    return out;
}

__global__ void __launch_bounds__(kSmallT, 1)
    k_expand_small(dfsim_base_graph b, dfsim_expand_plan p, int32_t n_refs, int32_t N, int32_t n_keys, int32_t bits,
                   int32_t D, int32_t *succ_off, int32_t *succ_idx, int32_t *indeg, int32_t *device, int32_t *sources,
                   int32_t *queue_off, unsigned long long *small) {
    extern __shared__ __align__(16) unsigned char small_raw[];
    SmallSmem &s = *reinterpret_cast<SmallSmem *>(small_raw);
    const int tid = threadIdx.x;
    constexpr uint32_t kSent = 0xFFFFFFFFu;
    for (int i = tid; i <= N; i += kSmallT) s.count[i] = 0;
    for (int i = tid; i <= D; i += kSmallT) s.dev_count[i] = 0;
    if (tid == 0) s.n_valid = 0;
    for (int i = tid; i < kSmallKeys; i += kSmallT) s.u.keys[i] = kSent;
    __syncthreads();
    // nodes: in-degree, device, per-device counts (k_expand_nodes)
    const int32_t n_clone = p.replicas * b.n_base;
    for (int32_t i = tid; i < N; i += kSmallT) {
        int32_t r, deg, dev;
        if (i < n_clone) {
            const int k = i / b.n_base, v = i - k * b.n_base;
            r = p.clone_rank[i];
            deg = b.in_off[v + 1] - b.in_off[v];
            dev = b.remap[v] ? p.map_dev[k] : b.base_dev[v];
        } else if (!p.ps) {
            r = p.coll_rank[i - n_clone];
            deg = p.replicas;
            dev = p.fabric_dev;
        } else {
            const int32_t j = i - n_clone, per = 2 * p.replicas + 1;
            const int g = j / per, m = j - g * per;
            if (m < p.replicas) {
                r = p.push_rank[g * p.replicas + m];
                deg = 1;
                dev = p.up_dev[m];
            } else if (m == p.replicas) {
                r = p.coll_rank[g];
                deg = p.replicas;
                dev = p.ps_dev;
            } else {
                const int k = m - p.replicas - 1;
                r = p.pull_rank[g * p.replicas + k];
                deg = 1;
                dev = p.down_dev[k];
            }
        }
        indeg[r] = deg;
        device[r] = dev;
        atomicAdd(&s.dev_count[dev], 1);
    }
    // edges: packed keys at the same slots as k_expand_edges' 64-bit keys
    auto key = [bits, N](int32_t prod, int32_t cons) {
        DFSIM_CHECK(prod >= 0 && prod < N && cons >= 0 && cons < N, 13);
        return static_cast<uint32_t>(prod) << bits | static_cast<uint32_t>(cons);
    };
    for (int32_t i = tid; i < n_clone; i += kSmallT) {
        const int k = i / b.n_base, v = i - k * b.n_base;
        const int32_t cons = p.clone_rank[i];
        for (int j = b.in_off[v]; j < b.in_off[v + 1]; j++) {
            const int32_t u = b.in_src[j];
            uint32_t kk = kSent;
            if (u >= 0) {
                const int32_t g = p.replicas > 1 ? b.marked[u] : -1;
                const int32_t prod = g < 0 ? p.clone_rank[k * b.n_base + u]
                                           : (p.ps ? p.pull_rank[g * p.replicas + k] : p.coll_rank[g]);
                kk = key(prod, cons);
            }
            DFSIM_CHECK(k * n_refs + j < n_keys, 13);
            s.u.keys[k * n_refs + j] = kk;
        }
        const int32_t g = p.replicas > 1 ? b.marked[v] : -1;
        if (g >= 0 && !p.ps) {
            s.u.keys[p.replicas * n_refs + g * p.replicas + k] = key(p.clone_rank[i], p.coll_rank[g]);
        } else if (g >= 0) {
            const int32_t gk = g * p.replicas + k;
            uint32_t *out = s.u.keys + p.replicas * n_refs + 3 * gk;
            out[0] = key(p.clone_rank[i], p.push_rank[gk]);
            out[1] = key(p.push_rank[gk], p.coll_rank[g]);
            out[2] = key(p.coll_rank[g], p.pull_rank[gk]);
        }
    }
    __syncthreads();
    uint32_t kr[kSmallIPT];
#pragma unroll
    for (int i = 0; i < kSmallIPT; i++) kr[i] = s.u.keys[tid * kSmallIPT + i];
    __syncthreads();
    // valid keys < 2^(2 bits) - 1 (N < 2^bits), so the sentinel sorts last on the low 2*bits bits
    SmallSort(s.u.sort).Sort(kr, 0, 2 * bits);
    const uint32_t mask = (1u << bits) - 1;
    int valid = 0;
#pragma unroll
    for (int i = 0; i < kSmallIPT; i++) {
        const int pos = tid * kSmallIPT + i;
        if (kr[i] != kSent && pos < n_keys) {
            succ_idx[pos] = static_cast<int32_t>(kr[i] & mask);
            atomicAdd(&s.count[kr[i] >> bits], 1);
            valid++;
        }
    }
    if (valid) atomicAdd(&s.n_valid, valid);
    __syncthreads();
    // succ_off = exclusive scan of count[0..N] (blocked: thread t owns [t*P, t*P + P))
    {
        const int P = (N + 1 + kSmallT - 1) / kSmallT, lo = tid * P, hi = min(lo + P, N + 1);
        int32_t sum = 0;
        for (int i = lo; i < hi; i++) sum += s.count[i];
        int32_t total;
        int32_t run = block_exclusive_scan(s, sum, total);
        for (int i = lo; i < hi; i++) {
            succ_off[i] = run;
            run += s.count[i];
        }
    }
    // sources: nodes of in-degree 0, ascending (global indeg written by this block above)
    {
        const int P = (N + kSmallT - 1) / kSmallT, lo = tid * P, hi = min(lo + P, N);
        int32_t c = 0;
        for (int i = lo; i < hi; i++) c += indeg[i] == 0;
        int32_t total;
        int32_t at = block_exclusive_scan(s, c, total);
        for (int i = lo; i < hi; i++)
            if (indeg[i] == 0) sources[at++] = i;
        if (tid == 0) {
            small[0] = static_cast<unsigned long long>(s.n_valid);
            *reinterpret_cast<int32_t *>(small + 1) = total;
            int32_t acc = 0;
            for (int d = 0; d < D; d++) {
                queue_off[d] = acc;
                acc += s.dev_count[d];
            }
            queue_off[D] = acc;
        }
    }
}

size_t align_up(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

extern "C" int dfsim_expand_dp(dfsim_ctx *ctx, const dfsim_base_graph *base, const dfsim_expand_plan *plan,
                               int32_t *succ_off, int32_t *succ_idx, int64_t succ_capacity, int32_t *indeg,
                               int32_t *device, int32_t *sources, int32_t *queue_off, int32_t *topo,
                               int32_t n_devices, int64_t *n_edges_host, int32_t *n_sources_host,
                               int32_t *n_ordered_host) {
    if (!ctx || !base || !plan) return DFSIM_BAD_ARGUMENT;
    DFSIM_ARG_CHECK(ctx, (n_edges_host == nullptr) == (n_sources_host == nullptr) &&
                         (n_edges_host == nullptr) == (n_ordered_host == nullptr), "count outputs go together");
    DFSIM_ARG_CHECK(ctx, plan->replicas >= 1 && base->n_base >= 0, "bad replicas / base size");
    DFSIM_ARG_CHECK(ctx, plan->replicas > 1 || plan->n_collectives == 0, "collectives need replicas > 1");
    DFSIM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const int32_t R = plan->replicas, N0 = base->n_base, G = plan->n_collectives;
    DFSIM_ARG_CHECK(ctx, !plan->ps || (plan->push_rank && plan->pull_rank && plan->up_dev && plan->down_dev),
                    "PS mode needs push/pull ranks and link devices");
    const int64_t N = (int64_t)R * N0 + (int64_t)G * (plan->ps ? 2 * R + 1 : 1);
    DFSIM_ARG_CHECK(ctx, N < (1ll << 31), "expanded graph too large");
    // number of base refs: given by the caller, or read back from in_off[N0]
    int32_t n_refs32 = base->n_refs;
    if (n_refs32 < 0 && N0 > 0) {
        DFSIM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_small, base->in_off + N0, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        DFSIM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        n_refs32 = *static_cast<int32_t *>(ctx->host_small);
    }
    if (n_refs32 < 0) n_refs32 = 0;
    const int64_t n_refs = n_refs32;
    const int64_t n_keys = (int64_t)R * n_refs + (int64_t)G * R * (plan->ps ? 3 : 1);
    DFSIM_ARG_CHECK(ctx, succ_capacity >= n_keys, "succ_capacity below R*refs + G*R (3*G*R in PS mode)");

    int32_t bits = 1;
    while ((1ll << bits) <= N) bits++;  // N < 2^bits
    if (N <= kSmallN && n_keys <= kSmallKeys && n_devices <= kSmallD && 2 * bits <= 32 && N > 0 && n_refs32 >= 0 &&
        !std::getenv("DFSIM_K1_MULTI")) {
        void *p = nullptr;
        int rc = dfsim_scratch(ctx, align_up(64) + 4 * (size_t)(N + 1) + 256, &p);
        if (rc) return rc;
        auto *small = static_cast<unsigned long long *>(p);
        auto *left = reinterpret_cast<int32_t *>(static_cast<unsigned char *>(p) + align_up(64));
        static bool attr_set[64] = {};
        if (ctx->device < 64 && !attr_set[ctx->device]) {
            DFSIM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_expand_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     static_cast<int>(sizeof(SmallSmem))));
            attr_set[ctx->device] = true;
        }
        k_expand_small<<<1, kSmallT, sizeof(SmallSmem), ctx->stream>>>(*base, *plan, n_refs32, (int32_t)N,
                                                                         (int32_t)n_keys, bits, n_devices, succ_off,
                                                                         succ_idx, indeg, device, sources, queue_off,
                                                                         small);
        if ((rc = dfsim_after_launch(ctx, "k_expand_small"))) return rc;
        if (topo) {
            if ((rc = dfsim_topo_launch(ctx, (int32_t)N, succ_off, succ_idx, indeg, topo,
                                        reinterpret_cast<int32_t *>(small + 2), left))) return rc;
        }
        if (!n_edges_host) return DFSIM_OK;
        DFSIM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_small, small, 32, cudaMemcpyDeviceToHost, ctx->stream));
        DFSIM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        const unsigned long long *h = static_cast<const unsigned long long *>(ctx->host_small);
        *n_edges_host = (int64_t)h[0];
        *n_sources_host = *reinterpret_cast<const int32_t *>(h + 1);
        *n_ordered_host = topo ? *reinterpret_cast<const int32_t *>(h + 2) : (int32_t)N;
        return DFSIM_OK;
    }

    // cub temp sizes
    size_t sort_tmp = 0, scan_tmp = 0, sel_tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_tmp, (unsigned long long *)nullptr, (unsigned long long *)nullptr, (int)n_keys);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (int32_t *)nullptr, (int32_t *)nullptr, (int)(N + 1));
    cub::DeviceSelect::Flagged(nullptr, sel_tmp, cub::CountingInputIterator<int32_t>(0), (uint8_t *)nullptr,
                               (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    size_t tmp = std::max(sort_tmp, std::max(scan_tmp, sel_tmp));
    size_t off_keys_a = 0, off_keys_b = align_up(off_keys_a + 8 * (size_t)(n_keys + 1));
    size_t off_count = align_up(off_keys_b + 8 * (size_t)(n_keys + 1));
    size_t off_dev = align_up(off_count + 4 * (size_t)(N + 2));
    size_t off_flags = align_up(off_dev + 4 * (size_t)(n_devices + 1));
    size_t off_small = align_up(off_flags + (size_t)N + 1);
    size_t off_left = align_up(off_small + 64);
    size_t off_tmp = align_up(off_left + 4 * (size_t)(N + 1));
    void *p = nullptr;
    int rc = dfsim_scratch(ctx, off_tmp + tmp + 256, &p);
    if (rc) return rc;
    unsigned char *sc = static_cast<unsigned char *>(p);
    auto *keys_a = reinterpret_cast<unsigned long long *>(sc + off_keys_a);
    auto *keys_b = reinterpret_cast<unsigned long long *>(sc + off_keys_b);
    auto *count = reinterpret_cast<int32_t *>(sc + off_count);
    auto *dev_count = reinterpret_cast<int32_t *>(sc + off_dev);
    auto *flags = reinterpret_cast<uint8_t *>(sc + off_flags);
    auto *small = reinterpret_cast<unsigned long long *>(sc + off_small);
    auto *left = reinterpret_cast<int32_t *>(sc + off_left);
    void *cub_tmp = sc + off_tmp;

    const int threads = 256;
    auto blocks_for = [&](int64_t n) { int64_t b = (n + threads - 1) / threads; b = b < 1 ? 1 : b; return (unsigned)(b > 4096 ? 4096 : b); };
    DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(count, 0, 4 * (size_t)(N + 2), ctx->stream));
    DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(dev_count, 0, 4 * (size_t)(n_devices + 1), ctx->stream));
    DFSIM_CUDA_TRY(ctx, cudaMemsetAsync(small, 0, 64, ctx->stream));
    k_expand_nodes<<<blocks_for(N), threads, 0, ctx->stream>>>(*base, *plan, indeg, device, dev_count);
    if ((rc = dfsim_after_launch(ctx, "k_expand_nodes"))) return rc;
    if (n_keys > 0) {
        k_expand_edges<<<blocks_for((int64_t)R * N0), threads, 0, ctx->stream>>>(*base, *plan, n_refs, keys_a);
        if ((rc = dfsim_after_launch(ctx, "k_expand_edges"))) return rc;
        size_t t = tmp;
        DFSIM_CUDA_TRY(ctx, cub::DeviceRadixSort::SortKeys(cub_tmp, t, keys_a, keys_b, (int)n_keys, 0, 64, ctx->stream));
        ctx->launches++;
        k_csr_fill<<<blocks_for(n_keys), threads, 0, ctx->stream>>>(n_keys, keys_b, succ_idx, count, small);
        if ((rc = dfsim_after_launch(ctx, "k_csr_fill"))) return rc;
    }
    {
        size_t t = tmp;
        DFSIM_CUDA_TRY(ctx, cub::DeviceScan::ExclusiveSum(cub_tmp, t, count, succ_off, (int)(N + 1), ctx->stream));
        ctx->launches++;
    }
    k_sources_flags<<<blocks_for(N), threads, 0, ctx->stream>>>((int32_t)N, indeg, flags);
    if ((rc = dfsim_after_launch(ctx, "k_sources_flags"))) return rc;
    {
        size_t t = tmp;
        DFSIM_CUDA_TRY(ctx, cub::DeviceSelect::Flagged(cub_tmp, t, cub::CountingInputIterator<int32_t>(0), flags, sources,
                                                        reinterpret_cast<int32_t *>(small + 1), (int)N, ctx->stream));
        ctx->launches++;
    }
    k_queue_off<<<1, 32, 0, ctx->stream>>>(n_devices, dev_count, queue_off);
    if ((rc = dfsim_after_launch(ctx, "k_queue_off"))) return rc;
    if (topo && N > 0) {
        if ((rc = dfsim_topo_launch(ctx, (int32_t)N, succ_off, succ_idx, indeg, topo,
                                    reinterpret_cast<int32_t *>(small + 2), left))) return rc;
    }
    if (!n_edges_host) return DFSIM_OK;  // asynchronous re-expansion: counts are not read back
    DFSIM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_small, small, 32, cudaMemcpyDeviceToHost, ctx->stream));
    DFSIM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    const unsigned long long *h = static_cast<const unsigned long long *>(ctx->host_small);
    *n_edges_host = (int64_t)h[0];
    *n_sources_host = *reinterpret_cast<const int32_t *>(h + 1);
    *n_ordered_host = topo ? *reinterpret_cast<const int32_t *>(h + 2) : (int32_t)N;
    return DFSIM_OK;
}
