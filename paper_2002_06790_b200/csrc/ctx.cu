// Context lifecycle, scratch management and error plumbing of the C-ABI.
#include <cstdio>
#include <new>

#include "internal.cuh"

extern "C" int32_t dfsim_abi_version(void) { return 1; }

extern "C" int dfsim_ctx_create(int32_t device, void *stream, dfsim_ctx **out) {
    if (!out) return DFSIM_BAD_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return DFSIM_CUDA;
    dfsim_ctx *ctx = new (std::nothrow) dfsim_ctx();
    if (!ctx) return DFSIM_CUDA;
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
        cudaMallocHost(&ctx->host_small, 4096) != cudaSuccess) {
        delete ctx;
        return DFSIM_CUDA;
    }
    *out = ctx;
    return DFSIM_OK;
}

extern "C" int dfsim_ctx_destroy(dfsim_ctx *ctx) {
    if (!ctx) return DFSIM_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto &e : ctx->per_stream) {
        if (e.stream) cudaStreamSynchronize(e.stream);
        if (e.scratch) cudaFree(e.scratch);
        if (e.aux) cudaFree(e.aux);
    }
    if (ctx->host_small) cudaFreeHost(ctx->host_small);
    delete ctx;
    return DFSIM_OK;
}

extern "C" int dfsim_ctx_set_stream(dfsim_ctx *ctx, void *stream) {
    if (!ctx) return DFSIM_BAD_ARGUMENT;
    ctx->stream = static_cast<cudaStream_t>(stream);
    return DFSIM_OK;
}

extern "C" int64_t dfsim_ctx_launch_count(const dfsim_ctx *ctx) { return ctx ? ctx->launches : 0; }

extern "C" const char *dfsim_ctx_last_error(const dfsim_ctx *ctx) {
    return ctx ? ctx->last_error.c_str() : "null context";
}

int dfsim_after_launch_base(dfsim_ctx *ctx, const char *what) {
    ctx->launches++;
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        ctx->last_error = std::string(what) + ": " + cudaGetErrorString(err);
        return DFSIM_CUDA;
    }
    return DFSIM_OK;
}

static int grow(dfsim_ctx *ctx, void **buf, size_t *have, size_t bytes, void **out) {
    if (bytes > *have) {
        DFSIM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        if (*buf) DFSIM_CUDA_TRY(ctx, cudaFree(*buf));
        *buf = nullptr;
        *have = 0;
        size_t grown = bytes + bytes / 4 + (1 << 20);
        DFSIM_CUDA_TRY(ctx, cudaMalloc(buf, grown));
        *have = grown;
    }
    *out = *buf;
    return DFSIM_OK;
}

static dfsim_stream_scratch &entry(dfsim_ctx *ctx) {
    std::lock_guard<std::mutex> guard(ctx->mu);
    for (auto &e : ctx->per_stream)
        if (e.stream == ctx->stream) return e;
    ctx->per_stream.emplace_back();
    ctx->per_stream.back().stream = ctx->stream;
    return ctx->per_stream.back();
}

int dfsim_scratch(dfsim_ctx *ctx, size_t bytes, void **out) {
    auto &e = entry(ctx);
    return grow(ctx, &e.scratch, &e.scratch_bytes, bytes, out);
}

int dfsim_aux(dfsim_ctx *ctx, size_t bytes, void **out) {
    auto &e = entry(ctx);
    return grow(ctx, &e.aux, &e.aux_bytes, bytes, out);
}
