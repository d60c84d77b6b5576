// ctx.cu -- the C-ABI (include/igs_b200.h): context, device memory,
// validation with the reference's error kinds/messages, and the host-side
// drivers of the kernels in render.cu / train.cu / cull.cu / bsp.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <random>
#include <string>

#include "igs_internal.cuh"

#include <atomic>

// contexts alive in the process (igs_coop_barriers)
static std::atomic<int> g_live_contexts{0};

using namespace igs_dev;

// train.cu
int igs_status_reset(igs_ctx* ctx);
int igs_stage_samples(igs_ctx* ctx, const uint32_t* host_pinned, uint32_t* dsidx, uint32_t ns);
int igs_stage_draws(igs_ctx* ctx, const unsigned long long* host_raw, uint32_t* dsidx, uint32_t ns);
int igs_publish(igs_ctx* ctx, const double* dloss, long long* host_res);
int igs_codec_pack(igs_ctx* ctx, uint16_t* dev_out);
int igs_codec_unpack(igs_ctx* ctx, const uint16_t* dev_in, const double* dev_src, uint32_t n, double* dev_out);
uint16_t igs_host_double_to_half(double d);
double igs_host_half_to_double(uint16_t h);
bool igs_host_encodable(double v);
extern "C" uint32_t igs_partition_source_size(igs_ctx* ctx);
int igs_forward_backward(igs_ctx* ctx, uint32_t ns, int k, int mode, const uint32_t* dev_sidx,
                         const double* dev_samples5, double* dev_loss, double inv_n, const double* fuse_lr4 = nullptr,
                         long long t = 0, bool* fused = nullptr, const StageJob* job = nullptr);
int igs_grad_check(igs_ctx* ctx);
int igs_adam_launch(igs_ctx* ctx, const double* lr4, long long t);
int igs_weights(igs_ctx* ctx, const double* q, const uint32_t* idx, size_t total, double* w);
int igs_blend_points(igs_ctx* ctx, const double* lq, const uint32_t* li, uint32_t npts, int kk, double* rgb);
// cull.cu
int igs_raster_culled(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out, uint32_t* topk);
int igs_cull_lists(igs_ctx* ctx, int W, int H, int k, uint32_t* ntiles, uint64_t* total, uint32_t* offsets,
                   uint32_t* members, double* tau);
// metrics.cu
int igs_error_map(igs_ctx* ctx, const float* dev_rendered, int W, int H, double* dev_p, int normalize);
extern "C" void igs_internal_kahan_normalize(double* p, size_t n);
int igs_psnr_dev(igs_ctx* ctx, const float* dev_a, const float* dev_b, size_t count, double* out);
int igs_ssim_dev(igs_ctx* ctx, const float* a, const float* b, int W, int H, double* out);
int igs_sobel_dev(igs_ctx* ctx, const float* img, int W, int H, double* dev_mag);
extern "C" void igs_internal_gradient_mixture(const double* mag, size_t n, double lambda, double* p);


// ---------------------------------------------------------------------------
// plumbing
// ---------------------------------------------------------------------------
int igs_fail(igs_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int igs_cuda_check(igs_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return IGS_OK;
    return igs_fail(ctx, IGS_E_CUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void* igs_scratch(igs_ctx* ctx, int slot, size_t bytes) {
    DevBuf& b = ctx->scratch[slot];
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return b.p;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = std::max(bytes, b.bytes * 3 / 2);
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
            cudaGetLastError();
            b.p = nullptr;
            return nullptr;
        }
        want = bytes;
    }
    b.bytes = want;
    return b.p;
}

static void* grow(DevBuf& b, size_t bytes) {
    if (b.bytes >= bytes) return b.p;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        return nullptr;
    }
    b.bytes = bytes;
    return b.p;
}

void* igs_pinned(igs_ctx* ctx, size_t bytes) {
    if (ctx->pinned_bytes >= bytes) return ctx->pinned;
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    if (cudaMallocHost(&ctx->pinned, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    ctx->pinned_bytes = bytes;
    return ctx->pinned;
}

int igs_ensure_image(igs_ctx* ctx, int w, int h) {
    if (!grow(ctx->image, (size_t)w * h * 3 * sizeof(float)))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (image)");
    ctx->img_w = w;
    ctx->img_h = h;
    return IGS_OK;
}

static int ensure_capacity(igs_ctx* ctx, uint32_t n, bool keep) {
    if (n <= ctx->cap) return IGS_OK;
    uint32_t cap = std::max<uint32_t>(n, ctx->cap + ctx->cap / 2);
    // slack: the sharded Adam's all-gather moves ceil(n/R) * R records
    cap = std::max<uint32_t>(cap, n + 64);
    double *p = nullptr, *g = nullptr, *m = nullptr, *v = nullptr;
    ScanRec* s = nullptr;
    ShadeRec* h = nullptr;
    const size_t rb = (size_t)cap * 8 * sizeof(double);
    if (cudaMalloc(&p, rb) != cudaSuccess || cudaMalloc(&g, rb) != cudaSuccess || cudaMalloc(&m, rb) != cudaSuccess ||
        cudaMalloc(&v, rb) != cudaSuccess || cudaMalloc(&s, (size_t)cap * sizeof(ScanRec)) != cudaSuccess ||
        cudaMalloc(&h, (size_t)cap * sizeof(ShadeRec)) != cudaSuccess) {
        cudaGetLastError();
        // release whatever this call did get; the resident set is untouched
        cudaFree(p);
        cudaFree(g);
        cudaFree(m);
        cudaFree(v);
        cudaFree(s);
        cudaFree(h);
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (Gaussian set)");
    }
    if (keep && ctx->n) {
        const size_t ob = (size_t)ctx->n * 8 * sizeof(double);
        IGS_CUDA(ctx, cudaMemcpyAsync(p, ctx->params, ob, cudaMemcpyDeviceToDevice, ctx->stream));
        IGS_CUDA(ctx, cudaMemcpyAsync(g, ctx->grads, ob, cudaMemcpyDeviceToDevice, ctx->stream));
        IGS_CUDA(ctx, cudaMemcpyAsync(m, ctx->adam_m, ob, cudaMemcpyDeviceToDevice, ctx->stream));
        IGS_CUDA(ctx, cudaMemcpyAsync(v, ctx->adam_v, ob, cudaMemcpyDeviceToDevice, ctx->stream));
        IGS_CUDA(ctx, cudaMemcpyAsync(s, ctx->scan, (size_t)ctx->n * sizeof(ScanRec), cudaMemcpyDeviceToDevice,
                                      ctx->stream));
        IGS_CUDA(ctx, cudaMemcpyAsync(h, ctx->shade, (size_t)ctx->n * sizeof(ShadeRec), cudaMemcpyDeviceToDevice,
                                      ctx->stream));
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    cudaFree(ctx->params);
    cudaFree(ctx->grads);
    cudaFree(ctx->adam_m);
    cudaFree(ctx->adam_v);
    cudaFree(ctx->scan);
    cudaFree(ctx->shade);
    ctx->params = p;
    ctx->grads = g;
    ctx->adam_m = m;
    ctx->adam_v = v;
    ctx->scan = s;
    ctx->shade = h;
    ctx->cap = cap;
    return IGS_OK;
}

static int host_to_dev(igs_ctx* ctx, void* dst, const void* src, size_t bytes) {
    // Stage through pinned memory so the copy is a true async DMA.
    void* pin = igs_pinned(ctx, bytes);
    if (!pin) {
        IGS_CUDA(ctx, cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
        return IGS_OK;
    }
    std::memcpy(pin, src, bytes);
    IGS_CUDA(ctx, cudaMemcpyAsync(dst, pin, bytes, cudaMemcpyHostToDevice, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

static int dev_to_host(igs_ctx* ctx, void* dst, const void* src, size_t bytes) {
    void* pin = igs_pinned(ctx, bytes);
    if (!pin) {
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        IGS_CUDA(ctx, cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        return IGS_OK;
    }
    IGS_CUDA(ctx, cudaMemcpyAsync(pin, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(dst, pin, bytes);
    return IGS_OK;
}

#define CHECK_CTX(ctx) \
    if (!(ctx)) return IGS_E_INVALID_PARAMETER

// renderer.cpp:12-14 require_nonempty
static int require_nonempty(igs_ctx* ctx) {
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "operation requires a non-empty GaussianSet");
    return IGS_OK;
}
static int require_k(igs_ctx* ctx, int k) {
    if (k < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "k must be >= 1");
    return IGS_OK;
}

extern "C" {

// internal (not in igs_b200.h): lets host-side drivers (fit.cpp) record errors
int igs_internal_fail(igs_ctx* ctx, int code, const char* msg) { return igs_fail(ctx, code, msg); }

int igs_ctx_create(int device, igs_ctx** out) {
    if (!out) return IGS_E_INVALID_PARAMETER;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return IGS_E_CUDA;
    }
    if (device < 0 || device >= ndev) return IGS_E_INVALID_PARAMETER;
    if (cudaSetDevice(device) != cudaSuccess) return IGS_E_CUDA;
    igs_ctx* ctx = new igs_ctx();
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&ctx->status, 4 * sizeof(long long)) != cudaSuccess) {
        delete ctx;
        return IGS_E_CUDA;
    }
    *out = ctx;
    g_live_contexts.fetch_add(1);
    return IGS_OK;
}

int igs_live_contexts() { return g_live_contexts.load(std::memory_order_relaxed); }

void igs_ctx_destroy(igs_ctx* ctx) {
    if (!ctx) return;
    g_live_contexts.fetch_sub(1);
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    igs_partition_release(ctx);
    igs_cull_free(ctx);
    igs_knn_free(ctx);
    igs_comm_release(ctx);
    igs_scan_free(ctx);
    cudaFree(ctx->params);
    cudaFree(ctx->grads);
    cudaFree(ctx->adam_m);
    cudaFree(ctx->adam_v);
    cudaFree(ctx->scan);
    cudaFree(ctx->shade);
    cudaFree(ctx->image.p);
    cudaFree(ctx->target.p);
    cudaFree(ctx->samples.p);
    cudaFree(ctx->alias_prob.p);
    cudaFree(ctx->alias_idx.p);
    cudaFree(ctx->status);
    cudaFree(ctx->flush.p);
    cudaFree(ctx->prof_dev_work);
    for (auto& b : ctx->scratch) cudaFree(b.p);
    for (auto& v : ctx->prof_ev)
        for (auto e : v) cudaEventDestroy(e);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    for (auto e : ctx->marks) cudaEventDestroy(e);
    for (auto e : ctx->timer)
        if (e) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (auto& b : ctx->async_pin)
        if (b.p) cudaFreeHost(b.p);
    for (auto e : ctx->async_ev)
        if (e) cudaEventDestroy(e);
    cudaStreamSynchronize(ctx->side);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
    cudaStreamDestroy(ctx->side);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* igs_last_error(const igs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int igs_sync(igs_ctx* ctx) {
    CHECK_CTX(ctx);
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

uint64_t igs_kernel_launches(const igs_ctx* ctx) { return ctx ? ctx->launches : 0; }

int igs_set_option(igs_ctx* ctx, int option, int64_t value) {
    CHECK_CTX(ctx);
    switch (option) {
        case IGS_OPT_CULL: ctx->opt_cull = value ? 1 : 0; return IGS_OK;
        case IGS_OPT_DETERMINISTIC: ctx->opt_deterministic = value ? 1 : 0; return IGS_OK;
        case IGS_OPT_RASTER: ctx->opt_raster = value ? 1 : 0; return IGS_OK;
        case IGS_OPT_SHARD_ADAM: ctx->opt_shard_adam = value ? 1 : 0; return IGS_OK;
        case IGS_OPT_TILE:
            if (value != 8 && value != 16 && value != 32)
                return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "tile must be 8, 16 or 32");
            ctx->opt_tile = (int)value;
            return IGS_OK;
    }
    return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "unknown option");
}

int64_t igs_get_option(const igs_ctx* ctx, int option) {
    if (!ctx) return -1;
    switch (option) {
        case IGS_OPT_CULL: return ctx->opt_cull;
        case IGS_OPT_DETERMINISTIC: return ctx->opt_deterministic;
        case IGS_OPT_RASTER: return ctx->opt_raster;
        case IGS_OPT_SHARD_ADAM: return ctx->opt_shard_adam;
        case IGS_OPT_TILE: return ctx->opt_tile;
    }
    return -1;
}

// ---- Gaussian set ----------------------------------------------------------
// (collective) every rank's slice of the Adam moments to every rank, after
// sharded updates (IGS_OPT_SHARD_ADAM); a no-op otherwise
static int gather_moments(igs_ctx* ctx) {
    if (!ctx->moments_local) return IGS_OK;
    const uint32_t R = (uint32_t)ctx->nranks, B = (ctx->n + R - 1) / R;
    int e;
    if ((e = igs_comm_allgather(ctx, ctx->adam_m, (size_t)B * 64))) return e;
    if ((e = igs_comm_allgather(ctx, ctx->adam_v, (size_t)B * 64))) return e;
    ctx->moments_local = false;
    return IGS_OK;
}

int igs_comm_gather_moments(igs_ctx* ctx) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    return gather_moments(ctx);
}

int igs_set_params(igs_ctx* ctx, const double* params8, uint32_t n) {
    CHECK_CTX(ctx);
    ctx->moments_local = false;  // fresh (zero) moments everywhere
    if (n && !params8) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "null params");
    cudaSetDevice(ctx->device);
    int e = ensure_capacity(ctx, n, false);
    if (e) return e;
    ctx->n = n;
    ctx->grads_valid = false;
    ctx->params_version++;
    // a partition outlives the set like the reference's BspPartition; renders
    // through it reject a changed count (bsp.cpp:278-282)
    if (n == 0) return IGS_OK;
    const size_t rb = (size_t)n * 8 * sizeof(double);
    if ((e = host_to_dev(ctx, ctx->params, params8, rb))) return e;
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->adam_m, 0, rb, ctx->stream));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->adam_v, 0, rb, ctx->stream));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->grads, 0, rb, ctx->stream));
    return igs_prepare_all(ctx, 0);
}

int igs_append_params(igs_ctx* ctx, const double* params8, uint32_t n) {
    CHECK_CTX(ctx);
    if (n == 0) return IGS_OK;
    if (!params8) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "null params");
    cudaSetDevice(ctx->device);
    const uint32_t old = ctx->n;
    // the slices move with n: re-replicate sharded moments first (collective)
    int e = gather_moments(ctx);
    if (e) return e;
    e = ensure_capacity(ctx, old + n, true);
    if (e) return e;
    const size_t rb = (size_t)n * 8 * sizeof(double);
    if ((e = host_to_dev(ctx, ctx->params + (size_t)old * 8, params8, rb))) return e;
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->adam_m + (size_t)old * 8, 0, rb, ctx->stream));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->adam_v + (size_t)old * 8, 0, rb, ctx->stream));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->grads + (size_t)old * 8, 0, rb, ctx->stream));
    ctx->n = old + n;
    ctx->grads_valid = false;
    ctx->params_version++;
    return igs_prepare_all(ctx, old);
}

int igs_get_params(igs_ctx* ctx, double* params8, uint32_t n) {
    CHECK_CTX(ctx);
    if (n != ctx->n) return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "parameter count mismatch");
    if (n == 0) return IGS_OK;
    return dev_to_host(ctx, params8, ctx->params, (size_t)n * 8 * sizeof(double));
}

uint32_t igs_num_gaussians(const igs_ctx* ctx) { return ctx ? ctx->n : 0; }

int igs_get_prepared(igs_ctx* ctx, double* scan6, uint32_t n) {
    CHECK_CTX(ctx);
    if (n != ctx->n) return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "count mismatch");
    if (n == 0) return IGS_OK;
    static_assert(sizeof(ScanRec) == 6 * sizeof(double), "ScanRec layout");
    return dev_to_host(ctx, scan6, ctx->scan, (size_t)n * sizeof(ScanRec));
}
const double* igs_device_params(const igs_ctx* ctx) { return ctx ? ctx->params : nullptr; }
const float* igs_device_image(const igs_ctx* ctx) { return ctx ? (const float*)ctx->image.p : nullptr; }
const double* igs_device_grads(const igs_ctx* ctx) { return ctx ? ctx->grads : nullptr; }

// ---- renderer ---------------------------------------------------------------
static int render_rows(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out_rgb, uint32_t* topk_idx) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    int e;
    if ((e = require_nonempty(ctx))) return e;
    if (W < 1 || H < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "render target must be at least 1x1");
    if ((e = require_k(ctx, k))) return e;
    if (row0 < 0 || row1 > H || row0 >= row1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bad row range");
    if ((e = igs_ensure_image(ctx, W, row1 - row0))) return e;
    ctx->img_h = row1 - row0;
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    uint32_t* dtopk = nullptr;
    if (topk_idx) {
        dtopk = (uint32_t*)igs_scratch(ctx, 16, (size_t)W * H * kk * sizeof(uint32_t));
        if (!dtopk) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (top-k dump)");
    }
    float* dout = (float*)ctx->image.p;
    if (ctx->opt_cull && ctx->opt_raster == 0 && kk <= 32) e = igs_raster_knn(ctx, W, H, k, row0, row1, dout, dtopk);
    else if (ctx->opt_cull) e = igs_raster_culled(ctx, W, H, k, row0, row1, dout, dtopk);
    else e = igs_raster_global(ctx, W, H, k, row0, row1, dout, dtopk);
    if (e) return e;
    if (out_rgb && (e = dev_to_host(ctx, out_rgb, dout, (size_t)W * (row1 - row0) * 3 * sizeof(float)))) return e;
    if (topk_idx &&
        (e = dev_to_host(ctx, topk_idx + (size_t)row0 * W * kk, dtopk + (size_t)row0 * W * kk,
                         (size_t)W * (row1 - row0) * kk * sizeof(uint32_t))))
        return e;
    return IGS_OK;
}

int igs_render_image(igs_ctx* ctx, int width, int height, int k, float* out_rgb, uint32_t* topk_idx) {
    return render_rows(ctx, width, height, k, 0, height, out_rgb, topk_idx);
}

int igs_render_image_rows(igs_ctx* ctx, int width, int height, int k, int row0, int row1, float* out_rgb) {
    return render_rows(ctx, width, height, k, row0, row1, out_rgb, nullptr);
}

static int points_topk(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t** dli, double** dlq,
                       int* kk_out) {
    int e;
    if ((e = require_nonempty(ctx))) return e;
    if ((e = require_k(ctx, k))) return e;
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    double* duv = (double*)igs_scratch(ctx, 17, (size_t)npts * 2 * sizeof(double));
    uint32_t* li = (uint32_t*)igs_scratch(ctx, 18, (size_t)npts * kk * sizeof(uint32_t));
    double* lq = (double*)igs_scratch(ctx, 19, (size_t)npts * kk * sizeof(double));
    if (!duv || !li || !lq) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (points)");
    if ((e = host_to_dev(ctx, duv, uv, (size_t)npts * 2 * sizeof(double)))) return e;
    if (ctx->opt_cull) e = igs_topk_knn(ctx, duv, npts, k, li, lq);
    else e = igs_topk_points(ctx, duv, npts, k, li, lq);
    if (e) return e;
    *dli = li;
    *dlq = lq;
    *kk_out = kk;
    return IGS_OK;
}

int igs_select_top_k(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* idx, double* weights,
                     int32_t* counts) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (npts == 0) return IGS_OK;
    uint32_t* li;
    double* lq;
    int kk, e;
    if ((e = points_topk(ctx, uv, npts, k, &li, &lq, &kk))) return e;
    const size_t total = (size_t)npts * kk;
    double* w = (double*)igs_scratch(ctx, 20, total * sizeof(double));
    if (!w) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    if ((e = igs_weights(ctx, lq, li, total, w))) return e;
    std::string tmp;
    if (idx && (e = dev_to_host(ctx, idx, li, total * sizeof(uint32_t)))) return e;
    if (weights && (e = dev_to_host(ctx, weights, w, total * sizeof(double)))) return e;
    if (counts) {
        uint32_t* h = idx;
        std::vector<uint32_t> local;
        if (!h) {
            local.resize(total);
            if ((e = dev_to_host(ctx, local.data(), li, total * sizeof(uint32_t)))) return e;
            h = local.data();
        }
        for (uint32_t p = 0; p < npts; ++p) {
            int c = 0;
            while (c < kk && h[(size_t)p * kk + c] != kNoIdx) ++c;
            counts[p] = c;
        }
    }
    return IGS_OK;
}

int igs_render_points(igs_ctx* ctx, const double* uv, uint32_t npts, int k, double* rgb) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (npts == 0) return IGS_OK;
    uint32_t* li;
    double* lq;
    int kk, e;
    if ((e = points_topk(ctx, uv, npts, k, &li, &lq, &kk))) return e;
    double* drgb = (double*)igs_scratch(ctx, 20, (size_t)npts * 3 * sizeof(double));
    if (!drgb) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    if ((e = igs_blend_points(ctx, lq, li, npts, kk, drgb))) return e;
    if (rgb) return dev_to_host(ctx, rgb, drgb, (size_t)npts * 3 * sizeof(double));
    return IGS_OK;
}

int igs_backward(igs_ctx* ctx, const double* samples5, uint32_t ns, int k, double* grads8) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    int e;
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "backward requires a non-empty GaussianSet");
    if ((e = require_k(ctx, k))) return e;
    // renderer.cpp:224-226: validate before any work
    for (uint32_t i = 0; i < ns; ++i)
        for (int c = 2; c < 5; ++c)
            if (!std::isfinite(samples5[(size_t)i * 5 + c]))
                return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "non-finite upstream gradient");
    if (ns == 0) {
        IGS_CUDA(ctx, cudaMemsetAsync(ctx->grads, 0, (size_t)ctx->n * 64, ctx->stream));
    } else {
        double* ds = (double*)igs_scratch(ctx, 15, (size_t)ns * 5 * sizeof(double));
        if (!ds) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
        if ((e = host_to_dev(ctx, ds, samples5, (size_t)ns * 5 * sizeof(double)))) return e;
        if ((e = igs_status_reset(ctx))) return e;
        if ((e = igs_forward_backward(ctx, ns, k, 1, nullptr, ds, nullptr, 1.0))) return e;
    }
    ctx->grads_valid = true;
    if (grads8) return dev_to_host(ctx, grads8, ctx->grads, (size_t)ctx->n * 64);
    return IGS_OK;
}

// ---- training -----------------------------------------------------------------
int igs_set_target(igs_ctx* ctx, const float* rgb, int width, int height) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (width < 1 || height < 1 || !rgb) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bad target image");
    const size_t bytes = (size_t)width * height * 3 * sizeof(float);
    if (!grow(ctx->target, bytes)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (target)");
    ctx->tgt_w = width;
    ctx->tgt_h = height;
    return host_to_dev(ctx, ctx->target.p, rgb, bytes);
}

}  // extern "C"

// In-place all-gather of `bytes` per rank: rank r's block sits at
// buf + r * bytes (train.cu's sample-ordered exchange of contributions).
extern "C" {


// Gradient + loss all-reduce, for the paths that do not exchange
// contributions (fp64-atomics mode, the brute-force fallback); after an
// exchange the gradients and the loss are already global.
static int allreduce_grads(igs_ctx* ctx, double* dev_loss) {
    if (igs_has_comm(ctx) && !ctx->exchanged) {  // a 1-rank communicator still runs (exercises the path on one GPU)
        int e;
        if ((e = igs_comm_allreduce_sum(ctx, ctx->grads, (size_t)ctx->n * 8))) return e;
        if (dev_loss && (e = igs_comm_allreduce_sum(ctx, dev_loss, 1))) return e;
    }
    return IGS_OK;
}

static int train_checks(igs_ctx* ctx, uint32_t ns, int k) {
    int e;
    if ((e = require_nonempty(ctx))) return e;
    if ((e = require_k(ctx, k))) return e;
    if (!ctx->target.p) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no target image (igs_set_target)");
    if (ns < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "sample count must be >= 1");
    return IGS_OK;
}

// status block layout on device: [0] first bad grad slot, [1] first bad
// constrained Gaussian, [2] first non-finite loss sample (LLONG_MAX = none)
static int read_status(igs_ctx* ctx, double* dev_loss, double* loss_out, int check_grads) {
    struct {
        long long st[4];
        double loss;
    } h;
    int e;
    if ((e = dev_to_host(ctx, h.st, ctx->status, sizeof(h.st)))) return e;
    h.loss = 0.0;
    if (dev_loss && (e = dev_to_host(ctx, &h.loss, dev_loss, sizeof(double)))) return e;
    ctx->knn_grown = h.st[3];
    if (h.st[2] != LLONG_MAX) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "training loss became non-finite");
    if (check_grads && h.st[0] != LLONG_MAX) {
        static const char* names[8] = {"mu_u", "mu_v", "theta", "s1", "s2", "r", "g", "b"};
        const long long slot = h.st[0];
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER,
                        "non-finite gradient for Gaussian " + std::to_string(slot / 8) + " parameter " +
                            names[slot % 8]);
    }
    if (h.st[1] != LLONG_MAX) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "non-finite Gaussian parameters");
    if (loss_out) *loss_out = h.loss;
    return IGS_OK;
}

// fit.cpp:87-89: the loss is the per-sample L1 losses summed in sample
// order, times 1/ns.  A sequential sum has no exact parallel form (and one
// device thread takes ~60 us for 10k terms), so the per-sample losses come
// to the host -- mirrored by the search epilogue into mapped memory on the
// asynchronous path -- and are summed here exactly as the reference does.
static double sequential_loss(const double* l, uint32_t n) {
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += l[i];
    return s * (1.0 / (double)n);
}

// the per-sample losses of the last forward/backward are on the device for
// every rank's samples (single rank, or the deterministic exchange)
static bool losses_complete(const igs_ctx* ctx) { return !igs_has_comm(ctx) || ctx->exchanged; }

static int host_loss_from_device(igs_ctx* ctx, uint32_t ns_total, double* loss) {
    std::vector<double> l(ns_total);
    const double* dl = (const double*)igs_scratch(ctx, 9, (size_t)std::max<uint32_t>(ns_total, 1) * sizeof(double));
    int e;
    if ((e = dev_to_host(ctx, l.data(), dl, (size_t)ns_total * sizeof(double)))) return e;
    *loss = sequential_loss(l.data(), ns_total);
    return IGS_OK;
}

static int upload_sidx(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, uint32_t** dev) {
    const uint64_t npx = (uint64_t)ctx->tgt_w * ctx->tgt_h;
    for (uint32_t i = 0; i < ns; ++i)
        if (sample_idx[i] >= npx) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "sample index outside the target");
    uint32_t* d = (uint32_t*)igs_scratch(ctx, 21, (size_t)ns * sizeof(uint32_t));
    if (!d) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    int e = host_to_dev(ctx, d, sample_idx, (size_t)ns * sizeof(uint32_t));
    *dev = d;
    return e;
}

int igs_train_step(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, int k, double* loss, double* grads8) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    int e;
    if ((e = train_checks(ctx, ns, k))) return e;
    uint32_t* dsidx;
    if ((e = upload_sidx(ctx, sample_idx, ns, &dsidx))) return e;
    double* dloss = (double*)igs_scratch(ctx, 14, 64 * sizeof(double));
    if ((e = igs_status_reset(ctx))) return e;
    const uint32_t ns_total = ns * (uint32_t)ctx->nranks;
    if ((e = igs_forward_backward(ctx, ns, k, 0, dsidx, nullptr, dloss, 1.0 / (double)ns_total))) return e;
    if ((e = allreduce_grads(ctx, dloss))) return e;
    if ((e = read_status(ctx, dloss, loss, 0))) return e;
    if (loss && losses_complete(ctx) && (e = host_loss_from_device(ctx, ns_total, loss))) return e;
    if (grads8) return dev_to_host(ctx, grads8, ctx->grads, (size_t)ctx->n * 64);
    return IGS_OK;
}

int igs_adam_step(igs_ctx* ctx, const double* lr4, long long t) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (t < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "Adam step index must be >= 1");
    if (!lr4) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "null learning rates");
    if (ctx->n == 0) return IGS_OK;
    int e;
    if ((e = gather_moments(ctx))) return e;
    if ((e = igs_status_reset(ctx))) return e;
    if ((e = igs_grad_check(ctx))) return e;
    if ((e = igs_adam_launch(ctx, lr4, t))) return e;
    return read_status(ctx, nullptr, nullptr, 1);
}

int igs_train_iteration(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, int k, const double* lr4,
                        long long t, double* loss) {
    CHECK_CTX(ctx);
    // = the asynchronous form plus its wait (after any outstanding ones)
    if (ctx->async_count)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "asynchronous iterations are outstanding (igs_train_wait)");
    int e;
    if ((e = igs_train_iteration_async(ctx, sample_idx, ns, k, lr4, t))) return e;
    return igs_train_wait(ctx, loss);
}

static int stage_rendered(igs_ctx* ctx, const float* rendered, int W, int H, const float** dev);

// Pinned staging for the async iterations: [slot] sample buffer, [2 + slot]
// result block {status[4], loss}.
static void* async_pinned(igs_ctx* ctx, int which, size_t bytes) {
    DevBuf& b = ctx->async_pin[which];
    if (b.bytes >= bytes) return b.p;
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMallocHost(&b.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    b.bytes = bytes;
    return b.p;
}

// One enqueued iteration; the samples are either indices (sample_idx) or
// raw engine outputs to draw from the uploaded alias table (raw2: 2 per
// sample, the fit driver).
static int train_iteration_enqueue(igs_ctx* ctx, const uint32_t* sample_idx, const unsigned long long* raw2,
                                   uint32_t ns, int k, const double* lr4, long long t) {
    int e;
    if (ctx->async_count >= 2) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "two iterations are already outstanding");
    if ((e = train_checks(ctx, ns, k))) return e;
    if (t < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "Adam step index must be >= 1");
    if (sample_idx) {
        const uint64_t npx = (uint64_t)ctx->tgt_w * ctx->tgt_h;
        for (uint32_t i = 0; i < ns; ++i)
            if (sample_idx[i] >= npx)
                return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "sample index outside the target");
    } else if (ctx->alias_n != (uint64_t)ctx->tgt_w * ctx->tgt_h) {
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no sampling table for the target");
    }
    const int slot = (ctx->async_head + ctx->async_count) & 1;
    const size_t in_bytes = sample_idx ? (size_t)ns * 4 : (size_t)ns * 16;
    void* pin = async_pinned(ctx, slot, in_bytes);
    long long* res = (long long*)async_pinned(ctx, 2 + slot, 64);
    // the device sample buffer is shared: the next iteration's copy into it
    // is ordered after this iteration's kernels on the stream
    uint32_t* dsidx = (uint32_t*)igs_scratch(ctx, 21, (size_t)ns * sizeof(uint32_t));
    double* dloss = (double*)igs_scratch(ctx, 14, 64 * sizeof(double));
    if (!pin || !res || !dsidx || !dloss) return igs_fail(ctx, IGS_E_CUDA, "out of memory (async iteration)");
    if (!ctx->async_ev[slot]) IGS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->async_ev[slot], cudaEventDisableTiming));
    dloss += slot;
    std::memcpy(pin, sample_idx ? (const void*)sample_idx : (const void*)raw2, in_bytes);
    // status reset + H2D (or device draws): run by the step's first kernel
    StageJob job;
    job.kind = sample_idx ? 2 : 3;
    job.status = ctx->status;
    job.host = pin;
    job.dsidx = dsidx;
    job.ns = ns;
    job.prob = (const double*)ctx->alias_prob.p;
    job.alias = (const uint32_t*)ctx->alias_idx.p;
    job.table_n = ctx->alias_n;
    const uint32_t ns_total = ns * (uint32_t)ctx->nranks;
    double* hl = (double*)async_pinned(ctx, 4 + slot, (size_t)std::max<uint32_t>(ns_total, 1) * sizeof(double));
    if (!hl) return igs_fail(ctx, IGS_E_CUDA, "out of memory (async iteration)");
    ctx->async_ns[slot] = ns_total;
    bool fused = false;
    ctx->loss_mirror = hl;
    ctx->loss_mirrored = false;
    e = igs_forward_backward(ctx, ns, k, 0, dsidx, nullptr, dloss, 1.0 / (double)ns_total, lr4, t, &fused, &job);
    ctx->loss_mirror = nullptr;
    if (e) return e;
    if (!ctx->loss_mirrored && losses_complete(ctx)) {
        // the search did not mirror them (other search paths, or the
        // multi-rank exchange, whose gathered array holds every rank's)
        const double* dl = (const double*)igs_scratch(ctx, 9, (size_t)ns_total * sizeof(double));
        IGS_CUDA(ctx, cudaMemcpyAsync(hl, dl, (size_t)ns_total * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (!losses_complete(ctx)) ctx->async_ns[slot] = 0;  // fp64-atomics multi-rank: the device's loss
    if (!fused) {
        if ((e = allreduce_grads(ctx, dloss))) return e;
        if ((igs_has_comm(ctx) || !ctx->grads_checked) && (e = igs_grad_check(ctx))) return e;
        if ((e = igs_adam_launch(ctx, lr4, t))) return e;
    }
    if ((e = igs_publish(ctx, dloss, res))) return e;  // D2H of status + loss
    IGS_CUDA(ctx, cudaEventRecord(ctx->async_ev[slot], ctx->stream));
    ctx->async_count++;
    return IGS_OK;
}

int igs_train_iteration_async(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, int k, const double* lr4,
                              long long t) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (!sample_idx) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "null sample indices");
    return train_iteration_enqueue(ctx, sample_idx, nullptr, ns, k, lr4, t);
}

// fit driver (fit.cpp), not part of the public header: the sampling table
// on the device, and iterations whose samples are drawn there
int igs_internal_set_sampler(igs_ctx* ctx, const double* prob, const uint32_t* alias, uint64_t n) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    ctx->alias_n = 0;
    if (!grow(ctx->alias_prob, n * 8) || !grow(ctx->alias_idx, n * 4))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (sampler)");
    int e;
    if ((e = host_to_dev(ctx, ctx->alias_prob.p, prob, n * 8))) return e;
    if ((e = host_to_dev(ctx, ctx->alias_idx.p, alias, n * 4))) return e;
    ctx->alias_n = n;
    return IGS_OK;
}

int igs_internal_train_iteration_async_raw(igs_ctx* ctx, const unsigned long long* raw2, uint32_t ns, int k,
                                           const double* lr4, long long t) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    return train_iteration_enqueue(ctx, nullptr, raw2, ns, k, lr4, t);
}

int igs_train_wait(igs_ctx* ctx, double* loss) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (ctx->async_count == 0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no outstanding iteration");
    const int slot = ctx->async_head;
    ctx->async_head ^= 1;
    ctx->async_count--;
    IGS_CUDA(ctx, cudaEventSynchronize(ctx->async_ev[slot]));
    const long long* st = (const long long*)ctx->async_pin[2 + slot].p;
    ctx->knn_grown = st[3];
    if (st[2] != LLONG_MAX) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "training loss became non-finite");
    if (st[0] != LLONG_MAX) {
        static const char* names[8] = {"mu_u", "mu_v", "theta", "s1", "s2", "r", "g", "b"};
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER,
                        "non-finite gradient for Gaussian " + std::to_string(st[0] / 8) + " parameter " +
                            names[st[0] % 8]);
    }
    if (st[1] != LLONG_MAX) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "non-finite Gaussian parameters");
    if (loss) {
        if (ctx->async_ns[slot])
            *loss = sequential_loss((const double*)ctx->async_pin[4 + slot].p, ctx->async_ns[slot]);
        else
            std::memcpy(loss, st + 4, sizeof(double));
    }
    return IGS_OK;
}

int igs_ssim(igs_ctx* ctx, const float* rendered, int width, int height, double* out) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    const float* dr;
    int e;
    if ((e = stage_rendered(ctx, rendered, width, height, &dr))) return e;
    return igs_ssim_dev(ctx, dr, (const float*)ctx->target.p, width, height, out);
}

int igs_upload_samples(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, uint32_t steps) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (!ctx->target.p) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no target image (igs_set_target)");
    const size_t total = (size_t)ns * steps;
    const uint64_t npx = (uint64_t)ctx->tgt_w * ctx->tgt_h;
    for (size_t i = 0; i < total; ++i)
        if (sample_idx[i] >= npx) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "sample index outside the target");
    if (!grow(ctx->samples, total * sizeof(uint32_t))) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    ctx->samples_ns = ns;
    ctx->samples_steps = steps;
    return host_to_dev(ctx, ctx->samples.p, sample_idx, total * sizeof(uint32_t));
}

int igs_train_iterations(igs_ctx* ctx, uint32_t steps, int k, const double* lr4, long long t0, double* losses) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    int e;
    const uint32_t ns = ctx->samples_ns;
    if ((e = train_checks(ctx, ns, k))) return e;
    if (ctx->samples_steps == 0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no uploaded samples");
    if (t0 < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "Adam step index must be >= 1");
    double* dloss = (double*)igs_scratch(ctx, 22, (size_t)std::max<uint32_t>(steps, 1) * sizeof(double));
    StageJob reset;  // the status reset, run by the first step's first kernel
    reset.kind = 1;
    reset.status = ctx->status;
    const uint32_t ns_total = ns * (uint32_t)ctx->nranks;
    // per-step per-sample losses (only when the caller wants the losses)
    double* step_losses = nullptr;
    if (losses) {
        step_losses = (double*)igs_scratch(ctx, 37, (size_t)std::max<uint32_t>(steps, 1) * ns_total * sizeof(double));
        if (!step_losses) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (losses)");
    }
    for (uint32_t s = 0; s < steps; ++s) {
        // step t uses uploaded slot (t-1) mod steps_uploaded
        const uint32_t slot = (uint32_t)((t0 + s - 1) % (long long)ctx->samples_steps);
        const uint32_t* dsidx = (const uint32_t*)ctx->samples.p + (size_t)slot * ns;
        if (s > 0) ctx->knn_grown = -1;  // no read-back inside the device loop: re-bucket
        bool fused = false;
        if ((e = igs_forward_backward(ctx, ns, k, 0, dsidx, nullptr, dloss + s, 1.0 / (double)ns_total, lr4, t0 + s,
                                      &fused, s == 0 ? &reset : nullptr)))
            return e;
        if (step_losses && losses_complete(ctx)) {
            const double* dl = (const double*)igs_scratch(ctx, 9, (size_t)ns_total * sizeof(double));
            IGS_CUDA(ctx, cudaMemcpyAsync(step_losses + (size_t)s * ns_total, dl, (size_t)ns_total * sizeof(double),
                                          cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if (!fused) {
            if ((e = allreduce_grads(ctx, dloss + s))) return e;
            if ((igs_has_comm(ctx) || !ctx->grads_checked) && (e = igs_grad_check(ctx))) return e;
            if ((e = igs_adam_launch(ctx, lr4, t0 + s))) return e;
        }
    }
    igs_timer_autostop(ctx);  // device time of the loop excludes the status readback
    if ((e = read_status(ctx, nullptr, nullptr, 1))) return e;
    if (!losses) return IGS_OK;
    if ((e = dev_to_host(ctx, losses, dloss, (size_t)steps * sizeof(double)))) return e;
    if (losses_complete(ctx)) {
        std::vector<double> l((size_t)steps * ns_total);
        if ((e = dev_to_host(ctx, l.data(), step_losses, l.size() * sizeof(double)))) return e;
        for (uint32_t s = 0; s < steps; ++s) losses[s] = sequential_loss(l.data() + (size_t)s * ns_total, ns_total);
    }
    return IGS_OK;
}

int igs_get_grads(igs_ctx* ctx, double* grads8, uint32_t n) {
    CHECK_CTX(ctx);
    if (n != ctx->n) return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "gradient count != Gaussian count");
    if (n == 0) return IGS_OK;
    return dev_to_host(ctx, grads8, ctx->grads, (size_t)n * 64);
}

int igs_set_grads(igs_ctx* ctx, const double* grads8, uint32_t n) {
    CHECK_CTX(ctx);
    if (n != ctx->n) return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "gradient count != Gaussian count");
    if (n == 0) return IGS_OK;
    ctx->grads_valid = true;
    ctx->grads_checked = false;
    return host_to_dev(ctx, ctx->grads, grads8, (size_t)n * 64);
}

int igs_get_adam_state(igs_ctx* ctx, double* m, double* v, uint32_t n) {
    CHECK_CTX(ctx);
    if (n != ctx->n) return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "state size mismatch");
    if (ctx->moments_local)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER,
                        "Adam moments are sharded across ranks: call igs_comm_gather_moments on every rank first");
    if (n == 0) return IGS_OK;
    int e;
    if (m && (e = dev_to_host(ctx, m, ctx->adam_m, (size_t)n * 64))) return e;
    if (v && (e = dev_to_host(ctx, v, ctx->adam_v, (size_t)n * 64))) return e;
    return IGS_OK;
}

int igs_set_adam_state(igs_ctx* ctx, const double* m, const double* v, uint32_t n) {
    CHECK_CTX(ctx);
    ctx->moments_local = false;
    if (n != ctx->n) return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "state size mismatch");
    if (n == 0) return IGS_OK;
    int e;
    if (m && (e = host_to_dev(ctx, ctx->adam_m, m, (size_t)n * 64))) return e;
    if (v && (e = host_to_dev(ctx, ctx->adam_v, v, (size_t)n * 64))) return e;
    return IGS_OK;
}

// ---- error map & metrics -----------------------------------------------------
static int stage_rendered(igs_ctx* ctx, const float* rendered, int W, int H, const float** dev) {
    if (W != ctx->tgt_w || H != ctx->tgt_h || !ctx->target.p)
        return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "rendered/target dimensions differ");
    if (!rendered) {
        if (!ctx->image.p || ctx->img_w != W || ctx->img_h != H)
            return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "rendered/target dimensions differ");
        *dev = (const float*)ctx->image.p;
        return IGS_OK;
    }
    const size_t bytes = (size_t)W * H * 3 * sizeof(float);
    float* d = (float*)igs_scratch(ctx, 23, bytes);
    if (!d) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    *dev = d;
    return host_to_dev(ctx, d, rendered, bytes);
}

int igs_add_distribution(igs_ctx* ctx, const float* rendered, int width, int height, double* p) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    const float* dr;
    int e;
    if ((e = stage_rendered(ctx, rendered, width, height, &dr))) return e;
    double* dp = (double*)igs_scratch(ctx, 12, (size_t)width * height * sizeof(double));
    if (!dp) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    if ((e = igs_error_map(ctx, dr, width, height, dp, p == nullptr))) return e;
    if (!p) return IGS_OK;
    // sampling.cpp:84-93: the raw L1 map comes back and is normalised by the
    // reference's sequential Kahan total on the host (bit-identical table)
    if ((e = dev_to_host(ctx, p, dp, (size_t)width * height * sizeof(double)))) return e;
    igs_internal_kahan_normalize(p, (size_t)width * height);
    return IGS_OK;
}

int igs_psnr(igs_ctx* ctx, const float* rendered, int width, int height, double* out) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    const float* dr;
    int e;
    if ((e = stage_rendered(ctx, rendered, width, height, &dr))) return e;
    return igs_psnr_dev(ctx, dr, (const float*)ctx->target.p, (size_t)width * height * 3, out);
}

// ---- the fit driver's multi-rank pieces (fit.cpp) ------------------------------
extern "C" void igs_internal_ranks(const igs_ctx* ctx, int* rank, int* nranks) {
    *rank = ctx->rank;
    *nranks = ctx->nranks;
}

// fit.cpp:34-37 render_current: build_partition(set, 64) + render_image_blocked
// into the context's image.  With R ranks every rank renders its band of
// ceil(H/R) rows and an in-place all-gather assembles the image on every
// rank, so the metrics and the densification table that follow are computed
// from the same image everywhere (replicated, identical bits).
extern "C" int igs_internal_eval_render(igs_ctx* ctx, int W, int H, int k) {
    int e;
    if ((e = igs_partition_build(ctx, 64))) return e;
    const int R = ctx->nranks;
    if (R == 1 || !igs_has_comm(ctx)) return igs_blocked_render_rows(ctx, W, H, k, 0, H);
    const int hb = (H + R - 1) / R;
    const int r0 = std::min(H, ctx->rank * hb), r1 = std::min(H, r0 + hb);
    if (!grow(ctx->image, (size_t)W * hb * R * 3 * sizeof(float)))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (image)");
    if ((e = igs_blocked_render_rows(ctx, W, H, k, r0, r1))) return e;
    return igs_comm_allgather(ctx, ctx->image.p, (size_t)W * hb * 3 * sizeof(float));
}

// ---- sampling tables (sampling.cpp:25-75) ----------------------------------------

// device copy of an arbitrary float image (img == nullptr: the target)
static int stage_image(igs_ctx* ctx, const float* img, int W, int H, const float** dev) {
    if (W < 1 || H < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "image must be at least 1x1");
    if (!img) {
        if (!ctx->target.p || ctx->tgt_w != W || ctx->tgt_h != H)
            return igs_fail(ctx, IGS_E_DIMENSION_MISMATCH, "no target image of these dimensions");
        *dev = (const float*)ctx->target.p;
        return IGS_OK;
    }
    const size_t bytes = (size_t)W * H * 3 * sizeof(float);
    float* d = (float*)igs_scratch(ctx, 23, bytes);
    if (!d) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    *dev = d;
    return host_to_dev(ctx, d, img, bytes);
}

int igs_image_gradient_magnitude(igs_ctx* ctx, const float* img, int width, int height, double* mag) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    const float* di;
    int e;
    if ((e = stage_image(ctx, img, width, height, &di))) return e;
    const size_t npx = (size_t)width * height;
    double* dm = (double*)igs_scratch(ctx, 12, npx * sizeof(double));
    if (!dm) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    if ((e = igs_sobel_dev(ctx, di, width, height, dm))) return e;
    if (mag) return dev_to_host(ctx, mag, dm, npx * sizeof(double));
    return IGS_OK;
}

int igs_gradient_mixture(igs_ctx* ctx, const float* img, int width, int height, double lambda, double* p) {
    CHECK_CTX(ctx);
    if (lambda < 0.0 || lambda > 1.0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "lambda must lie in [0,1]");
    if (!p) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "null output table");
    int e;
    // the magnitude on the device, the Kahan total and mixture on the host
    if ((e = igs_image_gradient_magnitude(ctx, img, width, height, p))) return e;
    igs_internal_gradient_mixture(p, (size_t)width * height, lambda, p);
    return IGS_OK;
}

// bsp.cpp:343-406 bench_render: random continuous points (Rng(seed), two
// next_double() per point), the global top-K baseline, then per n_max a
// build_partition and the blocked point query.  Device time per trial
// (CUDA events around the launch), scaled to ms per 10k points; mean and
// population std over the trials as the reference computes them.
// Candidates per point = |shell_members[locate_block(x)]| (the reference's
// count, bit-identical); the baseline row reports N (its global scan).
// The partition of the last n_max stays resident.
int igs_bench_render(igs_ctx* ctx, int pixels, const int* n_max_values, int n_values, uint64_t seed, int trials,
                     int warmup, igs_bench_row* rows) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "bench requires a non-empty GaussianSet");
    if (pixels < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "pixel count must be >= 1");
    if (trials < 1 || warmup < 0 || n_values < 0 || (n_values && !n_max_values) || !rows)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bench needs trials >= 1 and a row buffer");
    std::mt19937_64 rng(seed);
    std::vector<double> uv((size_t)pixels * 2);
    for (auto& x : uv) x = (double)(rng() >> 11) * 0x1.0p-53;  // rng.hpp next_double, u then v
    const uint32_t npts = (uint32_t)pixels;
    const int kk = (int)std::min<uint32_t>(10u, ctx->n);  // kDefaultTopK
    double* duv = (double*)igs_scratch(ctx, 38, (size_t)npts * 16);
    double* drgb = (double*)igs_scratch(ctx, 39, (size_t)npts * 24);
    uint32_t* li = (uint32_t*)igs_scratch(ctx, 18, (size_t)npts * kk * sizeof(uint32_t));
    double* lq = (double*)igs_scratch(ctx, 19, (size_t)npts * kk * sizeof(double));
    if (!duv || !drgb || !li || !lq) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bench)");
    int e;
    if ((e = host_to_dev(ctx, duv, uv.data(), uv.size() * sizeof(double)))) return e;
    cudaEvent_t a, b;
    IGS_CUDA(ctx, cudaEventCreate(&a));
    IGS_CUDA(ctx, cudaEventCreate(&b));
    const double to_10k = 10000.0 / pixels;
    auto time_trials = [&](auto&& body, double* mean_out, double* sd_out) -> int {
        std::vector<double> ms(trials);
        int e2;
        for (int t = 0; t < warmup; ++t)
            if ((e2 = body())) return e2;
        for (int t = 0; t < trials; ++t) {
            IGS_CUDA(ctx, cudaEventRecord(a, ctx->stream));
            if ((e2 = body())) return e2;
            IGS_CUDA(ctx, cudaEventRecord(b, ctx->stream));
            IGS_CUDA(ctx, cudaEventSynchronize(b));
            float f = 0.0f;
            IGS_CUDA(ctx, cudaEventElapsedTime(&f, a, b));
            ms[t] = f * to_10k;
        }
        double mean = 0.0;
        for (double v : ms) mean += v;
        mean /= trials;
        double var = 0.0;
        for (double v : ms) var += (v - mean) * (v - mean);
        *mean_out = mean;
        *sd_out = std::sqrt(var / trials);
        return IGS_OK;
    };
    rows[0] = {0, 0, 0.0, 0.0, (double)ctx->n};
    e = time_trials([&]() -> int {
        const int e2 = ctx->opt_cull && kk <= 32 ? igs_topk_knn(ctx, duv, npts, kk, li, lq)
                                                 : igs_topk_points(ctx, duv, npts, kk, li, lq);
        return e2 ? e2 : igs_blend_points(ctx, lq, li, npts, kk, drgb);
    }, &rows[0].mean_ms_per_10k, &rows[0].std_ms);
    for (int r = 0; !e && r < n_values; ++r) {
        if ((e = igs_partition_build(ctx, n_max_values[r]))) break;
        uint32_t nb = 0;
        uint64_t tot = 0;
        if ((e = igs_partition_info(ctx, &nb, &tot))) break;
        std::vector<uint32_t> off(nb + 1);
        std::vector<int32_t> blk(npts);
        if ((e = igs_partition_get(ctx, nullptr, nullptr, off.data(), nullptr))) break;
        if ((e = igs_locate_blocks(ctx, uv.data(), npts, blk.data()))) break;
        double cand = 0.0;
        for (uint32_t i = 0; i < npts; ++i) cand += (double)(off[blk[i] + 1] - off[blk[i]]);
        rows[r + 1] = {n_max_values[r], (int)nb, 0.0, 0.0, cand / pixels};
        e = time_trials([&]() { return igs_blocked_points_dev(ctx, duv, npts, kk, drgb); },
                        &rows[r + 1].mean_ms_per_10k, &rows[r + 1].std_ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return e;
}

int igs_tile_lists(igs_ctx* ctx, int width, int height, int k, uint32_t* ntiles, uint64_t* total, uint32_t* offsets,
                   uint32_t* members, double* tau) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    int e;
    if ((e = require_nonempty(ctx))) return e;
    if (width < 1 || height < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "render target must be at least 1x1");
    if ((e = require_k(ctx, k))) return e;
    return igs_cull_lists(ctx, width, height, k, ntiles, total, offsets, members, tau);
}


// ---- IGS2 container (codec.cpp) ------------------------------------------------
static void put16(uint8_t* b, uint16_t v) {
    b[0] = (uint8_t)(v & 0xff);
    b[1] = (uint8_t)(v >> 8);
}
static void put32(uint8_t* b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b[i] = (uint8_t)((v >> (8 * i)) & 0xff);
}
static uint16_t get16(const uint8_t* b) { return (uint16_t)(b[0] | (b[1] << 8)); }
static uint32_t get32(const uint8_t* b) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)b[i] << (8 * i);
    return v;
}

int igs_encode(igs_ctx* ctx, int with_partition, uint32_t width, uint32_t height, int k, uint8_t* out, size_t cap,
               size_t* size_out) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    // codec.cpp:142-154 validation, in the reference's order
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "cannot encode an empty GaussianSet");
    if (width == 0 || height == 0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "encoded dimensions must be positive");
    if (width > 0xffff || height > 0xffff)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "encoded dimensions exceed the u16 header fields");
    if (k < 1 || k > 0xffff) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "k out of range for the header");
    if (with_partition && !ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    if (with_partition && igs_partition_source_size(ctx) != ctx->n)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "partition was not built over this set");
    uint32_t nb = 0;
    int e;
    if (with_partition && (e = igs_partition_info(ctx, &nb, nullptr))) return e;
    const uint32_t n = ctx->n;
    const size_t total = 20 + 16ull * n + 8ull * nb;
    if (size_out) *size_out = total;
    if (!out || cap < total) return IGS_OK;  // size query
    uint16_t* dev = (uint16_t*)igs_scratch(ctx, 33, (size_t)n * 16);
    if (!dev) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (encode)");
    if ((e = igs_status_reset(ctx))) return e;
    if ((e = igs_codec_pack(ctx, dev))) return e;
    long long st[4];
    if ((e = dev_to_host(ctx, st, ctx->status, sizeof(st)))) return e;
    if (st[1] != LLONG_MAX)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "value of Gaussian parameter outside binary16 finite range");
    std::memcpy(out, "IGS2", 4);
    out[4] = 1;  // version
    out[5] = 0;  // flags
    put16(out + 6, (uint16_t)k);
    put16(out + 8, (uint16_t)width);
    put16(out + 10, (uint16_t)height);
    put32(out + 12, n);
    put32(out + 16, nb);
    if ((e = dev_to_host(ctx, out + 20, dev, (size_t)n * 16))) return e;  // little-endian halves
    if (nb) {
        std::vector<double> rects((size_t)nb * 4);
        if ((e = igs_partition_get(ctx, rects.data(), nullptr, nullptr, nullptr))) return e;
        uint8_t* b = out + 20 + 16ull * n;
        for (size_t i = 0; i < rects.size(); ++i) {
            if (!igs_host_encodable(rects[i]))
                return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "value of block corner outside binary16 finite range");
            put16(b + 2 * i, igs_host_double_to_half(rects[i]));
        }
    }
    return IGS_OK;
}

int igs_decode(igs_ctx* ctx, const uint8_t* bytes, size_t size, uint32_t* width, uint32_t* height, int* k,
               uint32_t* n_blocks) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    // codec.cpp:186-224, the reference's checks and messages
    if (!bytes || size < 20) return igs_fail(ctx, IGS_E_TRUNCATED, "file shorter than the 20-byte header");
    if (std::memcmp(bytes, "IGS2", 4) != 0) return igs_fail(ctx, IGS_E_BAD_MAGIC, "not an IGS2 file");
    if (bytes[4] != 1)
        return igs_fail(ctx, IGS_E_BAD_VERSION, "unsupported IGS2 version " + std::to_string((int)bytes[4]));
    const int kk = get16(bytes + 6);
    const uint32_t w = get16(bytes + 8), h = get16(bytes + 10), n = get32(bytes + 12), nb = get32(bytes + 16);
    if (n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "IGS2 file contains zero Gaussians");
    const size_t expected = 20 + 16ull * n + 8ull * nb;
    if (size != expected)
        return igs_fail(ctx, IGS_E_TRUNCATED,
                        "file length " + std::to_string(size) + " != expected " + std::to_string(expected));
    if (kk < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "header k must be >= 1");
    if (w == 0 || h == 0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "header dimensions must be positive");
    // decode() is a pure function in the reference: a file that fails
    // validation leaves the caller's set untouched.  Unpack into scratch,
    // check, and only then replace the resident set.
    uint16_t* dev = (uint16_t*)igs_scratch(ctx, 33, (size_t)n * 16);
    double* staged = (double*)igs_scratch(ctx, 36, (size_t)n * 8 * sizeof(double));
    if (!dev || !staged) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (decode)");
    int e;
    if ((e = host_to_dev(ctx, dev, bytes + 20, (size_t)n * 16))) return e;
    if ((e = igs_status_reset(ctx))) return e;
    if ((e = igs_codec_unpack(ctx, dev, nullptr, n, staged))) return e;
    long long st[4];
    if ((e = dev_to_host(ctx, st, ctx->status, sizeof(st)))) return e;
    if (st[1] != LLONG_MAX) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "non-finite Gaussian parameters");
    if ((e = ensure_capacity(ctx, n, false))) return e;
    const size_t rb = (size_t)n * 8 * sizeof(double);
    IGS_CUDA(ctx, cudaMemcpyAsync(ctx->params, staged, rb, cudaMemcpyDeviceToDevice, ctx->stream));
    // a new set: fresh moments and gradients, as igs_set_params
    ctx->moments_local = false;
    ctx->n = n;
    ctx->grads_valid = false;
    ctx->params_version++;
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->adam_m, 0, rb, ctx->stream));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->adam_v, 0, rb, ctx->stream));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->grads, 0, rb, ctx->stream));
    if ((e = igs_prepare_all(ctx, 0))) return e;
    if (nb) {
        // codec.cpp:213-223: stored corners -> rebuild_partition over the set
        std::vector<double> rects((size_t)nb * 4);
        const uint8_t* b = bytes + 20 + 16ull * n;
        for (size_t i = 0; i < rects.size(); ++i) rects[i] = igs_host_half_to_double(get16(b + 2 * i));
        if ((e = igs_partition_rebuild(ctx, rects.data(), nb))) return e;
    }
    if (width) *width = w;
    if (height) *height = h;
    if (k) *k = kk;
    if (n_blocks) *n_blocks = nb;
    return IGS_OK;
}

int igs_quantize_set(igs_ctx* ctx) {
    CHECK_CTX(ctx);
    cudaSetDevice(ctx->device);
    if (ctx->n == 0) return IGS_OK;
    int e;
    // quantize_set returns a new set (codec.cpp:69-81): round into scratch and
    // commit only when every record is finite
    double* staged = (double*)igs_scratch(ctx, 36, (size_t)ctx->n * 8 * sizeof(double));
    if (!staged) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (quantize)");
    if ((e = igs_status_reset(ctx))) return e;
    if ((e = igs_codec_unpack(ctx, nullptr, ctx->params, ctx->n, staged))) return e;
    long long st[4];
    if ((e = dev_to_host(ctx, st, ctx->status, sizeof(st)))) return e;
    if (st[1] != LLONG_MAX) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "non-finite Gaussian parameters");
    IGS_CUDA(ctx, cudaMemcpyAsync(ctx->params, staged, (size_t)ctx->n * 8 * sizeof(double), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    ctx->params_version++;
    return igs_prepare_all(ctx, 0);
}

}  // extern "C"
