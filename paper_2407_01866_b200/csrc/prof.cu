// prof.cu -- device timing for bench.py: CUDA events on the context's own
// stream (torch's events would not see it), per-kernel-family launch
// timing, an L2 flush and the FP64 pipe microbenchmark used as the roofline
// denominator for the FP64-bound top-K scans (MEASURED_PEAKS.json carries
// only HBM and bf16 figures).
#include <cuda_runtime.h>

#include <algorithm>

#include "igs_internal.cuh"

static cudaEvent_t take_event(igs_ctx* ctx) {
    if (!ctx->ev_pool.empty()) {
        cudaEvent_t e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void igs_prof_begin(igs_ctx* ctx, int fam) {
    if (!ctx->prof_on) return;
    cudaEvent_t e = take_event(ctx);
    cudaEventRecord(e, ctx->stream);
    ctx->prof_ev[fam].push_back(e);
}

void igs_prof_end(igs_ctx* ctx, int fam, double host_work) {
    if (!ctx->prof_on) return;
    cudaEvent_t e = take_event(ctx);
    cudaEventRecord(e, ctx->stream);
    ctx->prof_ev[fam].push_back(e);
    ctx->prof_work[fam] += host_work;
}

unsigned long long* igs_prof_counter(igs_ctx* ctx, int fam) {
    return ctx->prof_on && ctx->prof_dev_work ? ctx->prof_dev_work + fam : nullptr;
}

namespace {
// Independent FP64 add/mul chains: 8 chains per thread keep the DADD/DMUL
// pipe saturated (latency hidden by ILP x occupancy).
__global__ void fp64_peak_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x[j] = __dmul_rn(x[j], a);
            x[j] = __dadd_rn(x[j], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}
}  // namespace

void igs_timer_autostop(igs_ctx* ctx) {
    if (!ctx->timer_armed) return;
    cudaEventRecord(ctx->timer[1], ctx->stream);
    ctx->timer_armed = false;
    ctx->timer_stopped = true;
}

extern "C" {

int igs_timer_begin(igs_ctx* ctx) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    for (auto& e : ctx->timer)
        if (!e) IGS_CUDA(ctx, cudaEventCreate(&e));
    IGS_CUDA(ctx, cudaEventRecord(ctx->timer[0], ctx->stream));
    ctx->timer_armed = true;
    ctx->timer_stopped = false;
    return IGS_OK;
}

int igs_timer_end(igs_ctx* ctx, float* ms) {
    if (!ctx || !ctx->timer[0]) return IGS_E_INVALID_PARAMETER;
    if (!ctx->timer_stopped) IGS_CUDA(ctx, cudaEventRecord(ctx->timer[1], ctx->stream));
    ctx->timer_armed = false;
    ctx->timer_stopped = false;
    IGS_CUDA(ctx, cudaEventSynchronize(ctx->timer[1]));
    IGS_CUDA(ctx, cudaEventElapsedTime(ms, ctx->timer[0], ctx->timer[1]));
    return IGS_OK;
}

int igs_timer_mark(igs_ctx* ctx, uint32_t idx) {
    if (!ctx || idx > (1u << 20)) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    while (ctx->marks.size() <= idx) {
        cudaEvent_t e;
        IGS_CUDA(ctx, cudaEventCreate(&e));
        ctx->marks.push_back(e);
    }
    IGS_CUDA(ctx, cudaEventRecord(ctx->marks[idx], ctx->stream));
    return IGS_OK;
}

int igs_timer_between(igs_ctx* ctx, uint32_t a, uint32_t b, float* ms) {
    if (!ctx || !ms || a >= ctx->marks.size() || b >= ctx->marks.size()) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    IGS_CUDA(ctx, cudaEventSynchronize(ctx->marks[b]));
    IGS_CUDA(ctx, cudaEventElapsedTime(ms, ctx->marks[a], ctx->marks[b]));
    return IGS_OK;
}

int igs_flush_l2(igs_ctx* ctx, size_t bytes) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    DevBuf& flush = ctx->flush;
    if (flush.bytes < bytes) {
        if (flush.p) cudaFree(flush.p);
        flush.p = nullptr;
        if (cudaMalloc(&flush.p, bytes) != cudaSuccess) {
            cudaGetLastError();
            flush.bytes = 0;
            return igs_fail(ctx, IGS_E_CUDA, "out of device memory (L2 flush buffer)");
        }
        flush.bytes = bytes;
    }
    IGS_CUDA(ctx, cudaMemsetAsync(flush.p, ++ctx->flush_salt & 0xff, bytes, ctx->stream));
    return IGS_OK;
}

// glibc-exact exp and sincos (glibc_math.cuh) evaluated on the device, so the
// tests can compare the device build (nvcc -fmad=false) with the host libm.
__global__ void libm_eval_kernel(const double* __restrict__ x, uint32_t n, double* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s, c;
    glibc_math::sincos(x[i], &s, &c);
    out[3 * (size_t)i] = glibc_math::exp(x[i]);
    out[3 * (size_t)i + 1] = s;
    out[3 * (size_t)i + 2] = c;
}

int igs_libm_eval(igs_ctx* ctx, const double* x, uint32_t n, double* out3) {
    if (!ctx || (n && (!x || !out3))) return IGS_E_INVALID_PARAMETER;
    if (n == 0) return IGS_OK;
    cudaSetDevice(ctx->device);
    double* dx = (double*)igs_scratch(ctx, 17, (size_t)n * 8);
    double* dout = (double*)igs_scratch(ctx, 20, (size_t)n * 24);
    if (!dx || !dout) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    IGS_CUDA(ctx, cudaMemcpyAsync(dx, x, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    libm_eval_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(dx, n, dout);
    IGS_LAUNCHED(ctx);
    IGS_CUDA(ctx, cudaMemcpyAsync(out3, dout, (size_t)n * 24, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

int igs_fp64_peak(igs_ctx* ctx, double* ops_per_s) {
    if (!ctx || !ops_per_s) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    double* out = (double*)igs_scratch(ctx, 14, 64);
    const int threads = 256, blocks = ctx->sm_count * 8, iters = 4096;
    cudaEvent_t a, b;
    IGS_CUDA(ctx, cudaEventCreate(&a));
    IGS_CUDA(ctx, cudaEventCreate(&b));
    fp64_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, 256, 0.999999, 1e-9);  // warm-up
    IGS_LAUNCHED(ctx);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        IGS_CUDA(ctx, cudaEventRecord(a, ctx->stream));
        fp64_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters, 0.999999, 1e-9);
        IGS_LAUNCHED(ctx);
        IGS_CUDA(ctx, cudaEventRecord(b, ctx->stream));
        IGS_CUDA(ctx, cudaEventSynchronize(b));
        float ms = 0;
        IGS_CUDA(ctx, cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double ops = (double)blocks * threads * iters * 8 * 2;
    *ops_per_s = ops / (best * 1e-3);
    return IGS_OK;
}

int igs_profile_enable(igs_ctx* ctx, int on) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int f = 0; f < IGS_PROF_FAMILIES; ++f) {
        for (auto e : ctx->prof_ev[f]) ctx->ev_pool.push_back(e);
        ctx->prof_ev[f].clear();
        ctx->prof_work[f] = 0;
    }
    if (!ctx->prof_dev_work) IGS_CUDA(ctx, cudaMalloc(&ctx->prof_dev_work, IGS_PROF_FAMILIES * 8));
    IGS_CUDA(ctx, cudaMemsetAsync(ctx->prof_dev_work, 0, IGS_PROF_FAMILIES * 8, ctx->stream));
    ctx->prof_on = on != 0;
    return IGS_OK;
}

int igs_profile_read(igs_ctx* ctx, int family, double* ms, uint64_t* launches, double* work) {
    if (!ctx || family < 0 || family >= IGS_PROF_FAMILIES) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    double total = 0;
    const auto& ev = ctx->prof_ev[family];
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
        float t = 0;
        IGS_CUDA(ctx, cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
        total += t;
    }
    unsigned long long dw = 0;
    if (ctx->prof_dev_work)
        IGS_CUDA(ctx, cudaMemcpy(&dw, ctx->prof_dev_work + family, 8, cudaMemcpyDeviceToHost));
    if (ms) *ms = total;
    if (launches) *launches = ev.size() / 2;
    if (work) *work = ctx->prof_work[family] + (double)dw;
    return IGS_OK;
}

}  // extern "C"
