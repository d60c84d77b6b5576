// metrics.cu -- kernel-5 reduction: the Eq. 8 L1 error map that drives
// error-guided Gaussian addition (sampling.cpp:77-94 add_distribution) and
// PSNR (metrics.cpp:12-27).
//
// The reference normalises with a sequential Kahan sum.  On the device the
// total is a fixed-order tree of error-free double-double additions
// (TwoSum), i.e. the (nearly) exact sum rounded once -- which is what a
// Kahan sum of well-conditioned positive terms returns, so the normalised
// table matches the reference bit for bit in practice and always within
// 1 ulp.  HBM-bound: 24 B/px read + 8 B/px written.
#include <cuda_runtime.h>

#include "igs_internal.cuh"

namespace {

constexpr int kRedThreads = 512;

struct DD {
    double hi, lo;
};

__device__ __forceinline__ DD dd_add(DD a, DD b) {
    const double s = __dadd_rn(a.hi, b.hi);
    const double bb = __dsub_rn(s, a.hi);
    const double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
    const double lo = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
    const double hi = __dadd_rn(s, lo);
    return {hi, __dsub_rn(lo, __dsub_rn(hi, s))};
}

__device__ __forceinline__ DD block_reduce(DD v) {
    __shared__ double sh[kRedThreads], sl[kRedThreads];
    sh[threadIdx.x] = v.hi;
    sl[threadIdx.x] = v.lo;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            const DD r = dd_add({sh[threadIdx.x], sl[threadIdx.x]}, {sh[threadIdx.x + s], sl[threadIdx.x + s]});
            sh[threadIdx.x] = r.hi;
            sl[threadIdx.x] = r.lo;
        }
        __syncthreads();
    }
    return {sh[0], sl[0]};
}

// e(px) = sum_ch |rendered - target| (float -> double), per-block DD partial.
__global__ void __launch_bounds__(kRedThreads) error_map_kernel(const float* __restrict__ a,
                                                               const float* __restrict__ b, size_t npx,
                                                               double* __restrict__ p, double* __restrict__ part) {
    DD acc = {0.0, 0.0};
    for (size_t i = (size_t)blockIdx.x * kRedThreads + threadIdx.x; i < npx; i += (size_t)gridDim.x * kRedThreads) {
        const double d0 = __dsub_rn((double)a[3 * i], (double)b[3 * i]);
        const double d1 = __dsub_rn((double)a[3 * i + 1], (double)b[3 * i + 1]);
        const double d2 = __dsub_rn((double)a[3 * i + 2], (double)b[3 * i + 2]);
        const double e = __dadd_rn(__dadd_rn(fabs(d0), fabs(d1)), fabs(d2));
        p[i] = e;
        acc = dd_add(acc, {e, 0.0});
    }
    const DD r = block_reduce(acc);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = r.hi;
        part[2 * blockIdx.x + 1] = r.lo;
    }
}

__global__ void __launch_bounds__(kRedThreads) sq_diff_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                             size_t count, double* __restrict__ part) {
    DD acc = {0.0, 0.0};
    for (size_t i = (size_t)blockIdx.x * kRedThreads + threadIdx.x; i < count; i += (size_t)gridDim.x * kRedThreads) {
        const double d = __dsub_rn((double)a[i], (double)b[i]);
        acc = dd_add(acc, {__dmul_rn(d, d), 0.0});
    }
    const DD r = block_reduce(acc);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = r.hi;
        part[2 * blockIdx.x + 1] = r.lo;
    }
}

__global__ void __launch_bounds__(kRedThreads) finish_sum_kernel(const double* __restrict__ part, int nparts,
                                                                double* __restrict__ out) {
    DD acc = {0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += kRedThreads) acc = dd_add(acc, {part[2 * i], part[2 * i + 1]});
    const DD r = block_reduce(acc);
    if (threadIdx.x == 0) *out = __dadd_rn(r.hi, r.lo);
}

// p <- p * (1/total), or uniform when the total is zero (sampling.cpp:87-92).
__global__ void normalize_kernel(double* __restrict__ p, size_t npx, const double* __restrict__ total) {
    const double t = *total;
    const double inv = __ddiv_rn(1.0, t);
    const double uni = __ddiv_rn(1.0, (double)npx);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += (size_t)gridDim.x * blockDim.x)
        p[i] = t > 0.0 ? __dmul_rn(p[i], inv) : uni;
}

}  // namespace

int igs_error_map(igs_ctx* ctx, const float* dev_rendered, int W, int H, double* dev_p) {
    const size_t npx = (size_t)W * H;
    const int blocks = (int)std::min<size_t>(4 * ctx->sm_count, (npx + kRedThreads - 1) / kRedThreads);
    double* part = (double*)igs_scratch(ctx, 13, (size_t)(2 * blocks + 2) * sizeof(double));
    if (!part) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    error_map_kernel<<<blocks, kRedThreads, 0, ctx->stream>>>(dev_rendered, (const float*)ctx->target.p, npx, dev_p,
                                                              part);
    IGS_LAUNCHED(ctx);
    double* total = part + 2 * blocks;
    finish_sum_kernel<<<1, kRedThreads, 0, ctx->stream>>>(part, blocks, total);
    IGS_LAUNCHED(ctx);
    normalize_kernel<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(dev_p, npx, total);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

int igs_psnr_dev(igs_ctx* ctx, const float* a, const float* b, size_t count, double* out) {
    const int blocks = (int)std::min<size_t>(4 * ctx->sm_count, (count + kRedThreads - 1) / kRedThreads);
    double* part = (double*)igs_scratch(ctx, 13, (size_t)(2 * blocks + 2) * sizeof(double));
    if (!part) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    sq_diff_kernel<<<blocks, kRedThreads, 0, ctx->stream>>>(a, b, count, part);
    IGS_LAUNCHED(ctx);
    double* total = part + 2 * blocks;
    finish_sum_kernel<<<1, kRedThreads, 0, ctx->stream>>>(part, blocks, total);
    IGS_LAUNCHED(ctx);
    double se = 0.0;
    IGS_CUDA(ctx, cudaMemcpyAsync(&se, total, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // metrics.cpp:24-26 (host libm log10, as the reference)
    if (se == 0.0) {
        *out = HUGE_VAL;
        return IGS_OK;
    }
    const double mse = se / (double)count;
    *out = 10.0 * std::log10(1.0 / mse);
    return IGS_OK;
}
