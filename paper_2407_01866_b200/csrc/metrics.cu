// metrics.cu -- kernel-5 reduction: the Eq. 8 L1 error map that drives
// error-guided Gaussian addition (sampling.cpp:77-94 add_distribution) and
// PSNR (metrics.cpp:12-27).
//
// The reference normalises with a sequential Kahan sum (sampling.cpp:14-23,
// 86).  A sequential recurrence has no exact parallel form, and one ulp of
// the total moves every normalised entry and with them the alias table's
// `scaled < 1.0` splits (sampling.cpp:114), so when the table goes to the
// host (igs_add_distribution with a host buffer, and every densification of
// igs_fit) the device writes the raw map and the host sums it in the
// reference's order (fit.cpp igs_internal_kahan_normalize).  The device-only
// form normalises by a fixed-order tree of error-free double-double
// additions (the nearly exact sum rounded once; within 1 ulp of Kahan's).
// HBM-bound: 24 B/px read + 8 B/px written.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <thread>

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

int igs_error_map(igs_ctx* ctx, const float* dev_rendered, int W, int H, double* dev_p, int normalize) {
    const size_t npx = (size_t)W * H;
    const int blocks = (int)std::min<size_t>(4 * ctx->sm_count, (npx + kRedThreads - 1) / kRedThreads);
    double* part = (double*)igs_scratch(ctx, 13, (size_t)(2 * blocks + 2) * sizeof(double));
    if (!part) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    error_map_kernel<<<blocks, kRedThreads, 0, ctx->stream>>>(dev_rendered, (const float*)ctx->target.p, npx, dev_p,
                                                              part);
    IGS_LAUNCHED(ctx);
    if (!normalize) return IGS_OK;  // the host normalises with the reference's Kahan total
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

// ---------------------------------------------------------------------------
// SSIM (metrics.cpp:33-112): 11x11 separable Gaussian window (sigma 1.5),
// replicate padding, C1 = 0.01^2, C2 = 0.03^2, mean over pixels, averaged
// over RGB.  The window is built on the host with the same libm exp and
// sequential normalisation as ssim_window(); both filter passes accumulate
// the 11 taps in order (no FMA), so each filtered value matches the
// reference bit for bit; the per-channel mean is the double-double total.
// ---------------------------------------------------------------------------
namespace {

struct Win11 {
    double w[11];
};

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// horizontal pass of the five maps x, y, xx, yy, xy for channel c
__global__ void ssim_h_kernel(const float* __restrict__ a, const float* __restrict__ b, int W, int H, int c, Win11 win,
                              double* __restrict__ tmp /* 5 * H * W */) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x, h = blockIdx.y;
    if (w >= W) return;
    double s[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < 11; ++i) {
        const size_t o = ((size_t)h * W + clampi(w - 5 + i, W - 1)) * 3 + c;
        const double x = (double)a[o], y = (double)b[o];
        const double wi = win.w[i];
        s[0] = __dadd_rn(s[0], __dmul_rn(wi, x));
        s[1] = __dadd_rn(s[1], __dmul_rn(wi, y));
        s[2] = __dadd_rn(s[2], __dmul_rn(wi, __dmul_rn(x, x)));
        s[3] = __dadd_rn(s[3], __dmul_rn(wi, __dmul_rn(y, y)));
        s[4] = __dadd_rn(s[4], __dmul_rn(wi, __dmul_rn(x, y)));
    }
    const size_t n = (size_t)W * H, p = (size_t)h * W + w;
#pragma unroll
    for (int m = 0; m < 5; ++m) tmp[m * n + p] = s[m];
}

// vertical pass + the SSIM map (metrics.cpp:95-103, op for op); the
// per-channel mean is summed on the host in pixel order (the reference's
// plain sequential `acc += num / den`)
__global__ void ssim_v_kernel(const double* __restrict__ tmp, int W, int H, Win11 win, double* __restrict__ map) {
    const size_t n = (size_t)W * H;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
        const int h = (int)(p / W), w = (int)(p % W);
        double s[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < 11; ++i) {
            const size_t q = (size_t)clampi(h - 5 + i, H - 1) * W + w;
            const double wi = win.w[i];
#pragma unroll
            for (int m = 0; m < 5; ++m) s[m] = __dadd_rn(s[m], __dmul_rn(wi, tmp[m * n + q]));
        }
        const double mx = s[0], my = s[1];
        const double var_x = __dsub_rn(s[2], __dmul_rn(mx, mx));
        const double var_y = __dsub_rn(s[3], __dmul_rn(my, my));
        const double cov = __dsub_rn(s[4], __dmul_rn(mx, my));
        const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mx), my), c1), __dadd_rn(__dmul_rn(2.0, cov), c2));
        const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), c1),
                                     __dadd_rn(__dadd_rn(var_x, var_y), c2));
        map[p] = __ddiv_rn(num, den);
    }
}

// sampling.cpp:44-67 image_gradient_magnitude: six Sobel responses with
// replicate padding, L2 norm, op for op (no FMA, IEEE sqrt).  One thread
// per pixel; 12 B/px read (neighbours from L1/L2), 8 B/px written.
__global__ void sobel_kernel(const float* __restrict__ img, int W, int H, double* __restrict__ mag) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x, h = blockIdx.y * blockDim.y + threadIdx.y;
    if (w >= W || h >= H) return;
    const int hm = clampi(h - 1, H - 1), hp = clampi(h + 1, H - 1), wm = clampi(w - 1, W - 1), wp = clampi(w + 1, W - 1);
    auto at = [&](int y, int x, int c) { return (double)__ldg(img + ((size_t)y * W + x) * 3 + c); };
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double tl = at(hm, wm, c), tc = at(hm, w, c), tr = at(hm, wp, c);
        const double ml = at(h, wm, c), mr = at(h, wp, c);
        const double bl = at(hp, wm, c), bc = at(hp, w, c), br = at(hp, wp, c);
        const double gx = __dsub_rn(__dadd_rn(__dadd_rn(tr, __dmul_rn(2.0, mr)), br),
                                    __dadd_rn(__dadd_rn(tl, __dmul_rn(2.0, ml)), bl));
        const double gy = __dsub_rn(__dadd_rn(__dadd_rn(bl, __dmul_rn(2.0, bc)), br),
                                    __dadd_rn(__dadd_rn(tl, __dmul_rn(2.0, tc)), tr));
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
    }
    mag[(size_t)h * W + w] = __dsqrt_rn(acc);
}

}  // namespace

int igs_ssim_dev(igs_ctx* ctx, const float* a, const float* b, int W, int H, double* out) {
    if (W < 11 || H < 11) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "ssim: image smaller than the 11x11 window");
    Win11 win;
    double sum = 0.0;
    for (int i = 0; i < 11; ++i) {  // metrics.cpp:33-44
        const double d = i - (11 - 1) / 2.0;
        win.w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += win.w[i];
    }
    for (double& v : win.w) v /= sum;
    const size_t n = (size_t)W * H;
    double* tmp = (double*)igs_scratch(ctx, 27, 5 * n * sizeof(double));
    double* map = (double*)igs_scratch(ctx, 28, 3 * n * sizeof(double));
    double* host = (double*)igs_pinned(ctx, 3 * n * sizeof(double));
    if (!tmp || !map || !host) return igs_fail(ctx, IGS_E_CUDA, "out of memory (ssim)");
    const int blocks = (int)std::min<size_t>(8 * ctx->sm_count, (n + 255) / 256);
    for (int c = 0; c < 3; ++c) {
        ssim_h_kernel<<<dim3((W + 127) / 128, H), 128, 0, ctx->stream>>>(a, b, W, H, c, win, tmp);
        IGS_LAUNCHED(ctx);
        ssim_v_kernel<<<blocks, 256, 0, ctx->stream>>>(tmp, W, H, win, map + c * n);
        IGS_LAUNCHED(ctx);
    }
    IGS_CUDA(ctx, cudaMemcpyAsync(host, map, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // metrics.cpp:95-106: acc += num / den in pixel order per channel (the
    // three channels are independent sums: one host thread each)
    double acc[3];
    auto channel = [&](int c) {
        double s2 = 0.0;
        const double* m = host + c * n;
        for (size_t i = 0; i < n; ++i) s2 += m[i];
        acc[c] = s2;
    };
    std::thread t1(channel, 1), t2(channel, 2);
    channel(0);
    t1.join();
    t2.join();
    double channel_sum = 0.0;
    for (int c = 0; c < 3; ++c) channel_sum += acc[c] / (double)n;
    *out = channel_sum / 3.0;
    return IGS_OK;
}

// image_gradient_magnitude of a device image into dev_mag (H*W doubles)
int igs_sobel_dev(igs_ctx* ctx, const float* img, int W, int H, double* dev_mag) {
    sobel_kernel<<<dim3((W + 31) / 32, (H + 7) / 8), dim3(32, 8), 0, ctx->stream>>>(img, W, H, dev_mag);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}
