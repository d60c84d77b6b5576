// render.cu -- kernel 1 (preprocess) and kernel 3 (exact top-K raster),
// brute-force global mode.  Certified tile culling lives in cull.cu.
//
// Reference: renderer.cpp:32-51 (PreparedSet), :53-74 (select_top_k_entries),
// :76-89 (blend_entries), :161-191 (render_image_impl).
#include <cuda_runtime.h>

#include <algorithm>

#include "igs_internal.cuh"

using namespace igs_dev;

namespace {

// ---------------------------------------------------------------------------
// Kernel 1: PreparedSet.  One thread per Gaussian: glibc-exact sincos,
// IEEE reciprocals, 2 x 48 B records written with 16-B stores.
// ---------------------------------------------------------------------------
__global__ void prepare_kernel(const double* __restrict__ params, ScanRec* __restrict__ scan,
                               ShadeRec* __restrict__ shade, uint32_t first, uint32_t n) {
    const uint32_t i = first + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    prepare_one(params, i, scan, shade);
}

constexpr int kTile = 16;      // 16x16 pixel tile per CTA (256 threads)
constexpr int kChunk = 256;    // candidates staged per smem round (12 KB)

// Stage kChunk scan records [base, base+cnt) into shared memory with
// coalesced 16-B loads (3 per record).
__device__ __forceinline__ void stage_chunk(ScanRec* sm, const ScanRec* __restrict__ scan, uint32_t base,
                                            uint32_t cnt, int tid, int nthreads) {
    const double2* src = reinterpret_cast<const double2*>(scan + base);
    double2* dst = reinterpret_cast<double2*>(sm);
    for (uint32_t e = tid; e < cnt * 3; e += nthreads) dst[e] = __ldg(src + e);
}

// ---------------------------------------------------------------------------
// Kernel 3 (global, brute force): one thread per pixel, every candidate of
// the set streamed through shared memory in index order.
// ---------------------------------------------------------------------------
template <int KCAP>
__global__ void __launch_bounds__(256) raster_global_kernel(const ScanRec* __restrict__ scan,
                                                            const ShadeRec* __restrict__ shade, uint32_t n,
                                                            int W, int H, int row0, int row1, int kk,
                                                            float* __restrict__ out, uint32_t* __restrict__ topk) {
    __shared__ ScanRec sm[kChunk];
    const int tid = threadIdx.y * kTile + threadIdx.x;
    const int px = blockIdx.x * kTile + threadIdx.x;
    const int py = row0 + blockIdx.y * kTile + threadIdx.y;
    const bool live = px < W && py < row1;
    const double x = center(px, W), y = center(py, H);
    TopK<KCAP> t;
    t.init(kk);
    for (uint32_t base = 0; base < n; base += kChunk) {
        const uint32_t cnt = min((uint32_t)kChunk, n - base);
        __syncthreads();
        stage_chunk(sm, scan, base, cnt, tid, kTile * kTile);
        __syncthreads();
        // every thread runs the loop (warp votes need the full warp); only live
        // threads write results
#pragma unroll 1
            for (uint32_t c = 0; c < cnt; ++c) {
                const double q = maha(sm[c], x, y);
                if (__any_sync(0xffffffffu, q <= t.tq()))
                    if (q <= t.tq()) t.offer(q, base + c);
            }
    }
    if (!live) return;
    double col[3];
    blend_topk(t, shade, col);
    const size_t o = ((size_t)(py - row0) * W + px);
    out[o * 3 + 0] = clamp01f(col[0]);
    out[o * 3 + 1] = clamp01f(col[1]);
    out[o * 3 + 2] = clamp01f(col[2]);
    if (topk) store_topk(t, (double*)nullptr, topk + ((size_t)py * W + px) * kk);
}

// ---------------------------------------------------------------------------
// Point queries (top-K at arbitrary (u,v)): split-candidate scan.  Grid
// (point blocks, splits); each CTA scans one contiguous candidate range and
// writes a partial top-K per point; the merge kernel keeps the best kk of
// the union (order-independent because (q, idx) is a strict total order).
// ---------------------------------------------------------------------------
constexpr int kPtThreads = 128;

template <int KCAP>
__global__ void __launch_bounds__(kPtThreads) points_partial_kernel(const ScanRec* __restrict__ scan, uint32_t n,
                                                                    const double* __restrict__ uv, uint32_t npts,
                                                                    int kk, uint32_t per_split,
                                                                    double* __restrict__ pq, uint32_t* __restrict__ pi) {
    __shared__ ScanRec sm[kChunk];
    const int tid = threadIdx.x;
    const uint32_t p = blockIdx.x * kPtThreads + tid;
    const bool live = p < npts;
    const uint32_t c0 = blockIdx.y * per_split;
    const uint32_t c1 = min(n, c0 + per_split);
    double x = 0.0, y = 0.0;
    if (live) {
        x = uv[2 * (size_t)p];
        y = uv[2 * (size_t)p + 1];
    }
    TopK<KCAP> t;
    t.init(kk);
    for (uint32_t base = c0; base < c1; base += kChunk) {
        const uint32_t cnt = min((uint32_t)kChunk, c1 - base);
        __syncthreads();
        stage_chunk(sm, scan, base, cnt, tid, kPtThreads);
        __syncthreads();
        // every thread runs the loop (warp votes need the full warp); only live
        // threads write results
#pragma unroll 1
            for (uint32_t c = 0; c < cnt; ++c) {
                const double q = maha(sm[c], x, y);
                if (__any_sync(0xffffffffu, q <= t.tq()))
                    if (q <= t.tq()) t.offer(q, base + c);
            }
    }
    if (!live) return;
    const size_t o = ((size_t)blockIdx.y * npts + p) * kk;
    store_topk(t, pq + o, pi + o);
}

template <int KCAP>
__global__ void points_merge_kernel(const double* __restrict__ pq, const uint32_t* __restrict__ pi, uint32_t npts,
                                    int kk, int splits, double* __restrict__ oq, uint32_t* __restrict__ oi) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    TopK<KCAP> t;
    t.init(kk);
    for (int s = 0; s < splits; ++s) {
        const size_t o = ((size_t)s * npts + p) * kk;
        for (int j = 0; j < kk; ++j) {
            const uint32_t ci = pi[o + j];
            if (ci == kNoIdx) break;
            t.offer(pq[o + j], ci);
        }
    }
    store_topk(t, oq + (size_t)p * kk, oi + (size_t)p * kk);
}

// ---------------------------------------------------------------------------
// Generic path for kk > 32: the reference's insertion algorithm verbatim in
// per-item global scratch.  Items are points (uv != null) or pixels.
// ---------------------------------------------------------------------------
__global__ void topk_generic_kernel(const ScanRec* __restrict__ scan, uint32_t n, const double* __restrict__ uv,
                                    uint32_t nitems, int W, int H, int row0, int kk, double* __restrict__ oq,
                                    uint32_t* __restrict__ oi) {
    const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= nitems) return;
    double x, y;
    if (uv) {
        x = uv[2 * (size_t)it];
        y = uv[2 * (size_t)it + 1];
    } else {
        const int px = it % W, py = row0 + it / W;
        x = center(px, W);
        y = center(py, H);
    }
    double* q = oq + (size_t)it * kk;
    uint32_t* ix = oi + (size_t)it * kk;
    int cnt = 0;
    for (uint32_t c = 0; c < n; ++c) {
        const double cq = maha(scan[c], x, y);
        if (cnt == kk) {
            if (cq > q[cnt - 1] || (cq == q[cnt - 1] && c > ix[cnt - 1])) continue;
            --cnt;
        }
        int pos = cnt;
        while (pos > 0 && (cq < q[pos - 1] || (cq == q[pos - 1] && c < ix[pos - 1]))) {
            q[pos] = q[pos - 1];
            ix[pos] = ix[pos - 1];
            --pos;
        }
        q[pos] = cq;
        ix[pos] = c;
        ++cnt;
    }
    for (int j = cnt; j < kk; ++j) {
        q[j] = __longlong_as_double(0x7ff0000000000000LL);
        ix[j] = kNoIdx;
    }
}

// Blend from (q, idx) lists: image pixels (clamped float) for the generic path.
__global__ void blend_list_image_kernel(const double* __restrict__ lq, const uint32_t* __restrict__ li,
                                        const ShadeRec* __restrict__ shade, uint32_t nitems, int W, int row0,
                                        int kk, float* __restrict__ out, uint32_t* __restrict__ topk) {
    const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= nitems) return;
    double total = 0.0, ar = 0.0, ag = 0.0, ab = 0.0;
    for (int j = 0; j < kk; ++j) {
        const uint32_t ci = li[(size_t)it * kk + j];
        if (ci == kNoIdx) break;
        const double w = glibc_math::exp(__dmul_rn(-0.5, lq[(size_t)it * kk + j]));
        const ShadeRec s = shade[ci];
        total = __dadd_rn(total, w);
        ar = __dadd_rn(ar, __dmul_rn(w, s.r));
        ag = __dadd_rn(ag, __dmul_rn(w, s.g));
        ab = __dadd_rn(ab, __dmul_rn(w, s.b));
    }
    const double inv = __ddiv_rn(1.0, __dadd_rn(kNormEps, total));
    out[(size_t)it * 3 + 0] = clamp01f(__dmul_rn(ar, inv));
    out[(size_t)it * 3 + 1] = clamp01f(__dmul_rn(ag, inv));
    out[(size_t)it * 3 + 2] = clamp01f(__dmul_rn(ab, inv));
    if (topk) {
        const size_t o = ((size_t)row0 * W + it) * kk;
        for (int j = 0; j < kk; ++j) topk[o + j] = li[(size_t)it * kk + j];
    }
}

template <int KCAP>
int launch_points(igs_ctx* ctx, const double* uv, uint32_t npts, int kk, uint32_t* oi, double* oq) {
    const uint32_t n = ctx->n;
    const uint32_t pblocks = (npts + kPtThreads - 1) / kPtThreads;
    // enough CTAs for ~4 waves of 148 SMs, each split >= 1024 candidates
    uint32_t splits = std::max<uint32_t>(1, (4u * ctx->sm_count + pblocks - 1) / pblocks);
    splits = std::min<uint32_t>(splits, std::max<uint32_t>(1, n / 1024));
    const uint32_t per = (n + splits - 1) / splits;
    splits = (n + per - 1) / per;
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    if (splits == 1) {
        points_partial_kernel<KCAP><<<dim3(pblocks, 1), kPtThreads, 0, ctx->stream>>>(ctx->scan, n, uv, npts, kk,
                                                                                        per, oq, oi);
        IGS_LAUNCHED(ctx);
        igs_prof_end(ctx, IGS_PROF_SCAN, (double)npts * n);
        return IGS_OK;
    }
    const size_t part = (size_t)splits * npts * kk;
    double* pq = (double*)igs_scratch(ctx, 10, part * sizeof(double));
    uint32_t* pi = (uint32_t*)igs_scratch(ctx, 11, part * sizeof(uint32_t));
    if (!pq || !pi) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (point scan)");
    points_partial_kernel<KCAP><<<dim3(pblocks, splits), kPtThreads, 0, ctx->stream>>>(ctx->scan, n, uv, npts, kk,
                                                                                         per, pq, pi);
    IGS_LAUNCHED(ctx);
    points_merge_kernel<KCAP><<<(npts + 127) / 128, 128, 0, ctx->stream>>>(pq, pi, npts, kk, (int)splits, oq, oi);
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_SCAN, (double)npts * n);
    return IGS_OK;
}

template <int KCAP>
int launch_raster(igs_ctx* ctx, int W, int H, int row0, int row1, int kk, float* out, uint32_t* topk) {
    dim3 grid((W + kTile - 1) / kTile, (row1 - row0 + kTile - 1) / kTile);
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    raster_global_kernel<KCAP><<<grid, dim3(kTile, kTile), 0, ctx->stream>>>(ctx->scan, ctx->shade, ctx->n, W, H,
                                                                              row0, row1, kk, out, topk);
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_SCAN, (double)W * (row1 - row0) * ctx->n);
    return IGS_OK;
}

}  // namespace

int igs_prepare_all(igs_ctx* ctx, uint32_t first) {
    if (ctx->n <= first) return IGS_OK;
    const uint32_t cnt = ctx->n - first;
    prepare_kernel<<<(cnt + 255) / 256, 256, 0, ctx->stream>>>(ctx->params, ctx->scan, ctx->shade, first, ctx->n);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

int igs_raster_global(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out, uint32_t* topk) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk <= 4) return launch_raster<4>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 8) return launch_raster<8>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 10) return launch_raster<10>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 16) return launch_raster<16>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 32) return launch_raster<32>(ctx, W, H, row0, row1, kk, out, topk);
    const uint32_t items = (uint32_t)W * (uint32_t)(row1 - row0);
    double* lq = (double*)igs_scratch(ctx, 12, (size_t)items * kk * sizeof(double));
    uint32_t* li = (uint32_t*)igs_scratch(ctx, 13, (size_t)items * kk * sizeof(uint32_t));
    if (!lq || !li) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (generic top-k)");
    topk_generic_kernel<<<(items + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, ctx->n, nullptr, items, W, H, row0,
                                                                      kk, lq, li);
    IGS_LAUNCHED(ctx);
    blend_list_image_kernel<<<(items + 127) / 128, 128, 0, ctx->stream>>>(lq, li, ctx->shade, items, W, row0, kk,
                                                                          out, topk);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

// Final top-K (q ascending, idx) at device points; kk = min(k, n) per point.
int igs_topk_points(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (npts == 0) return IGS_OK;
    if (kk <= 4) return launch_points<4>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 8) return launch_points<8>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 10) return launch_points<10>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 16) return launch_points<16>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 32) return launch_points<32>(ctx, uv, npts, kk, oi, oq);
    topk_generic_kernel<<<(npts + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, ctx->n, uv, npts, 0, 0, 0, kk, oq,
                                                                     oi);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}
