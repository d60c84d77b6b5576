// train.cu -- kernel 4 (backward with sample-ordered reduction), kernel 5
// (fused short-segment sum + Adam + constrain + re-prepare + kNN tree
// accumulation), and the iteration's staging / publication kernels.
//
// Reference: renderer.cpp:91-122 (sample_gradients), :193-252
// (backward_into / ordered reduction), fit.cpp:51-106
// (train_step_gradients), adam.cpp:10-52 (adam_step), gaussian.cpp:74-90
// (constrain).
//
// Gradient reduction.  The reference accumulates grads[idx] += d in sample
// order (renderer.cpp:251, fit.cpp:91-104).  Each sample contributes at most
// once per Gaussian (its top-K indices are distinct), so the per-Gaussian
// sum is the sequence of that Gaussian's contributions in ascending sample
// index.  Deterministic mode (default) reproduces it bit for bit: the
// search epilogue counts contributions per Gaussian, an exclusive scan gives
// each Gaussian a segment, a scatter fills it with slot ids (slot = sample *
// K + entry, so slot order is sample order), and each segment is put in slot
// order and summed sequentially from 0.0 -- the exact operation sequence of
// the reference: short segments inside the fused Adam kernel (one thread per
// Gaussian), long ones by long_segment_kernel (a CTA each).  Fast mode
// accumulates with fp64 atomics instead (order-nondeterministic, ~1e-16
// relative).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "igs_internal.cuh"
#include "knn_tree.cuh"
#include "reduce.cuh"
#include "scan.cuh"
#include "adam.cuh"

using namespace igs_dev;

namespace {

__device__ __forceinline__ double sign_of(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// Per-sample coordinates from flat target indices (fit.cpp:67-70).
__global__ void sample_coords_kernel(const uint32_t* __restrict__ sidx, uint32_t ns, int W, int H,
                                     double* __restrict__ uv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const int f = (int)sidx[i];
    const int h = f / W, w = f % W;
    uv[2 * (size_t)i] = center(w, W);
    uv[2 * (size_t)i + 1] = center(h, H);
}

// One thread per sample: blend its top-K, derive the upstream gradient
// (train: sign(diff)/ns of the L1 loss; backward: given), and emit the K
// SampleContrib records (renderer.cpp:91-122) plus a sort key per record.
// mode 0 = train (target image), 1 = backward (samples5 upstream).
__global__ void sample_finish_kernel(const ScanRec* __restrict__ scan, const ShadeRec* __restrict__ shade,
                                     uint32_t n, const double* __restrict__ lq, const uint32_t* __restrict__ li,
                                     int kk, uint32_t ns, const double* __restrict__ uv, int mode,
                                     const uint32_t* __restrict__ sidx, const float* __restrict__ target, int W,
                                     const double* __restrict__ samples5, double inv_n, double* __restrict__ losses,
                                     double* __restrict__ contrib, uint32_t* __restrict__ keys,
                                     double* __restrict__ grads_atomic, long long* __restrict__ status) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const double x = uv[2 * (size_t)s], y = uv[2 * (size_t)s + 1];
    const double* q = lq + (size_t)s * kk;
    const uint32_t* ix = li + (size_t)s * kk;
    int cnt = 0;
    double total = 0.0, ar = 0.0, ag = 0.0, ab = 0.0;
    for (int j = 0; j < kk; ++j) {
        const uint32_t ci = ix[j];
        if (ci == kNoIdx) break;
        const double w = glibc_math::exp(__dmul_rn(-0.5, q[j]));
        const ShadeRec h = shade[ci];
        total = __dadd_rn(total, w);
        ar = __dadd_rn(ar, __dmul_rn(w, h.r));
        ag = __dadd_rn(ag, __dmul_rn(w, h.g));
        ab = __dadd_rn(ab, __dmul_rn(w, h.b));
        ++cnt;
    }
    const double inv_denom = __ddiv_rn(1.0, __dadd_rn(kNormEps, total));
    const double c0 = __dmul_rn(ar, inv_denom), c1 = __dmul_rn(ag, inv_denom), c2 = __dmul_rn(ab, inv_denom);
    double up0, up1, up2;
    if (mode == 0) {
        const float* t = target + (size_t)sidx[s] * 3;
        const double d0 = __dsub_rn(c0, (double)t[0]);
        const double d1 = __dsub_rn(c1, (double)t[1]);
        const double d2 = __dsub_rn(c2, (double)t[2]);
        const double l = __dadd_rn(__dadd_rn(fabs(d0), fabs(d1)), fabs(d2));
        losses[s] = l;
        if (!isfinite(l)) atomicMin(status + 2, (long long)s);  // fit.cpp:155 non-finite loss
        up0 = __dmul_rn(sign_of(d0), inv_n);
        up1 = __dmul_rn(sign_of(d1), inv_n);
        up2 = __dmul_rn(sign_of(d2), inv_n);
    } else {
        up0 = samples5[(size_t)s * 5 + 2];
        up1 = samples5[(size_t)s * 5 + 3];
        up2 = samples5[(size_t)s * 5 + 4];
    }
    for (int j = 0; j < kk; ++j) {
        const size_t slot = (size_t)s * kk + j;
        if (j >= cnt) {
            if (keys) keys[slot] = n;  // sorts past every real index
            continue;
        }
        const uint32_t ci = ix[j];
        const ScanRec g = scan[ci];
        const ShadeRec h = shade[ci];
        const double w = glibc_math::exp(__dmul_rn(-0.5, q[j]));
        const double dL_dw = __dmul_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(up0, __dsub_rn(h.r, c0)), __dmul_rn(up1, __dsub_rn(h.g, c1))),
                      __dmul_rn(up2, __dsub_rn(h.b, c2))),
            inv_denom);
        const double wc = __dmul_rn(w, inv_denom);
        const double dx = __dsub_rn(x, g.mu_x);
        const double dy = __dsub_rn(y, g.mu_y);
        const double e1 = __dadd_rn(__dmul_rn(g.cos_t, dx), __dmul_rn(g.sin_t, dy));
        const double e2 = __dadd_rn(__dmul_rn(-g.sin_t, dx), __dmul_rn(g.cos_t, dy));
        const double v1 = __dmul_rn(e1, g.inv_a);
        const double v2 = __dmul_rn(e2, g.inv_b);
        const double lw = __dmul_rn(dL_dw, w);
        double d[8];
        d[0] = __dmul_rn(lw, __dsub_rn(__dmul_rn(g.cos_t, v1), __dmul_rn(g.sin_t, v2)));
        d[1] = __dmul_rn(lw, __dadd_rn(__dmul_rn(g.sin_t, v1), __dmul_rn(g.cos_t, v2)));
        d[2] = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(dL_dw, -w), e1), e2), __dsub_rn(g.inv_a, g.inv_b));
        d[3] = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(lw, e1), e1), g.inv_a), h.inv_s1);
        d[4] = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(lw, e2), e2), g.inv_b), h.inv_s2);
        d[5] = __dmul_rn(up0, wc);
        d[6] = __dmul_rn(up1, wc);
        d[7] = __dmul_rn(up2, wc);
        if (grads_atomic) {
#pragma unroll
            for (int p = 0; p < 8; ++p) atomicAdd(grads_atomic + (size_t)ci * 8 + p, d[p]);
        } else {
            double2* o = reinterpret_cast<double2*>(contrib + slot * 8);
            o[0] = make_double2(d[0], d[1]);
            o[1] = make_double2(d[2], d[3]);
            o[2] = make_double2(d[4], d[5]);
            o[3] = make_double2(d[6], d[7]);
            keys[slot] = ci;
        }
    }
}

// --- counting-sort reduction (deterministic, reference summation order) ----
// keys[slot] = Gaussian of contribution slot (slot = sample * kk + entry, so
// slot order is sample order).  gcnt/goff: per-Gaussian count / offset.
// (also queues every Gaussian with a long segment for long_segment_kernel)
__global__ void scatter_slots_kernel(const uint32_t* __restrict__ keys, uint32_t items, uint32_t n,
                                     const uint32_t* __restrict__ goff, const uint32_t* __restrict__ gcnt,
                                     uint32_t* __restrict__ gcur, uint32_t* __restrict__ perm,
                                     uint32_t* __restrict__ long_count, uint32_t* __restrict__ long_list) {
    pdl_wait();
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= items) return;
    const uint32_t g = keys[slot];
    if (g >= n) return;
    const uint32_t pos = atomicAdd(gcur + g, 1u);
    perm[goff[g] + pos] = slot;
    if (pos == 0 && gcnt[g] > kShortSeg) long_list[atomicAdd(long_count, 1u)] = g;
}

// Segment offsets (exclusive scan of the per-Gaussian counts) and the slot
// scatter in one persistent launch: every CTA scans its chunk of the counts,
// a grid barrier publishes the chunk totals, each CTA adds its base and
// writes the offsets, a second barrier, then scatter_slots_kernel's work.
// The grid is sized to be co-resident (a few CTAs per SM), so the spinning
// barrier cannot wait on a CTA that is not running; bar[0] counts arrivals,
// bar[1] exits, and the last CTA out resets both for the next launch.


__global__ void __launch_bounds__(kOffThreads) offsets_scatter_kernel(OffArgs A) {
    pdl_wait();
    if (offsets_scatter_body(A, 0)) grid_exit(A.bar);  // (a barrier was used: reset the counters)
}

__device__ __forceinline__ void sum_row(const double* __restrict__ contrib, uint32_t slot, double* acc) {
    const double2* c = reinterpret_cast<const double2*>(contrib + (size_t)slot * 8);
    const double2 a = c[0], b = c[1], cc = c[2], d = c[3];
    acc[0] = __dadd_rn(acc[0], a.x);
    acc[1] = __dadd_rn(acc[1], a.y);
    acc[2] = __dadd_rn(acc[2], b.x);
    acc[3] = __dadd_rn(acc[3], b.y);
    acc[4] = __dadd_rn(acc[4], cc.x);
    acc[5] = __dadd_rn(acc[5], cc.y);
    acc[6] = __dadd_rn(acc[6], d.x);
    acc[7] = __dadd_rn(acc[7], d.y);
}

__device__ __forceinline__ void sum_sorted(const double* __restrict__ contrib, const uint32_t* slots, uint32_t m,
                                           double* acc) {
    for (uint32_t e = 0; e < m; ++e) sum_row(contrib, slots[e], acc);
}

// Sums segment [o, o + m) of perm (m <= kShortSeg) in ascending slot order.
// m <= 2 -- nearly every Gaussian -- stays in registers.
__device__ __forceinline__ void sum_segment(const double* __restrict__ contrib, const uint32_t* __restrict__ perm,
                                            uint32_t o, uint32_t m, double* acc) {
    if (m == 0) return;
    if (m <= 2) {
        uint32_t a = perm[o], b = m == 2 ? perm[o + 1] : 0u;
        if (m == 2 && b < a) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        sum_row(contrib, a, acc);
        if (m == 2) sum_row(contrib, b, acc);
        return;
    }
    uint32_t sl[kShortSeg];
    for (uint32_t e = 0; e < m; ++e) {
        const uint32_t val = perm[o + e];
        uint32_t pos = e;
        while (pos > 0 && sl[pos - 1] > val) {
            sl[pos] = sl[pos - 1];
            --pos;
        }
        sl[pos] = val;
    }
    sum_sorted(contrib, sl, m, acc);
}

__device__ __forceinline__ void store_grad(double* __restrict__ grads, uint32_t g, const double* acc,
                                           long long* __restrict__ status) {
    double2* o = reinterpret_cast<double2*>(grads + (size_t)g * 8);
    o[0] = make_double2(acc[0], acc[1]);
    o[1] = make_double2(acc[2], acc[3]);
    o[2] = make_double2(acc[4], acc[5]);
    o[3] = make_double2(acc[6], acc[7]);
#pragma unroll
    for (int p = 0; p < 8; ++p)
        if (!isfinite(acc[p])) {  // adam.cpp:29-31: first offending (i, p)
            atomicMin(status, (long long)g * 8 + p);
            break;
        }
}

// Thread per Gaussian: sort its (short) slot list, sum from 0.0 in slot
// (= sample) order -- the reference's operation sequence.  Long segments are
// queued for long_segment_kernel.
__global__ void segment_sum_kernel(const uint32_t* __restrict__ gcnt, const uint32_t* __restrict__ goff,
                                   const uint32_t* __restrict__ perm, const double* __restrict__ contrib, uint32_t n,
                                   double* __restrict__ grads, long long* __restrict__ status) {
    pdl_wait();
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const uint32_t m = gcnt[g];
    if (m > kShortSeg) return;  // long_segment_kernel
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    sum_segment(contrib, perm, goff[g], m, acc);
    store_grad(grads, g, acc, status);
}

// One CTA per long segment, and the loss: reduce.cuh (long_segments,
// loss_chunk); this launch is the path where the search's hard-point launch
// does not take them over.
__global__ void __launch_bounds__(kLongThreads) long_segment_kernel(LongArgs A) {
    __shared__ __align__(16) unsigned char s_raw[kLongSmemBytes];
    pdl_wait();
    if (A.dloss && blockIdx.x >= gridDim.x - kLossCtas) {
        // the last kLossCtas CTAs form the loss while the others take the
        // long segments
        loss_chunk<kLongThreads>(A, blockIdx.x - (gridDim.x - kLossCtas), reinterpret_cast<double*>(s_raw));
        return;
    }
    long_segments<kLongThreads>(A, blockIdx.x, A.dloss ? gridDim.x - kLossCtas : gridDim.x,
                                reinterpret_cast<uint32_t*>(s_raw), reinterpret_cast<uint32_t*>(s_raw) + kLongCap,
                                reinterpret_cast<double(*)[8]>(s_raw + (kLongCap + kLongRank) * 4));
}

// Multi-rank exchange: per-Gaussian counts over every rank's contributions,
// and the non-finite loss check over the gathered losses (first global
// sample index, as a single rank would flag it).
__global__ void count_check_kernel(const uint32_t* __restrict__ keys, uint32_t items, uint32_t n,
                                   uint32_t* __restrict__ gcnt, const double* __restrict__ losses, uint32_t ns,
                                   long long* __restrict__ status) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < items) {
        const uint32_t g = keys[i];
        if (g < n) atomicAdd(gcnt + g, 1u);
    }
    if (losses && i < ns && !isfinite(losses[i])) atomicMin(status + 2, (long long)i);
}

__global__ void count_keys_kernel(const uint32_t* __restrict__ keys, uint32_t items, uint32_t n,
                                  uint32_t* __restrict__ gcnt) {
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= items) return;
    const uint32_t g = keys[slot];
    if (g < n) atomicAdd(gcnt + g, 1u);
}

// Deterministic loss sum (fixed tree order), times 1/ns.  One CTA.
__global__ void loss_reduce_kernel(const double* __restrict__ losses, uint32_t ns, double inv_n,
                                   double* __restrict__ out) {
    __shared__ double sm[1024];
    double acc = 0.0;
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) acc = __dadd_rn(acc, losses[i]);
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sm[threadIdx.x] = __dadd_rn(sm[threadIdx.x], sm[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = __dmul_rn(sm[0], inv_n);
}

// Non-finite gradient scan: status[0] <- first bad slot i*8+p (min).
__global__ void grad_check_kernel(const double* __restrict__ grads, uint32_t n, long long* __restrict__ status) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int p = 0; p < 8; ++p)
        if (!isfinite(grads[(size_t)i * 8 + p])) {
            atomicMin(status, (long long)i * 8 + p);
            return;
        }
}

// Kernel 5: Adam (adam.cpp:21-51) + constrain (gaussian.cpp:74-90) +
// PreparedSet refresh for the next step, for one Gaussian.  HBM: 256 B read
// + 192 B written for params/grads/m/v, plus 96 B of refreshed scan/shade.
__device__ __forceinline__ void adam_load(uint32_t i, const double* __restrict__ params, const double* __restrict__ m,
                                          const double* __restrict__ v, double* gp, double* mm, double* vv) {
    const double2* P = reinterpret_cast<const double2*>(params + (size_t)i * 8);
    const double2* M = reinterpret_cast<const double2*>(m + (size_t)i * 8);
    const double2* V = reinterpret_cast<const double2*>(v + (size_t)i * 8);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const double2 a = P[h], c = M[h], d = V[h];
        gp[2 * h] = a.x; gp[2 * h + 1] = a.y;
        mm[2 * h] = c.x; mm[2 * h + 1] = c.y;
        vv[2 * h] = d.x; vv[2 * h + 1] = d.y;
    }
}

// gp/mm/vv: Gaussian i's parameters and moments (adam_load), updated in place.
__device__ __forceinline__ void adam_one(uint32_t i, const double* gg, double* gp, double* mm, double* vv,
                                         double* __restrict__ params, double* __restrict__ m, double* __restrict__ v,
                                         ScanRec* __restrict__ scan, ShadeRec* __restrict__ shade, double lr_mu,
                                         double lr_color, double lr_scale, double lr_theta, double bc1, double bc2,
                                         double ibc1, double ibc2, long long* __restrict__ status,
                                         const TreeAcc& ta) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;  // adam.hpp:33-35
    const double omb1 = 1.0 - b1, omb2 = 1.0 - b2;  // folded exactly like the reference's constants
    const double lr8[8] = {lr_mu, lr_mu, lr_theta, lr_scale, lr_scale, lr_color, lr_color, lr_color};
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const double g = gg[p];
        mm[p] = __dadd_rn(__dmul_rn(b1, mm[p]), __dmul_rn(omb1, g));
        vv[p] = __dadd_rn(__dmul_rn(b2, vv[p]), __dmul_rn(__dmul_rn(omb2, g), g));
        const double m_hat = div_const(mm[p], bc1, ibc1);
        const double v_hat = div_const(vv[p], bc2, ibc2);
        const double upd = div_rn(__dmul_rn(lr8[p], m_hat), __dadd_rn(__dsqrt_rn(v_hat), eps));
        gp[p] = __dsub_rn(gp[p], upd);
    }
    // constrain (gaussian.cpp:74-90); a non-finite result raises there.
    bool finite_all = true;
#pragma unroll
    for (int p = 0; p < 8; ++p) finite_all = finite_all && isfinite(gp[p]);
    if (!finite_all) {
        atomicMin(status + 1, (long long)i);
        tree_acc_add(ta, i, scan[i]);  // unchanged
        return;
    }
    gp[0] = clamp01d(gp[0]);
    gp[1] = clamp01d(gp[1]);
    double th = fmod(gp[2], kPi);
    if (th < 0.0) th = __dadd_rn(th, kPi);
    if (th >= kPi) th = 0.0;
    gp[2] = th;
    gp[3] = clamp_scale(gp[3]);
    gp[4] = clamp_scale(gp[4]);
    gp[5] = clamp01d(gp[5]);
    gp[6] = clamp01d(gp[6]);
    gp[7] = clamp01d(gp[7]);
    double2* Pw = reinterpret_cast<double2*>(params + (size_t)i * 8);
    double2* Mw = reinterpret_cast<double2*>(m + (size_t)i * 8);
    double2* Vw = reinterpret_cast<double2*>(v + (size_t)i * 8);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        Pw[h] = make_double2(gp[2 * h], gp[2 * h + 1]);
        Mw[h] = make_double2(mm[2 * h], mm[2 * h + 1]);
        Vw[h] = make_double2(vv[2 * h], vv[2 * h + 1]);
    }
    // refresh the prepared records (renderer.cpp:37-50) for the next step
    double s, co;
    glibc_math::sincos(gp[2], &s, &co);
    const double inv_s1 = __ddiv_rn(1.0, gp[3]);
    const double inv_s2 = __ddiv_rn(1.0, gp[4]);
    ScanRec r;
    r.mu_x = gp[0];
    r.mu_y = gp[1];
    r.cos_t = co;
    r.sin_t = s;
    r.inv_a = __dmul_rn(inv_s1, inv_s1);
    r.inv_b = __dmul_rn(inv_s2, inv_s2);
    scan[i] = r;
    tree_acc_add(ta, i, r);
    ShadeRec hh;
    hh.r = gp[5];
    hh.g = gp[6];
    hh.b = gp[7];
    hh.inv_s1 = inv_s1;
    hh.inv_s2 = inv_s2;
    hh.pad = 0.0;
    shade[i] = hh;
}

// Adam over the resident gradients.  Skips all writes when a non-finite
// gradient or loss was flagged (checked by an earlier launch), so a failed
// step leaves the set untouched.
__global__ void adam_kernel(double* __restrict__ params, const double* __restrict__ grads, double* __restrict__ m,
                            double* __restrict__ v, ScanRec* __restrict__ scan, ShadeRec* __restrict__ shade,
                            uint32_t n, double lr_mu, double lr_color, double lr_scale, double lr_theta, double bc1,
                            double bc2, double ibc1, double ibc2, long long* __restrict__ status, TreeAcc ta) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (status[0] != LLONG_MAX || status[2] != LLONG_MAX) {
        tree_acc_add(ta, i, scan[i]);  // (unchanged)
        return;
    }
    double gg[8], gp[8], mm[8], vv[8];
    const double2* G = reinterpret_cast<const double2*>(grads + (size_t)i * 8);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const double2 b = G[h];
        gg[2 * h] = b.x;
        gg[2 * h + 1] = b.y;
    }
    adam_load(i, params, m, v, gp, mm, vv);
    adam_one(i, gg, gp, mm, vv, params, m, v, scan, shade, lr_mu, lr_color, lr_scale, lr_theta, bc1, bc2, ibc1, ibc2,
             status, ta);
}

// Sharded multi-rank update, after the parameter all-gather: the Gaussians
// outside this rank's slice get their prepared records (kernel 1), their
// member-ordered records for the tree refit (as the Adam kernel does for its own) and their
// contribution counters cleared for the next step.
__global__ void complement_prepare_kernel(const double* __restrict__ params, uint32_t n, uint32_t lo, uint32_t hi,
                                          ScanRec* __restrict__ scan, ShadeRec* __restrict__ shade,
                                          uint32_t* __restrict__ gcnt, TreeAcc ta) {
    pdl_wait();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n - (hi - lo)) return;
    const uint32_t g = j < lo ? j : j + (hi - lo);
    const ScanRec r = prepare_one(params, g, scan, shade);
    tree_acc_add(ta, g, r);
    gcnt[g] = 0;
    gcnt[n + g] = 0;
}

// status words [0..2] = the first flagged slot over all ranks (each rank
// flagged only its own slice); [3] (a count) stays per rank
__global__ void status_fold_kernel(const long long* __restrict__ gathered, int nranks, long long* __restrict__ status) {
    pdl_wait();
    const int j = threadIdx.x;
    if (j >= 3) return;
    long long v = gathered[j];
    for (int r = 1; r < nranks; ++r) v = min(v, gathered[4 * r + j]);
    status[j] = v;
}

// Start of an iteration fed from host memory: resets the status block and
// copies the sample indices straight from the pinned (device-mapped) host
// buffer -- a kernel rather than a copy-engine transfer, so the step's
// kernels stay one programmatic-dependent-launch chain.
__global__ void stage_kernel(long long* __restrict__ status, const uint32_t* __restrict__ host_sidx,
                             uint32_t* __restrict__ dsidx, uint32_t ns, L2Prefetch pf) {
    // the host buffer was filled before the launch and the prefetch is a
    // hint: both overlap the previous kernel; the writes wait for it
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    prefetch_l2(pf, i, gridDim.x * blockDim.x);  // the tree refit's inputs
    const uint32_t v = i < ns ? host_sidx[i] : 0u;
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x < 4) status[threadIdx.x] = threadIdx.x == 3 ? 0 : LLONG_MAX;
    if (i < ns) dsidx[i] = v;
}

// Same, drawing the samples on the device from raw engine outputs: sample j
// is AliasTable::sample (sampling.cpp:126-133) with rng.next_index(n) =
// raw[2j] % n and rng.next_double() = (raw[2j+1] >> 11) * 2^-53 -- the
// reference's draw, bit for bit, with the table lookups (random accesses
// into a W*H table) done here instead of on the host.
__global__ void draw_stage_kernel(long long* __restrict__ status, const unsigned long long* __restrict__ host_raw,
                                  const double* __restrict__ prob, const uint32_t* __restrict__ alias,
                                  unsigned long long table_n, uint32_t* __restrict__ dsidx, uint32_t ns,
                                  L2Prefetch pf) {
    // reads (host buffer, the fixed sampling table) before the wait, as stage_kernel
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    prefetch_l2(pf, i, gridDim.x * blockDim.x);
    uint32_t v = 0;
    if (i < ns) {
        const unsigned long long r0 = host_raw[2 * (size_t)i], r1 = host_raw[2 * (size_t)i + 1];
        const unsigned long long j = r0 % table_n;
        const double coin = (double)(r1 >> 11) * 0x1.0p-53;
        v = coin < prob[j] ? (uint32_t)j : alias[j];
    }
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x < 4) status[threadIdx.x] = threadIdx.x == 3 ? 0 : LLONG_MAX;
    if (i < ns) dsidx[i] = v;
}

// End of an iteration: status block + loss into the pinned result block.
__global__ void publish_kernel(const long long* __restrict__ status, const double* __restrict__ dloss,
                               long long* __restrict__ host_res) {
    pdl_wait();
    if (threadIdx.x < 4) host_res[threadIdx.x] = status[threadIdx.x];
    if (threadIdx.x == 4) host_res[4] = __double_as_longlong(*dloss);
}

__global__ void reset_status_kernel(long long* status, L2Prefetch pf) {
    pdl_wait();
    prefetch_l2(pf, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
    if (blockIdx.x) return;
    if (threadIdx.x < 3) status[threadIdx.x] = LLONG_MAX;
    if (threadIdx.x == 3) status[3] = 0;  // a count (kNN tree growth)
}

__global__ void weights_kernel(const double* __restrict__ q, const uint32_t* __restrict__ idx, size_t total,
                               double* __restrict__ w) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    w[i] = idx[i] == kNoIdx ? 0.0 : glibc_math::exp(__dmul_rn(-0.5, q[i]));
}

__global__ void blend_points_kernel(const double* __restrict__ lq, const uint32_t* __restrict__ li,
                                    const ShadeRec* __restrict__ shade, uint32_t npts, int kk,
                                    double* __restrict__ rgb) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    double total = 0.0, ar = 0.0, ag = 0.0, ab = 0.0;
    for (int j = 0; j < kk; ++j) {
        const uint32_t ci = li[(size_t)p * kk + j];
        if (ci == kNoIdx) break;
        const double w = glibc_math::exp(__dmul_rn(-0.5, lq[(size_t)p * kk + j]));
        const ShadeRec s = shade[ci];
        total = __dadd_rn(total, w);
        ar = __dadd_rn(ar, __dmul_rn(w, s.r));
        ag = __dadd_rn(ag, __dmul_rn(w, s.g));
        ab = __dadd_rn(ab, __dmul_rn(w, s.b));
    }
    const double inv = __ddiv_rn(1.0, __dadd_rn(kNormEps, total));
    rgb[(size_t)p * 3 + 0] = __dmul_rn(ar, inv);
    rgb[(size_t)p * 3 + 1] = __dmul_rn(ag, inv);
    rgb[(size_t)p * 3 + 2] = __dmul_rn(ab, inv);
}

}  // namespace

// Scratch slot map (igs_scratch): 0 uv, 1 list q, 2 list idx, 3 contrib,
// 4 keys, 5 keys sorted, 6 vals, 7 vals sorted, 8 cub temp, 9 losses,
// 10/11 point partials, 12/13 generic lists, 14 loss out, 15 upstream samples,
// 21 staged sample indices, 22 per-step losses (device loop), 24 long-segment
// queue, 32 long-segment overflow ranks, 34 offsets launch barrier + chunk
// totals, 35 loss partials + ticket.

int igs_stage_samples(igs_ctx* ctx, const uint32_t* host_pinned, uint32_t* dsidx, uint32_t ns) {
    const L2Prefetch pf = igs_knn_tree_inputs(ctx);
    const unsigned blocks = std::max((ns + 255) / 256 + (ns == 0), (unsigned)ctx->sm_count);
    IGS_PDL(ctx, stage_kernel, blocks, 256, 0, ctx->status, host_pinned, dsidx, ns, pf);
    return IGS_OK;
}

int igs_stage_draws(igs_ctx* ctx, const unsigned long long* host_raw, uint32_t* dsidx, uint32_t ns) {
    const L2Prefetch pf = igs_knn_tree_inputs(ctx);
    const unsigned blocks = std::max((ns + 255) / 256 + (ns == 0), (unsigned)ctx->sm_count);
    IGS_PDL(ctx, draw_stage_kernel, blocks, 256, 0, ctx->status, host_raw, (const double*)ctx->alias_prob.p,
            (const uint32_t*)ctx->alias_idx.p, (unsigned long long)ctx->alias_n, dsidx, ns, pf);
    return IGS_OK;
}

int igs_publish(igs_ctx* ctx, const double* dloss, long long* host_res) {
    IGS_PDL(ctx, publish_kernel, 1, 32, 0, (const long long*)ctx->status, dloss, host_res);
    return IGS_OK;
}

int igs_status_reset(igs_ctx* ctx);

int igs_stage_launch(igs_ctx* ctx, const StageJob& J) {
    if (J.kind == 1) return igs_status_reset(ctx);
    if (J.kind == 2) return igs_stage_samples(ctx, (const uint32_t*)J.host, J.dsidx, J.ns);
    if (J.kind == 3) return igs_stage_draws(ctx, (const unsigned long long*)J.host, J.dsidx, J.ns);
    return IGS_OK;
}

int igs_status_reset(igs_ctx* ctx) {
    const L2Prefetch pf = igs_knn_tree_inputs(ctx);
    IGS_PDL(ctx, reset_status_kernel, pf.nr ? ctx->sm_count : 1, pf.nr ? 256 : 32, 0, ctx->status, pf);
    return IGS_OK;
}

// Shared forward/backward over ns device points.  mode 0: train (sidx +
// target), mode 1: backward (samples5 on device).  Writes ctx->grads and,
// in train mode, the loss into *dev_loss.
// Multi-rank (a communicator attached), deterministic mode: every rank
// computes the contributions of its contiguous share of the samples
// (rank r: global samples [r ns, (r+1) ns)) into its block of the full
// slot arrays, an in-place all-gather completes them, and every rank runs
// the single-GPU reduction and Adam on all NS contributions -- the same
// sample-ordered sums, so the result is bit-identical to one GPU's
// (SURVEY.md 8e's all-gather alternative; fewer bytes than an all-reduce
// of the gradients).
// barrier counters [0, 2) + chunk totals of the persistent offsets launch
// (one CTA per SM), zeroed once
static uint32_t* off_ctl(igs_ctx* ctx) {
    uint32_t* ctl = (uint32_t*)igs_scratch(ctx, 34, ((size_t)kOffCtasPerSm * ctx->sm_count + 2) * sizeof(uint32_t));
    if (ctl && !ctx->off_ctl_ready) {
        if (cudaMemsetAsync(ctl, 0, 2 * sizeof(uint32_t), ctx->stream) != cudaSuccess) return nullptr;
        ctx->off_ctl_ready = true;
    }
    return ctl;
}

int igs_forward_backward(igs_ctx* ctx, uint32_t ns, int k, int mode, const uint32_t* dev_sidx,
                         const double* dev_samples5, double* dev_loss, double inv_n, const double* fuse_lr4,
                         long long t, bool* fused, const StageJob* job) {
    if (fused) *fused = false;
    ctx->fuse_off.ready = false;
    ctx->fuse_off.done = false;
    ctx->fuse_off.fuse_long = false;
    const uint32_t n = ctx->n;
    const int kk = (int)std::min<uint32_t>((uint32_t)k, n);
    const bool knn_path = ctx->opt_cull && kk <= 32;
    bool adam_pf = false;  // the search prefetches the update's rows into L2
    // the iteration's staging: absorbed by the kNN tree launch, else its own
    if (job && job->kind && !knn_path) {
        const int es = igs_stage_launch(ctx, *job);
        if (es) return es;
    }
    const bool exch = igs_has_comm(ctx) && ctx->opt_deterministic && knn_path;
    const uint32_t R = exch ? (uint32_t)ctx->nranks : 1u, rk = exch ? (uint32_t)ctx->rank : 0u;
    ctx->exchanged = exch;
    const size_t items_local = (size_t)ns * kk;
    const size_t items = items_local * R;  // all ranks' contributions
    const uint32_t ns_all = ns * R;
    double* losses = (double*)igs_scratch(ctx, 9, (size_t)std::max<uint32_t>(ns_all, 1) * sizeof(double));
    double* contrib = nullptr;
    uint32_t *keys = nullptr, *gcnt = nullptr, *goff = nullptr, *perm = nullptr, *long_ctl = nullptr;
    // segment buckets, when the search files them (reduce.cuh)
    uint32_t *bucket = nullptr, *ovf = nullptr, *ovf_list = nullptr, *big = nullptr;
    double* loss_part = nullptr;
    bool long_fused = false;  // the long segments + loss ran in the search's hard-point launch
    bool loss_in_adam = false;  // the loss runs in the update's first CTAs instead
    auto long_args = [&]() {
        return LongArgs{(const uint32_t*)gcnt, (const uint32_t*)goff, (const uint32_t*)perm, (const double*)contrib,
                        ctx->grads, (const uint32_t*)(bucket ? ovf + 2 : long_ctl), (const uint32_t*)(long_ctl + 1),
                        ctx->status, big, (const double*)losses, ns_all, inv_n, mode == 0 ? dev_loss : nullptr,
                        loss_part, (unsigned*)(loss_part + kLossCtas), (const uint32_t*)bucket};
    };
    bool gcnt_filled = false;
    if (ctx->opt_deterministic) {
        contrib = (double*)igs_scratch(ctx, 3, items * 8 * sizeof(double));
        keys = (uint32_t*)igs_scratch(ctx, 4, items * sizeof(uint32_t));
        gcnt = (uint32_t*)igs_scratch(ctx, 5, (size_t)n * 2 * sizeof(uint32_t));  // counts | cursors
        goff = (uint32_t*)igs_scratch(ctx, 6, (size_t)n * sizeof(uint32_t));
        perm = (uint32_t*)igs_scratch(ctx, 7, items * sizeof(uint32_t));
        long_ctl = (uint32_t*)igs_scratch(ctx, 24, ((size_t)n + 1) * sizeof(uint32_t));
        big = (uint32_t*)igs_scratch(ctx, 32, items * sizeof(uint32_t));
        // loss partials + the combining ticket (zeroed once; the last CTA re-zeroes it)
        loss_part = (double*)igs_scratch(ctx, 35, kLossCtas * sizeof(double) + 16);
        if (!contrib || !keys || !gcnt || !goff || !perm || !long_ctl || !big || !loss_part)
            return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
        if (!ctx->loss_ticket_ready) {
            IGS_CUDA(ctx, cudaMemsetAsync(loss_part + kLossCtas, 0, 16, ctx->stream));
            ctx->loss_ticket_ready = true;
        }
        // counters | cursors: the fused Adam leaves them zeroed for the next step
        if (ctx->gcnt_clean != gcnt || ctx->gcnt_clean_n != n)
            IGS_CUDA(ctx, cudaMemsetAsync(gcnt, 0, (size_t)n * 2 * sizeof(uint32_t), ctx->stream));
        ctx->gcnt_clean = nullptr;
        // (long_ctl[0]: long-segment count, zeroed by the search kernel on the
        // fused path; long_ctl[1..]: the queue)
        if (!knn_path) IGS_CUDA(ctx, cudaMemsetAsync(long_ctl, 0, sizeof(uint32_t), ctx->stream));
    } else {
        IGS_CUDA(ctx, cudaMemsetAsync(ctx->grads, 0, (size_t)n * 8 * sizeof(double), ctx->stream));
    }
    if (!losses) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (train)");
    int e;
    if (knn_path) {
        // fused: exact top-K search + blend / loss / gradient epilogue per warp
        // the fused Adam's parameter rows and moments, prefetched during the search
        L2Prefetch pf{};
        // only while the rows fit comfortably in L2 (126 MB): at C4 (192 MB of
        // rows) the prefetch only slowed the search, 107.6 -> 80.5 us without
        // it, Adam unchanged (IGS_ADAM_PF_LIMIT_MB overrides the 48 MB limit)
        static const size_t pf_limit =
            (size_t)(getenv("IGS_ADAM_PF_LIMIT_MB") ? atol(getenv("IGS_ADAM_PF_LIMIT_MB")) : 48) << 20;
        adam_pf = fuse_lr4 && (size_t)n * 192 <= pf_limit;
        if (adam_pf) {
            l2pf_add(pf, ctx->params, (size_t)n * 64);
            l2pf_add(pf, ctx->adam_m, (size_t)n * 64);
            l2pf_add(pf, ctx->adam_v, (size_t)n * 64);
        }
        ctx->stage_job = job ? *job : StageJob{};  // knn_build runs it (or launches it) first
        // single rank, deterministic: the search's hard-point launch may run
        // the reduction's offsets + scatter too (hard_offsets_kernel)
        ctx->fuse_off.ready = false;
        ctx->fuse_off.done = false;
        if (ctx->opt_deterministic && !exch && !getenv("IGS_SCAN_LAUNCHES")) {
            uint32_t* ctl = off_ctl(ctx);
            if (!ctl) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (scan)");
            ctx->fuse_off.args = OffArgs{(const uint32_t*)gcnt, n, goff, ctl + 2, (const uint32_t*)keys, (uint32_t)items,
                                         gcnt + n, perm, long_ctl, long_ctl + 1, (unsigned*)ctl, nullptr, nullptr};
            ctx->fuse_off.ready = true;
            if (fuse_lr4 && !igs_has_comm(ctx) && !getenv("IGS_NO_BUCKET")) {
                // segment buckets (reduce.cuh): read by the fused Adam, so only
                // when it follows; two sets of counters used alternately (the
                // search zeroes the other set)
                bucket = (uint32_t*)igs_scratch(ctx, 46, ((size_t)n * kBucket + 2 * items) * sizeof(uint32_t));
                uint32_t* ctr = (uint32_t*)igs_scratch(ctx, 47, 8 * sizeof(uint32_t));
                if (!bucket || !ctr) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (buckets)");
                if (!ctx->ovf_ready) {
                    IGS_CUDA(ctx, cudaMemsetAsync(ctr, 0, 8 * sizeof(uint32_t), ctx->stream));
                    ctx->ovf_ready = true;
                }
                ctx->ovf_phase ^= 1;
                ovf = ctr + 4 * ctx->ovf_phase;
                ovf_list = bucket + (size_t)n * kBucket;
                ctx->fuse_off.bucket = bucket;
                ctx->fuse_off.ovf = ovf;
                ctx->fuse_off.ovf_list = ovf_list;
                ctx->fuse_off.long_list = long_ctl + 1;
                ctx->fuse_off.ovf_zero = ctr + 4 * (ctx->ovf_phase ^ 1);
                ctx->fuse_off.args.ovf = ovf;
                ctx->fuse_off.args.ovf_list = ovf_list;
                ctx->fuse_off.args.long_count = ovf + 2;
                ctx->fuse_off.long_args = long_args();
                ctx->fuse_off.fuse_long = getenv("IGS_LONG_LAUNCH") == nullptr;  // (A/B: the separate launch)
                if (ctx->fuse_off.fuse_long && getenv("IGS_LOSS_OFF") == nullptr) {
                    // the loss moves on into the update's first CTAs (LossTail)
                    ctx->fuse_off.long_args.dloss = nullptr;
                    loss_in_adam = mode == 0 && dev_loss;
                }
            }
        }
        e = igs_knn_forward_backward(ctx, mode, dev_sidx, dev_samples5, ns, kk, inv_n, losses + (size_t)rk * ns,
                                     contrib ? contrib + rk * items_local * 8 : nullptr,
                                     keys ? keys + rk * items_local : nullptr, exch ? nullptr : gcnt,
                                     ctx->opt_deterministic ? nullptr : ctx->grads, long_ctl, &pf, exch ? 1 : 0);
        ctx->stage_job = StageJob{};
        ctx->fuse_off.ready = false;
        ctx->fuse_off.bucket = nullptr;
        long_fused = ctx->fuse_off.done && ctx->fuse_off.fuse_long;
        ctx->fuse_off.fuse_long = false;
        if (e) return e;
        gcnt_filled = !exch;
    } else {
        double* uv = (double*)igs_scratch(ctx, 0, (size_t)ns * 2 * sizeof(double));
        double* lq = (double*)igs_scratch(ctx, 1, (size_t)ns * kk * sizeof(double));
        uint32_t* li = (uint32_t*)igs_scratch(ctx, 2, (size_t)ns * kk * sizeof(uint32_t));
        if (!uv || !lq || !li) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (train)");
        const int tb = 256;
        if (mode == 0) {
            sample_coords_kernel<<<(ns + tb - 1) / tb, tb, 0, ctx->stream>>>(dev_sidx, ns, ctx->tgt_w, ctx->tgt_h,
                                                                             uv);
            IGS_LAUNCHED(ctx);
        } else {
            IGS_CUDA(ctx, cudaMemcpy2DAsync(uv, 2 * sizeof(double), dev_samples5, 5 * sizeof(double),
                                            2 * sizeof(double), ns, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if ((e = igs_topk_points(ctx, uv, ns, k, li, lq))) return e;
        igs_prof_begin(ctx, IGS_PROF_FINISH);
        sample_finish_kernel<<<(ns + 127) / 128, 128, 0, ctx->stream>>>(
            ctx->scan, ctx->shade, n, lq, li, kk, ns, uv, mode, dev_sidx, (const float*)ctx->target.p, ctx->tgt_w,
            dev_samples5, inv_n, losses, contrib, keys, ctx->opt_deterministic ? nullptr : ctx->grads, ctx->status);
        IGS_LAUNCHED(ctx);
        igs_prof_end(ctx, IGS_PROF_FINISH, (double)items);
    }
    if (exch) {
        // every rank's contributions (and losses) in global slot order
        if ((e = igs_comm_allgather(ctx, keys, items_local * sizeof(uint32_t)))) return e;
        if ((e = igs_comm_allgather(ctx, contrib, items_local * 8 * sizeof(double)))) return e;
        if (mode == 0 && (e = igs_comm_allgather(ctx, losses, (size_t)ns * sizeof(double)))) return e;
        IGS_PDL(ctx, count_check_kernel, (unsigned)((std::max<size_t>(items, ns_all) + 255) / 256), 256, 0,
                (const uint32_t*)keys, (uint32_t)items, n, gcnt, mode == 0 ? (const double*)losses : nullptr, ns_all,
                ctx->status);
        gcnt_filled = true;
    }
    // the loss sum needs only the per-sample losses: it runs on the side
    // stream, overlapping the reduction and Adam, and is joined below
    // the loss sum rides in long_segment_kernel (deterministic mode), else on
    // the side stream
    const bool loss_side = mode == 0 && dev_loss && !ctx->opt_deterministic;
    if (loss_side) {
        IGS_CUDA(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
        IGS_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        loss_reduce_kernel<<<1, 1024, 0, ctx->side>>>(losses, ns_all, inv_n, dev_loss);
        IGS_LAUNCHED(ctx);
        IGS_CUDA(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
    }
    if (ctx->opt_deterministic) {
        igs_prof_begin(ctx, IGS_PROF_REDUCE);
        if (!gcnt_filled) {
            // fallback path: per-Gaussian counts from the keys
            count_keys_kernel<<<(unsigned)((items + 255) / 256), 256, 0, ctx->stream>>>(keys, (uint32_t)items, n,
                                                                                        gcnt);
            IGS_LAUNCHED(ctx);
        }
        if (ctx->fuse_off.done) {
            // done by the search's hard_offsets_kernel
        } else if (!getenv("IGS_SCAN_LAUNCHES")) {
            // offsets + scatter in one persistent launch (two grid barriers)
            uint32_t* ctl = off_ctl(ctx);
            if (!ctl) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (scan)");
            OffArgs A{(const uint32_t*)gcnt, n, goff, ctl + 2, (const uint32_t*)keys, (uint32_t)items, gcnt + n, perm,
                      bucket ? ovf + 2 : long_ctl, long_ctl + 1, (unsigned*)ctl, ovf, ovf_list};
            IGS_PDL_COOP(ctx, offsets_scatter_kernel, (unsigned)ctx->sm_count, kOffThreads, 0, A);
        } else {
            if ((e = igs_scan_excl_u32(ctx, gcnt, goff, (size_t)n))) return e;
            IGS_PDL(ctx, scatter_slots_kernel, (unsigned)((items + 255) / 256), 256, 0, (const uint32_t*)keys,
                    (uint32_t)items, n, (const uint32_t*)goff, (const uint32_t*)gcnt, gcnt + n, perm, long_ctl,
                    long_ctl + 1);
        }
        if (!long_fused) IGS_PDL(ctx, long_segment_kernel, 8 * ctx->sm_count, kLongThreads, 0, long_args());
        if (fuse_lr4 && (exch || !igs_has_comm(ctx))) {
            // short segments summed inside the Adam kernel (one pass over the set)
            const double bc1 = 1.0 - std::pow(0.9, (double)t);  // adam.cpp:16-17, host libm
            const double bc2 = 1.0 - std::pow(0.999, (double)t);
            const TreeAcc ta = igs_knn_tree_acc(ctx);
            ctx->params_version++;
            igs_prof_end(ctx, IGS_PROF_REDUCE, (double)items);
            igs_prof_begin(ctx, IGS_PROF_ADAM);
            // multi-rank: this rank's slice [lo, hi) of ceil(n/R)-record blocks
            const uint32_t B = (n + R - 1) / R;
            const bool shard = exch && R > 1 && ctx->opt_shard_adam && (size_t)B * R <= ctx->cap;
            const uint32_t lo = shard ? std::min(n, rk * B) : 0u, hi = shard ? std::min(n, lo + B) : n;
            // rows the search did not prefetch (above its L2 limit): one
            // resident wave walks the blocks, prefetching each next block's
            // rows (IGS_ADAM_LOOP_GRID: 0 never, g > 0 that grid always)
            const uint32_t nblk = (hi - lo + kAdamThreads / 2 - 1) / (kAdamThreads / 2);
            static int loop_per_sm = 0;
            if (!loop_per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                    &loop_per_sm, segment_adam_kernel<LossTail>, kAdamThreads, 0) != cudaSuccess)
                loop_per_sm = 1;
            const char* lg = getenv("IGS_ADAM_LOOP_GRID");
            uint32_t stride = lg ? (uint32_t)atol(lg)
                                 : adam_pf ? 0u : (uint32_t)std::max(loop_per_sm, 1) * (uint32_t)ctx->sm_count;
            AdamArgs aa{gcnt, (const uint32_t*)goff, perm, bucket,
                        (const double*)contrib, n, ctx->grads, ctx->params, ctx->adam_m, ctx->adam_v,
                        ctx->scan, ctx->shade, fuse_lr4[0], fuse_lr4[1], fuse_lr4[2], fuse_lr4[3], bc1, bc2,
                        1.0 / bc1, 1.0 / bc2, ctx->status, ta, lo, hi, nblk, 0};
            const LossTail tail{{}, loss_in_adam ? long_args() : LongArgs{}};
            if (stride) stride = std::max<uint32_t>(stride, kLossCtas);  // LossTail: CTAs 0..kLossCtas-1
            if (stride >= nblk) stride = 0;
            aa.loop_stride = stride;
            if (hi > lo) IGS_PDL(ctx, segment_adam_kernel<LossTail>, stride ? stride : nblk, kAdamThreads, 0, aa, tail);
            if (shard) {
                // flags of every slice, then every slice's parameters, then
                // the records (and member-ordered copies) of the other slices here
                long long* st = (long long*)igs_scratch(ctx, 40, (size_t)R * 4 * sizeof(long long));
                if (!st) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (shard)");
                IGS_CUDA(ctx, cudaMemcpyAsync(st + 4 * rk, ctx->status, 4 * sizeof(long long),
                                              cudaMemcpyDeviceToDevice, ctx->stream));
                if ((e = igs_comm_allgather(ctx, st, 4 * sizeof(long long)))) return e;
                IGS_PDL(ctx, status_fold_kernel, 1, 32, 0, (const long long*)st, (int)R, ctx->status);
                if ((e = igs_comm_allgather(ctx, ctx->params, (size_t)B * 8 * sizeof(double)))) return e;
                if (n > hi - lo)
                    IGS_PDL(ctx, complement_prepare_kernel, (n - (hi - lo) + 255) / 256, 256, 0,
                            (const double*)ctx->params, n, lo, hi, ctx->scan, ctx->shade, gcnt, ta);
                ctx->moments_local = true;
            }
            igs_prof_end(ctx, IGS_PROF_ADAM, (double)(hi - lo) * 596.0);
            ctx->gcnt_clean = gcnt;
            ctx->gcnt_clean_n = n;
            if (fused) *fused = true;
        } else {
            IGS_PDL(ctx, segment_sum_kernel, (n + 255) / 256, 256, 0, (const uint32_t*)gcnt, (const uint32_t*)goff,
                    (const uint32_t*)perm, (const double*)contrib, n, ctx->grads, ctx->status);
            igs_prof_end(ctx, IGS_PROF_REDUCE, (double)items);
        }
        ctx->grads_checked = true;
    } else {
        ctx->grads_checked = false;
    }
    if (loss_side) IGS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
    ctx->grads_valid = true;
    return IGS_OK;
}

int igs_grad_check(igs_ctx* ctx) {
    IGS_PDL(ctx, grad_check_kernel, (ctx->n + 255) / 256, 256, 0, (const double*)ctx->grads, ctx->n, ctx->status);
    return IGS_OK;
}

int igs_adam_launch(igs_ctx* ctx, const double* lr4, long long t) {
    // Bias corrections with the host libm pow, as adam.cpp:16-17.
    const double bc1 = 1.0 - std::pow(0.9, (double)t);
    const double bc2 = 1.0 - std::pow(0.999, (double)t);
    const TreeAcc ta = igs_knn_tree_acc(ctx);
    ctx->params_version++;
    igs_prof_begin(ctx, IGS_PROF_ADAM);
    IGS_PDL(ctx, adam_kernel, (ctx->n + 255) / 256, 256, 0, ctx->params, (const double*)ctx->grads, ctx->adam_m,
            ctx->adam_v, ctx->scan, ctx->shade, ctx->n, lr4[0], lr4[1], lr4[2], lr4[3], bc1, bc2, 1.0 / bc1,
            1.0 / bc2, ctx->status, ta);
    // algorithmic bytes: read params/grads/m/v (256 B), write params/m/v
    // (192 B) and the refreshed 96 B of scan+shade records
    igs_prof_end(ctx, IGS_PROF_ADAM, (double)ctx->n * 544.0);
    return IGS_OK;
}

int igs_weights(igs_ctx* ctx, const double* q, const uint32_t* idx, size_t total, double* w) {
    weights_kernel<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(q, idx, total, w);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

int igs_blend_points(igs_ctx* ctx, const double* lq, const uint32_t* li, uint32_t npts, int kk, double* rgb) {
    blend_points_kernel<<<(npts + 127) / 128, 128, 0, ctx->stream>>>(lq, li, ctx->shade, npts, kk, rgb);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}
