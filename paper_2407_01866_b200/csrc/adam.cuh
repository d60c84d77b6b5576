// adam.cuh -- kernel 5, the fused update: a Gaussian's sample-ordered
// gradient sum (its segment of contributions), Adam (adam.cpp:21-51),
// constrain (gaussian.cpp:74-90) and the prepared records for the next step
// (renderer.cpp:37-50), one lane pair per Gaussian.  The kernel takes a
// Tail: extra worker CTAs in the same launch (Tail::kWorkers).  A tail that
// ran the hard-point scan, the loss and the long segments in workers (so no
// launch sat between the search and the update) measured slower -- C2
// 92.4 vs 90.0 us per step at the fit start, 124-133 vs 128 us at t = 5,000
// -- so train.cu launches it with NoTail.
#pragma once

#include <climits>

#include "igs_internal.cuh"
#include "knn_tree.cuh"
#include "reduce.cuh"

namespace igs_dev {

// a / b correctly rounded; a zero dividend (every parameter of a Gaussian no
// sample selected) skips __ddiv_rn's slow path: 0 / b == 0 * b for finite
// nonzero b, sign included.
__device__ __forceinline__ double div_rn(double a, double b) {
    return (a == 0.0 && b != 0.0 && fabs(b) < __longlong_as_double(0x7ff0000000000000LL)) ? __dmul_rn(a, b)
                                                                                         : __ddiv_rn(a, b);
}

// a / b for the per-step constants b = bc1, bc2 with y = RN(1/b) from the
// host: two Markstein corrections (igs_math::div_by_recip), exact IEEE
// division outside its operand range (zero, tiny, huge, non-finite).
__device__ __forceinline__ double div_const(double a, double b, double y) {
    const double aa = fabs(a);
    if (aa >= 0x1p-960 && aa <= 0x1p1000) return igs_math::div_by_recip(a, b, y);
    return div_rn(a, b);
}

__device__ __forceinline__ double clamp01d(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
__device__ __forceinline__ double clamp_scale(double v) {
    return v < kScaleMin ? kScaleMin : (v > kScaleMax ? kScaleMax : v);
}

__device__ __forceinline__ double shx(double v) { return __shfl_xor_sync(0xffffffffu, v, 1); }

// Everything the fused update reads and writes.
struct AdamArgs {
    uint32_t* gcnt;          // per-Gaussian contribution counts | [n, 2n) cursors; left zeroed
    const uint32_t* goff;    // CSR mode: segment offsets
    uint32_t* perm;          // CSR mode: slot ids by segment (short ones put in order in place)
    uint32_t* bucket;        // bucket mode (reduce.cuh): slot ids by Gaussian, or null (ditto)
    const double* contrib;
    uint32_t n;
    double* grads;
    double* params;
    double* m;
    double* v;
    ScanRec* scan;
    ShadeRec* shade;
    double lr_mu, lr_color, lr_scale, lr_theta, bc1, bc2, ibc1, ibc2;
    long long* status;
    TreeAcc ta;
    uint32_t g_begin, g_end;  // the Gaussians of this launch (a rank's slice when sharded)
    uint32_t nblk;            // blocks of kAdamThreads / 2 Gaussians in [g_begin, g_end)
    uint32_t loop_stride;     // 0: one block per CTA; else the grid, walking the blocks
};

// The update of Gaussian g from its gradient, by lane h of its pair (h = 0:
// parameters 0-3 = mu, theta, s1; h = 1: 4-7 = s2, colour); G = this lane's
// four gradient components.  Unless the gradient is non-finite (status[0] =
// first (i, p), g left untouched -- every finite Gaussian is still updated,
// deterministically; the reference has updated 0..i-1 when it throws,
// adam.cpp:29-31) or the step is skipped (a non-finite loss, fit.cpp:155).
// The lane pair splits the chains: lane 1 forms sin/cos while lane 0 forms
// both reciprocals.  Whole warps call it (pair shuffles); !live lanes write
// nothing.
__device__ __forceinline__ void adam_pair_update(const AdamArgs& A, uint32_t g, int h, bool live, bool skip_all,
                                                 const double* G) {
    // first non-finite gradient component of the pair (h = 0's first)
    int badp = 8;
    for (int j = 3; j >= 0; --j)
        if (!isfinite(G[j])) badp = 4 * h + j;
    const int other = __shfl_xor_sync(0xffffffffu, badp, 1);
    const int firstbad = min(badp, other);
    if (skip_all || firstbad < 8) {
        if (live && h == 0) {
            if (!skip_all) atomicMin(A.status, (long long)g * 8 + firstbad);
            tree_acc_add(A.ta, g, A.scan[g]);
        }
        return;  // pair-uniform
    }
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double omb1 = 1.0 - b1, omb2 = 1.0 - b2;
    const double2* P2 = reinterpret_cast<const double2*>(A.params + (size_t)g * 8 + 4 * h);
    const double2* M2 = reinterpret_cast<const double2*>(A.m + (size_t)g * 8 + 4 * h);
    const double2* V2 = reinterpret_cast<const double2*>(A.v + (size_t)g * 8 + 4 * h);
    double gp[4], mm[4], vv[4];
    {
        const double2 p0 = P2[0], p1 = P2[1], m0 = M2[0], m1 = M2[1], v0 = V2[0], v1 = V2[1];
        gp[0] = p0.x; gp[1] = p0.y; gp[2] = p1.x; gp[3] = p1.y;
        mm[0] = m0.x; mm[1] = m0.y; mm[2] = m1.x; mm[3] = m1.y;
        vv[0] = v0.x; vv[1] = v0.y; vv[2] = v1.x; vv[3] = v1.y;
    }
    const double lrh[4] = {h ? A.lr_scale : A.lr_mu, h ? A.lr_color : A.lr_mu, h ? A.lr_color : A.lr_theta,
                           h ? A.lr_color : A.lr_scale};
    bool fin = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        mm[j] = __dadd_rn(__dmul_rn(b1, mm[j]), __dmul_rn(omb1, G[j]));
        vv[j] = __dadd_rn(__dmul_rn(b2, vv[j]), __dmul_rn(__dmul_rn(omb2, G[j]), G[j]));
        const double m_hat = div_const(mm[j], A.bc1, A.ibc1);
        const double v_hat = div_const(vv[j], A.bc2, A.ibc2);
        const double upd = div_rn(__dmul_rn(lrh[j], m_hat), __dadd_rn(__dsqrt_rn(v_hat), eps));
        gp[j] = __dsub_rn(gp[j], upd);
        fin = fin && isfinite(gp[j]);
    }
    const bool fin_pair = __shfl_xor_sync(0xffffffffu, fin ? 1 : 0, 1) && fin;
    if (!fin_pair) {
        if (live && h == 0) {
            atomicMin(A.status + 1, (long long)g);
            tree_acc_add(A.ta, g, A.scan[g]);
        }
        return;
    }
    // constrain (gaussian.cpp:74-90)
    if (h == 0) {
        gp[0] = clamp01d(gp[0]);
        gp[1] = clamp01d(gp[1]);
        double th = fmod(gp[2], kPi);
        if (th < 0.0) th = __dadd_rn(th, kPi);
        if (th >= kPi) th = 0.0;
        gp[2] = th;
        gp[3] = clamp_scale(gp[3]);
    } else {
        gp[0] = clamp_scale(gp[0]);
        gp[1] = clamp01d(gp[1]);
        gp[2] = clamp01d(gp[2]);
        gp[3] = clamp01d(gp[3]);
    }
    if (live) {
        double2* Pw = reinterpret_cast<double2*>(A.params + (size_t)g * 8 + 4 * h);
        double2* Mw = reinterpret_cast<double2*>(A.m + (size_t)g * 8 + 4 * h);
        double2* Vw = reinterpret_cast<double2*>(A.v + (size_t)g * 8 + 4 * h);
        Pw[0] = make_double2(gp[0], gp[1]);
        Pw[1] = make_double2(gp[2], gp[3]);
        Mw[0] = make_double2(mm[0], mm[1]);
        Mw[1] = make_double2(mm[2], mm[3]);
        Vw[0] = make_double2(vv[0], vv[1]);
        Vw[1] = make_double2(vv[2], vv[3]);
    }
    // prepared records: h = 1 gets theta and forms sin/cos; h = 0 gets s2
    // and forms both reciprocals
    const double theta = shx(gp[2]);  // on h = 1: lane 0's theta
    const double s2 = shx(gp[0]);     // on h = 0: lane 1's s2
    double a = 0.0, b = 0.0;          // h = 0: inv_s1, inv_s2; h = 1: sin, cos
    if (h == 0) {
        a = __ddiv_rn(1.0, gp[3]);
        b = __ddiv_rn(1.0, s2);
    } else {
        glibc_math::sincos(theta, &a, &b);
    }
    const double oa = shx(a), ob = shx(b);
    if (!live) return;
    if (h == 0) {
        ScanRec r;
        r.mu_x = gp[0];
        r.mu_y = gp[1];
        r.cos_t = ob;
        r.sin_t = oa;
        r.inv_a = __dmul_rn(a, a);
        r.inv_b = __dmul_rn(b, b);
        A.scan[g] = r;
        tree_acc_add(A.ta, g, r);
    } else {
        ShadeRec hh;
        hh.r = gp[1];
        hh.g = gp[2];
        hh.b = gp[3];
        hh.inv_s1 = oa;
        hh.inv_s2 = ob;
        hh.pad = 0.0;
        A.shade[g] = hh;
    }
}

// No tail: CTA b updates Gaussians [g_begin + 64 b, + 64); long segments
// were summed before the launch (their gradient is read from grads).
struct NoTail {
    static constexpr bool kWorkers = false;
    static constexpr size_t kSmemBytes = 0;
    __device__ void pre(unsigned char*) const {}
    __device__ void run(uint32_t, uint32_t, const AdamArgs&, unsigned char*) const {}
    __device__ bool hold() const { return false; }
    __device__ void wait() const {}
};

#ifndef IGS_ADAM_THREADS
#define IGS_ADAM_THREADS 128
#endif
constexpr int kAdamThreads = IGS_ADAM_THREADS;  // kAdamThreads / 2 Gaussians per CTA

// The loss chunks (reduce.cuh loss_chunk) by the first kLossCtas CTAs before
// their Gaussians: the launch before the update then has nothing to do in
// the common case (no hard points, no long segments).
struct LossTail : NoTail {
    static constexpr size_t kSmemBytes = kAdamThreads * sizeof(double);
    LongArgs L;
    __device__ void pre(unsigned char* smem) const {
        if (L.dloss && blockIdx.x < kLossCtas) {
            loss_chunk<kAdamThreads>(L, blockIdx.x, reinterpret_cast<double*>(smem));
            __syncthreads();  // (the shared memory is the sort's next)
        }
    }
};

}  // namespace igs_dev

namespace {  // the kernel: one copy per translation unit that launches it
using namespace igs_dev;

// Fused short-segment reduction + Adam.  With Tail::kWorkers the first
// T.nworkers CTAs to start (by ticket, so they are running before any
// update CTA can wait on them) run T.run; the update CTAs take the
// Gaussians by ticket order, leave long segments (> kShortSeg) to the
// workers and, when T.hold(), wait for the workers' hard points first.
// One block of kAdamThreads / 2 Gaussians: the short-segment sums and the
// update (the kernel body below, once or per pass of its loop).
template <class Tail>
__device__ __forceinline__ void adam_block(const AdamArgs& A, uint32_t blk) {
    // Gaussians [g_begin, g_end): the whole set, or this rank's slice when
    // the multi-rank update is sharded (n stays the set size: gcnt is [2n])
    const uint32_t g0 = A.g_begin + blk * (kAdamThreads / 2) + (threadIdx.x >> 1);
    const int h = threadIdx.x & 1;
    const uint32_t g = g0 < A.g_end ? g0 : A.g_end - 1;  // dead pairs shadow a live one (no writes): full shuffles
    // a short segment's slot ids: its bucket (reduce.cuh), else perm[goff[g] ...]
    const bool from_bucket = A.bucket != nullptr;
    uint32_t* __restrict__ seg = from_bucket ? A.bucket : A.perm;
    uint32_t cntg = 0;
    size_t og = 0;
    if (h == 0) {
        cntg = A.gcnt[g];
        og = from_bucket ? (size_t)g * kBucket : A.goff[g];
    }
    cntg = __shfl_sync(0xffffffffu, cntg, threadIdx.x & ~1);
    og = __shfl_sync(0xffffffffu, og, threadIdx.x & ~1);
    // with workers a long segment's Gaussian is theirs (this pair shadows)
    const bool live = g0 < A.g_end && !(Tail::kWorkers && cntg > kShortSeg);
    __syncwarp();
    if (live && h == 0) {
        A.gcnt[g] = 0;
        A.gcnt[A.n + g] = 0;
    }
    const bool skip_all = A.status[2] != LLONG_MAX;
    // segments of 5..kShortSeg slot ids: put in slot order in place by the
    // whole warp, one segment at a time -- lane e loads ids e, e + 32, ...
    // (one row of the bucket), takes each one's rank among the others by
    // shuffles (ids are distinct) and writes it back at its rank; the pair
    // then reads its segment in order.  Only live pairs sort (a dead pair
    // shadowing a Gaussian of another warp would sort the same ids
    // concurrently); a dead pair's sum reads whatever is there and is
    // never written.
    {
        constexpr int kPer = (kShortSeg + 31) / 32;
        const int lane = threadIdx.x & 31;
        unsigned med = __ballot_sync(0xffffffffu, live && !skip_all && h == 0 && cntg > 4 && cntg <= kShortSeg);
        while (med) {
            const int src = __ffs(med) - 1;
            med &= med - 1;
            const uint32_t mm = __shfl_sync(0xffffffffu, cntg, src);
            const size_t oo = __shfl_sync(0xffffffffu, og, src);
            uint32_t v[kPer], r[kPer];
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint32_t e = (uint32_t)(lane + 32 * j);
                v[j] = e < mm ? seg[oo + e] : 0xFFFFFFFFu;
                r[j] = 0;
            }
#pragma unroll
            for (int jj = 0; jj < kPer; ++jj) {
                if (32u * jj >= mm) break;  // (uniform)
                const uint32_t lim = min(32u, mm - 32u * jj);
                for (uint32_t sl = 0; sl < lim; ++sl) {
                    const uint32_t u = __shfl_sync(0xffffffffu, v[jj], sl);
#pragma unroll
                    for (int j = 0; j < kPer; ++j) r[j] += u < v[j];
                }
            }
            __syncwarp();  // every id read before any is overwritten
#pragma unroll
            for (int j = 0; j < kPer; ++j)
                if ((uint32_t)(lane + 32 * j) < mm) seg[oo + r[j]] = v[j];
        }
        __syncwarp();
    }
    // gradient components 4h .. 4h+3
    double G[4] = {0, 0, 0, 0};
    if (!skip_all) {
        if (cntg > kShortSeg) {
            if (!Tail::kWorkers) {  // summed by long_segment_kernel (with workers: not this pair's)
                const double2* src = reinterpret_cast<const double2*>(A.grads + (size_t)g * 8 + 4 * h);
                const double2 a = src[0], b = src[1];
                G[0] = a.x; G[1] = a.y; G[2] = b.x; G[3] = b.y;
            }
        } else if (cntg > 0) {
            auto add_row = [&](uint32_t slot) {
                const double2* c = reinterpret_cast<const double2*>(A.contrib + (size_t)slot * 8 + 4 * h);
                const double2 a = c[0], b = c[1];
                G[0] = __dadd_rn(G[0], a.x);
                G[1] = __dadd_rn(G[1], a.y);
                G[2] = __dadd_rn(G[2], b.x);
                G[3] = __dadd_rn(G[3], b.y);
            };
            if (cntg <= 4) {
                // nearly every segment: its slot ids sorted in registers
                // (a 5-exchange network), no local-memory array
                uint32_t s0 = seg[og], s1 = cntg > 1 ? seg[og + 1] : 0xFFFFFFFFu,
                         s2 = cntg > 2 ? seg[og + 2] : 0xFFFFFFFFu, s3 = cntg > 3 ? seg[og + 3] : 0xFFFFFFFFu;
                auto cx = [](uint32_t& a, uint32_t& b) {
                    const uint32_t lo = min(a, b), hi = max(a, b);
                    a = lo;
                    b = hi;
                };
                cx(s0, s1);
                cx(s2, s3);
                cx(s0, s2);
                cx(s1, s3);
                cx(s1, s2);
                add_row(s0);
                if (cntg > 1) add_row(s1);
                if (cntg > 2) add_row(s2);
                if (cntg > 3) add_row(s3);
            } else {
                for (uint32_t e = 0; e < cntg; ++e) add_row(seg[og + e]);  // (sorted in place above)
            }
            if (live) {
                double2* o2 = reinterpret_cast<double2*>(A.grads + (size_t)g * 8 + 4 * h);
                o2[0] = make_double2(G[0], G[1]);
                o2[1] = make_double2(G[2], G[3]);
            }
        } else if (live) {
            double2* o2 = reinterpret_cast<double2*>(A.grads + (size_t)g * 8 + 4 * h);
            o2[0] = make_double2(0.0, 0.0);
            o2[1] = make_double2(0.0, 0.0);
        }
    }
    adam_pair_update(A, g, h, live, skip_all, G);
}

#ifndef IGS_ADAM_MINB
#define IGS_ADAM_MINB 7
#endif
template <class Tail>
__global__ void __launch_bounds__(kAdamThreads, IGS_ADAM_MINB) segment_adam_kernel(AdamArgs A, Tail T) {
    __shared__ __align__(16) unsigned char s_raw[Tail::kSmemBytes > 16 ? Tail::kSmemBytes : 16];
    pdl_wait();
    T.pre(s_raw);
    uint32_t blk = blockIdx.x;
    if constexpr (Tail::kWorkers) {
        __shared__ uint32_t s_role;
        if (threadIdx.x == 0) s_role = atomicAdd(T.ticket, 1u) - T.tick_base;
        __syncthreads();
        const uint32_t role = s_role;
        if (role < T.nworkers) {
            T.run(role, T.nworkers, A, s_raw);
            return;
        }
        blk = role - T.nworkers;
        if (T.hold()) T.wait();
    }
    // large sets (loop_stride = the grid): a resident wave walks the
    // blocks; each pass first prefetches its next block's parameter and
    // moment rows into L2, so their DRAM latency hides behind this block's
    // chain and fp64 work (C4: 178 -> 164 us).  Otherwise one pass.
    const uint32_t stride = A.loop_stride ? A.loop_stride : A.nblk;
    for (; blk < A.nblk; blk += stride) {
        const uint32_t nb = blk + stride;
        if (nb < A.nblk) {
            const uint32_t gn = A.g_begin + nb * (kAdamThreads / 2) + (threadIdx.x >> 1);
            if (gn < A.g_end) {
                const size_t o = (size_t)gn * 8 + 4 * (threadIdx.x & 1);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(A.params + o));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(A.m + o));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(A.v + o));
            }
        }
        adam_block<Tail>(A, blk);
    }
}

}  // namespace
