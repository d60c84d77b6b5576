// knn_tree.cuh -- the loose-quadtree pieces shared by the kNN search
// (knn.cu) and the Adam kernels (train.cu), which accumulate each updated
// Gaussian into its cell's summary accumulator so the next search only
// re-derives the summaries (no re-bucketing) -- see knn.cu for the
// structure and the certified bound.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_internal.cuh"

namespace igs_dev {

constexpr int kMaxLv = 13;
// key[i] = cell | level << 27 (cells < 2^25 for G0 <= 4096)
constexpr int kKeyLevelShift = 27;
constexpr uint32_t kKeyCellMask = (1u << kKeyLevelShift) - 1;

struct Lq {
    int G0, levels;
    int lw[kMaxLv];    // cells per side
    int loff[kMaxLv];  // first cell id of the level
    const uint32_t* lcount;  // Gaussians stored per level (device)
};

__device__ __forceinline__ int cell_of(double v, int G) {
    const double f = floor(v * (double)G);
    return isfinite(f) ? (int)fmin(fmax(f, 0.0), (double)(G - 1)) : 0;
}

// Level whose cell (1/G_l) is >= 2 sigma_max: 4 G_l^2 <= lmin.
__device__ __forceinline__ int level_of(const Lq& L, double lmin) {
    int l = 0;
    while (l < L.levels - 1 && !(4.0 * (double)L.lw[l] * (double)L.lw[l] <= lmin)) ++l;
    return l;
}

__device__ __forceinline__ uint32_t key_of(const Lq& L, const ScanRec& r) {
    const int l = level_of(L, fmin(r.inv_a, r.inv_b));
    const int G = L.lw[l];
    return (uint32_t)(L.loff[l] + cell_of(r.mu_y, G) * G + cell_of(r.mu_x, G));
}

// Own-cell summaries are accumulated with order-preserving 32-bit min/max
// over the member-ordered records (lq_tree_kernel: warp shuffles, then
// shared or global atomics per run of equal cells): a float's bit pattern,
// sign-flipped, orders like the float itself.  Values are rounded
// in the direction that keeps the summary conservative (bbox outward,
// lambda_min down, anisotropy up), as the 32-byte Sum stores them.
struct Acc {
    unsigned x0, y0, x1, y1, lmin, aniso;
};

__device__ __forceinline__ unsigned okey(float f) {
    const unsigned b = __float_as_uint(f);
    return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float odec(unsigned k) { return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k); }

// Adds Gaussian r to a cell accumulator held by one thread.  A non-finite
// or degenerate record gets aniso = inf, whose slack 0 makes the cell never
// prunable.
__device__ __forceinline__ void acc_add_local(Acc& a, const ScanRec& r) {
    const double lo = fmin(r.inv_a, r.inv_b), hi = fmax(r.inv_a, r.inv_b);
    double aniso = hi / lo;
    if (!(lo > 0.0) || !isfinite(hi) || !isfinite(r.mu_x) || !isfinite(r.mu_y))
        aniso = __longlong_as_double(0x7ff0000000000000LL);
    a.x0 = min(a.x0, okey(__double2float_rd(r.mu_x)));
    a.y0 = min(a.y0, okey(__double2float_rd(r.mu_y)));
    a.x1 = max(a.x1, okey(__double2float_ru(r.mu_x)));
    a.y1 = max(a.y1, okey(__double2float_ru(r.mu_y)));
    a.lmin = min(a.lmin, okey(__double2float_rd(lo)));
    a.aniso = max(a.aniso, okey(__double2float_ru(aniso)));
}

// An accumulator other CTAs folded into with atomics: read through L2.
__device__ __forceinline__ Acc acc_ldcg(const Acc* a) {
    const unsigned* u = reinterpret_cast<const unsigned*>(a);
    return Acc{__ldcg(u), __ldcg(u + 1), __ldcg(u + 2), __ldcg(u + 3), __ldcg(u + 4), __ldcg(u + 5)};
}

__device__ __forceinline__ Acc acc_empty() {
    const float inf = __int_as_float(0x7f800000);
    return Acc{okey(inf), okey(inf), okey(-inf), okey(-inf), okey(inf), okey(1.0f)};
}

// What an Adam launch needs to keep the tree refittable: acc == nullptr
// means "do not accumulate" (the next search rebuilds).
struct TreeAcc {
    Acc* acc;
    const uint32_t* key;            // cell of every Gaussian at the last rebuild
    unsigned long long* grown;      // Gaussians now too large for their level
    Lq L;
    ScanRec* mrec;                  // the records in member order (kept current)
    const uint32_t* minv;           // position of every Gaussian there
};

// Stores Gaussian i's new record r at its member position (the refit reads
// it there) and counts it in *grown when its scale now calls for a coarser level than the one it is
// stored at: such a Gaussian weakens the bounds of its cell and every
// ancestor, so the host re-buckets before the next search (knn_build).  The
// level here is a float estimate of level_of: it only steers that decision.
__device__ __forceinline__ void tree_acc_add(const TreeAcc& ta, uint32_t i, const ScanRec& r) {
    if (!ta.acc) return;
    const uint32_t k = ta.key[i];
    // the member-ordered copy the searches read; the next refit re-derives
    // every cell summary from it (lq_tree_kernel), so no atomics here
    ta.mrec[ta.minv[i]] = r;
    // level_of: smallest l with cell 2^l / G0 >= 2 sigma_max = 2 / sqrt(lmin)
    const float lmin = (float)fmin(r.inv_a, r.inv_b);
    const float l = fminf(ceilf(log2f(2.0f * (float)ta.L.G0 * rsqrtf(lmin))), (float)(ta.L.levels - 1));
    const bool grew = l > (float)(k >> kKeyLevelShift);  // NaN compares false
    const unsigned act = __activemask();
    const unsigned m = __ballot_sync(act, grew);
    if (m && (threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(ta.grown, (unsigned long long)__popc(m));
}

}  // namespace igs_dev

// knn.cu: the accumulation target for an Adam launch that is about to bump
// params_version by exactly one ({nullptr, nullptr}: do not accumulate).
igs_dev::TreeAcc igs_knn_tree_acc(igs_ctx* ctx);
