// knn.cu -- exact top-K at scattered points (training samples, point
// queries) by branch-and-bound over a loose quadtree of the Gaussians.
//
// The reference scans all N Gaussians per sample (fit.cpp:65-84 ->
// select_top_k_entries over ps.all_indices(), renderer.cpp:53-74).
//
// Structure (rebuilt whenever the set changes): level l is a G_l x G_l grid
// (G_l = G0 >> l) over [0,1]^2.  Each Gaussian is stored at the finest
// level whose cell is at least twice its largest standard deviation
// (sigma_max = 1/sqrt(min(1/s1^2, 1/s2^2))), in the cell holding its
// centre -- so a cell's own members have sizes comparable to the cell and
// Adam's quickly diverging scales (0.2 px .. 30 px after a dozen steps at
// 2048^2) never loosen a bound.  Every cell keeps two summaries: its own
// members and its whole subtree (own + children): centre bbox, smallest
// Sigma^-1 eigenvalue lambda_min, a safety factor and a count.
//
// Certified bound: for every member g of a summary and point p,
//   fl(q(g, p)) >= lambda_min * dist(p, bbox)^2 * slack,
// since q >= lambda_min |p - mu|^2 in exact arithmetic and |fl(q) - q| <=
// 9u (ia+ib) L1^2 <= 18u (1 + aniso) q (forward error of renderer.cpp:17-23);
// slack = 1 - 2^-20 - 256u (1 + max aniso) also absorbs the bound's own
// rounding.  A summary is skipped only if its bound exceeds tq, the current
// kk-th best q (strictly, so index ties are never pruned).
//
// Query: one warp per point.  (1) Seed: the own members of the 3x3 cells
// around the point at every level (big Gaussians included) give a tight tq
// at once.  (2) Level-synchronous descent from the root: frontier nodes'
// own members (outside the seed windows) are evaluated, children whose
// subtree bound <= tq form the next frontier.  Members are evaluated 32 at a
// time with maha() (the scan's exact op sequence); those beating tq are
// inserted in lane order into a top-K replicated in every lane, so the kept
// set is exactly the kk smallest (q, idx) -- the reference's selection.
// A frontier larger than the per-warp queue restarts over all N (exact).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>

#include "igs_internal.cuh"

using namespace igs_dev;

namespace {

constexpr int kMaxLv = 13;
constexpr int kQueue = 512;  // per-warp frontier capacity

struct Sum {
    double x0, y0, x1, y1;  // centre bbox (empty: +inf/-inf)
    double lmin;            // smallest Sigma^-1 eigenvalue
    float slack;            // bound safety factor (0 = never prune)
    uint32_t count;
};

struct Lq {
    int G0, levels;
    int lw[kMaxLv];    // cells per side
    int loff[kMaxLv];  // first cell id of the level
};

__device__ __forceinline__ int cell_of(double v, int G) {
    const double f = floor(v * (double)G);
    return isfinite(f) ? (int)fmin(fmax(f, 0.0), (double)(G - 1)) : 0;
}

__device__ __forceinline__ float slack_for(double aniso) {
    const double s = 1.0 - (9.5367431640625e-07 + 256.0 * 1.1102230246251565e-16 * (1.0 + aniso));
    return s > 0.5 ? (float)(s - 1e-7) : 0.0f;
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

__global__ void lq_count(const ScanRec* __restrict__ scan, uint32_t n, Lq L, uint32_t* __restrict__ cnt,
                         uint32_t* __restrict__ key) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = key_of(L, scan[i]);
    key[i] = k;
    atomicAdd(cnt + k, 1u);
}

__global__ void lq_fill(uint32_t n, const uint32_t* __restrict__ key, const uint32_t* __restrict__ off,
                        uint32_t* __restrict__ cur, uint32_t* __restrict__ mem) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = key[i];
    mem[off[k] + atomicAdd(cur + k, 1u)] = i;
}

__device__ __forceinline__ Sum empty_sum() {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    Sum s;
    s.x0 = inf; s.y0 = inf; s.x1 = -inf; s.y1 = -inf;
    s.lmin = inf;
    s.slack = 1.0f;
    s.count = 0;
    return s;
}

__device__ __forceinline__ void merge(Sum& a, const Sum& b) {
    if (b.count == 0) return;
    a.x0 = fmin(a.x0, b.x0); a.x1 = fmax(a.x1, b.x1);
    a.y0 = fmin(a.y0, b.y0); a.y1 = fmax(a.y1, b.y1);
    a.lmin = fmin(a.lmin, b.lmin);
    a.slack = fminf(a.slack, b.slack);
    a.count += b.count;
}

// own summary of every cell (all levels), one thread per cell
__global__ void lq_own(const ScanRec* __restrict__ scan, uint32_t ncells, const uint32_t* __restrict__ cnt,
                       const uint32_t* __restrict__ off, const uint32_t* __restrict__ mem, Sum* __restrict__ own) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    Sum s = empty_sum();
    double aniso = 1.0;
    const uint32_t o = off[c], m = cnt[c];
    for (uint32_t j = 0; j < m; ++j) {
        const ScanRec r = scan[mem[o + j]];
        s.x0 = fmin(s.x0, r.mu_x); s.x1 = fmax(s.x1, r.mu_x);
        s.y0 = fmin(s.y0, r.mu_y); s.y1 = fmax(s.y1, r.mu_y);
        const double lo = fmin(r.inv_a, r.inv_b), hi = fmax(r.inv_a, r.inv_b);
        s.lmin = fmin(s.lmin, lo);
        aniso = fmax(aniso, hi / lo);
        if (!(lo > 0.0) || !isfinite(hi) || !isfinite(r.mu_x) || !isfinite(r.mu_y)) aniso = __longlong_as_double(0x7ff0000000000000LL);
    }
    s.slack = slack_for(aniso);
    s.count = m;
    own[c] = s;
}

// subtree summaries of one level from its own + the finer level's subtrees
__global__ void lq_subtree(Lq L, int level, const Sum* __restrict__ own, Sum* __restrict__ sub) {
    const int w = L.lw[level];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * w) return;
    Sum s = own[L.loff[level] + i];
    if (level > 0) {
        const int x = i % w, y = i / w, cw = L.lw[level - 1];
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const int cx = 2 * x + dx, cy = 2 * y + dy;
                if (cx < cw && cy < cw) merge(s, sub[L.loff[level - 1] + cy * cw + cx]);
            }
    }
    sub[L.loff[level] + i] = s;
}

__device__ __forceinline__ double sum_lb(const Sum& s, double px, double py) {
    if (s.count == 0) return __longlong_as_double(0x7ff0000000000000LL);
    const double dx = fmax(fmax(s.x0 - px, px - s.x1), 0.0);
    const double dy = fmax(fmax(s.y0 - py, py - s.y1), 0.0);
    return s.lmin * (dx * dx + dy * dy) * (double)s.slack;
}

// Evaluates the members of up to 32 cells (lane i: range [o_i, o_i + m_i)),
// flattened so that all lanes work on members.
template <int KCAP>
__device__ __forceinline__ void eval_members(TopK<KCAP>& t, uint32_t o_mine, uint32_t m_mine, int lane,
                                             const ScanRec* __restrict__ scan, const uint32_t* __restrict__ mem,
                                             double px, double py, unsigned long long& evaluated) {
    uint32_t incl = m_mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - m_mine;
    evaluated += total;
    for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t f = base + lane;
        // cell holding flat member f: largest i with excl_i <= f (excl is
        // non-decreasing; an empty cell never beats the one holding f)
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t ex = __shfl_sync(0xffffffffu, excl, lo + step);
            if (ex <= f) lo += step;
        }
        const uint32_t lo_ex = __shfl_sync(0xffffffffu, excl, lo);
        const uint32_t lo_o = __shfl_sync(0xffffffffu, o_mine, lo);
        double q = 0.0;
        uint32_t gi = kNoIdx;
        bool cand = false;
        if (f < total) {
            gi = __ldg(mem + lo_o + (f - lo_ex));
            q = maha(scan[gi], px, py);
            cand = t.beats(q, gi);
        }
        unsigned msk = __ballot_sync(0xffffffffu, cand);
        while (msk) {
            const int src = __ffs(msk) - 1;
            msk &= msk - 1;
            const double qq = __shfl_sync(0xffffffffu, q, src);
            const uint32_t ii = __shfl_sync(0xffffffffu, gi, src);
            t.offer(qq, ii);
        }
    }
}

__device__ __forceinline__ bool in_seed(const Lq& L, int l, int x, int y, double px, double py) {
    const int sx = cell_of(px, L.lw[l]), sy = cell_of(py, L.lw[l]);
    return x >= sx - 1 && x <= sx + 1 && y >= sy - 1 && y <= sy + 1;
}

// One warp per point.
constexpr uint32_t kHardCap = 256;

template <int KCAP>
__global__ void __launch_bounds__(128, 4) knn_points_kernel(const ScanRec* __restrict__ scan, uint32_t n, Lq L,
                                                            const Sum* __restrict__ own, const Sum* __restrict__ sub,
                                                            const uint32_t* __restrict__ off,
                                                            const uint32_t* __restrict__ mem,
                                                            const double* __restrict__ uv, uint32_t npts, int kk,
                                                            double* __restrict__ oq, uint32_t* __restrict__ oi,
                                                            unsigned long long* __restrict__ pairs,
                                                            uint32_t* __restrict__ hard_count,
                                                            uint32_t* __restrict__ hard_list) {
    __shared__ uint32_t queue[4][2][kQueue];
    const int warp = threadIdx.x >> 5;
    const uint32_t pt = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (pt >= npts) return;  // warp-uniform
    const double px = uv[2 * (size_t)pt], py = uv[2 * (size_t)pt + 1];
    TopK<KCAP> t;
    t.init(kk);
    unsigned long long evaluated = 0;

    // (1) seeds: own members of the 3x3 window at every level
    const int nseed = L.levels * 9;
    for (int base = 0; base < nseed; base += 32) {
        const int it = base + lane;
        uint32_t o = 0, m = 0;
        if (it < nseed) {
            const int l = it / 9, d = it % 9, G = L.lw[l];
            const int x = cell_of(px, G) + d % 3 - 1, y = cell_of(py, G) + d / 3 - 1;
            if (x >= 0 && x < G && y >= 0 && y < G) {
                const uint32_t c = (uint32_t)(L.loff[l] + y * G + x);
                o = off[c];
                m = own[c].count;
            }
        }
        eval_members(t, o, m, lane, scan, mem, px, py, evaluated);
    }

    // (2) descent: evaluate own members of frontier nodes, expand children
    uint32_t* cur = queue[warp][0];
    uint32_t* nxt = queue[warp][1];
    int ncur = 1;
    if (lane == 0) cur[0] = 0;  // root cell of the top level
    __syncwarp();
    bool overflow = false;
    for (int l = L.levels - 1; l >= 0 && ncur > 0; --l) {
        const int w = L.lw[l];
        // own members of the frontier (outside the seed window)
        for (int base = 0; base < ncur; base += 32) {
            const int i = base + lane;
            uint32_t o = 0, m = 0;
            if (i < ncur) {
                const uint32_t node = cur[i];
                const int x = node % w, y = node / w;
                const uint32_t c = (uint32_t)L.loff[l] + node;
                if (!in_seed(L, l, x, y, px, py)) {
                    const Sum so = own[c];
                    if (so.count && sum_lb(so, px, py) <= t.tq()) {
                        o = off[c];
                        m = so.count;
                    }
                }
            }
            eval_members(t, o, m, lane, scan, mem, px, py, evaluated);
        }
        if (l == 0) break;
        const int cw = L.lw[l - 1];
        int nnext = 0;
        for (int base = 0; base < ncur * 4; base += 32) {
            const int item = base + lane;
            bool keep = false;
            uint32_t child = 0;
            if (item < ncur * 4) {
                const uint32_t node = cur[item >> 2];
                const int x = node % w, y = node / w;
                const int ccx = 2 * x + (item & 1), ccy = 2 * y + ((item >> 1) & 1);
                if (ccx < cw && ccy < cw) {
                    child = (uint32_t)(ccy * cw + ccx);
                    keep = sum_lb(sub[L.loff[l - 1] + child], px, py) <= t.tq();
                }
            }
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            const int pos = nnext + __popc(msk & ((1u << lane) - 1));
            if (keep && pos < kQueue) nxt[pos] = child;
            nnext += __popc(msk);
        }
        __syncwarp();
        if (nnext > kQueue) {
            overflow = true;
            break;
        }
        uint32_t* tmp = cur;
        cur = nxt;
        nxt = tmp;
        ncur = nnext;
    }

    if (overflow) {
        // the frontier outgrew the queue: hand the point to hard_points_kernel
        // (one CTA scans all N); beyond its capacity, scan all N here
        uint32_t slot = 0;
        if (lane == 0) slot = atomicAdd(hard_count, 1u);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot < kHardCap) {
            if (lane == 0) hard_list[slot] = pt;
            return;
        }
        t.init(kk);
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t gi = base + lane;
            double q = 0.0;
            bool cand = false;
            if (gi < n) {
                q = maha(scan[gi], px, py);
                cand = t.beats(q, gi);
            }
            unsigned msk = __ballot_sync(0xffffffffu, cand);
            while (msk) {
                const int src = __ffs(msk) - 1;
                msk &= msk - 1;
                const double qq = __shfl_sync(0xffffffffu, q, src);
                t.offer(qq, base + src);
            }
        }
        evaluated += n;
    }
    if (pairs && lane == 0) atomicAdd(pairs, evaluated);
    if (lane == 0) store_topk(t, oq + (size_t)pt * kk, oi + (size_t)pt * kk);
}

// One CTA per hard point: 128 threads scan all N (coalesced 48-B records),
// each keeping a private top-K; warp 0 folds the 128 lists into 32 lane
// lists, then kk rounds of a warp-wide (q, idx) minimum emit the result.
// Exact: the kept set is the kk smallest (q, idx) of the union.
constexpr int kHardThreads = 128;

template <int KCAP>
__global__ void __launch_bounds__(kHardThreads) hard_points_kernel(const ScanRec* __restrict__ scan, uint32_t n,
                                                                   const double* __restrict__ uv, int kk,
                                                                   const uint32_t* __restrict__ hard_count,
                                                                   const uint32_t* __restrict__ hard_list,
                                                                   double* __restrict__ oq, uint32_t* __restrict__ oi,
                                                                   unsigned long long* __restrict__ pairs) {
    __shared__ double sq[kHardThreads * KCAP];
    __shared__ uint32_t si[kHardThreads * KCAP];
    const uint32_t cnt = min(*hard_count, kHardCap);
    if (blockIdx.x >= cnt) return;
    const uint32_t pt = hard_list[blockIdx.x];
    const double px = uv[2 * (size_t)pt], py = uv[2 * (size_t)pt + 1];
    TopK<KCAP> t;
    t.init(kk);
    for (uint32_t g = threadIdx.x; g < n; g += kHardThreads) {
        const double q = maha(scan[g], px, py);
        if (q <= t.tq()) t.offer(q, g);
    }
    store_topk(t, sq + threadIdx.x * KCAP, si + threadIdx.x * KCAP);
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    TopK<KCAP> m;
    m.init(kk);
    for (int th = lane; th < kHardThreads; th += 32)
        for (int j = 0; j < kk; ++j) {
            const uint32_t ci = si[th * KCAP + j];
            if (ci == kNoIdx) break;
            m.offer(sq[th * KCAP + j], ci);
        }
    __syncwarp();
    store_topk(m, sq + lane * KCAP, si + lane * KCAP);
    __syncwarp();
    int head = 0;
    for (int r = 0; r < kk; ++r) {
        double v = head < kk ? sq[lane * KCAP + head] : __longlong_as_double(0x7ff0000000000000LL);
        uint32_t vi = head < kk ? si[lane * KCAP + head] : kNoIdx;
        int who = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const uint32_t ovi = __shfl_xor_sync(0xffffffffu, vi, o);
            const int ow = __shfl_xor_sync(0xffffffffu, who, o);
            if (ov < v || (ov == v && ovi < vi) || (ov == v && ovi == vi && ow < who)) {
                v = ov;
                vi = ovi;
                who = ow;
            }
        }
        if (lane == who) ++head;
        if (lane == 0) {
            oq[(size_t)pt * kk + r] = v;
            oi[(size_t)pt * kk + r] = vi;
        }
    }
    if (pairs && lane == 0) atomicAdd(pairs, (unsigned long long)n);
}

struct KnnBufs {
    DevBuf cnt, off, key, mem, own, sub, cub_tmp, hard;
    uint64_t version = ~0ull;
    Lq lq{};
};

void* grow(DevBuf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return b.p;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    b.bytes = bytes;
    return b.p;
}

int knn_build(igs_ctx* ctx) {
    if (!ctx->knn) ctx->knn = new KnnBufs();
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    if (b.version == ctx->params_version) return IGS_OK;
    const uint32_t n = ctx->n;
    int G0 = 16;  // finest grid: about 2 centres per cell
    while (G0 < 4096 && (uint64_t)G0 * G0 * 2 < n) G0 *= 2;
    Lq L{};
    L.G0 = G0;
    int l = 0, w = G0, o = 0;
    for (;;) {
        L.lw[l] = w;
        L.loff[l] = o;
        o += w * w;
        ++l;
        if (w == 1) break;
        w /= 2;
    }
    L.levels = l;
    const uint32_t cells = (uint32_t)o;
    if (!grow(b.cnt, (size_t)cells * 8) || !grow(b.off, (size_t)cells * 4) || !grow(b.key, (size_t)n * 4) ||
        !grow(b.mem, (size_t)n * 4) || !grow(b.own, (size_t)cells * sizeof(Sum)) ||
        !grow(b.sub, (size_t)cells * sizeof(Sum)))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
    uint32_t* cnt = (uint32_t*)b.cnt.p;
    uint32_t* cur = cnt + cells;
    uint32_t* off = (uint32_t*)b.off.p;
    igs_prof_begin(ctx, IGS_PROF_CULL);
    IGS_CUDA(ctx, cudaMemsetAsync(cnt, 0, (size_t)cells * 8, ctx->stream));
    lq_count<<<(n + 255) / 256, 256, 0, ctx->stream>>>(ctx->scan, n, L, cnt, (uint32_t*)b.key.p);
    IGS_LAUNCHED(ctx);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)cells, ctx->stream);
    if (!grow(b.cub_tmp, tb)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn scan)");
    IGS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(b.cub_tmp.p, tb, cnt, off, (int)cells, ctx->stream));
    ctx->launches += 2;
    lq_fill<<<(n + 255) / 256, 256, 0, ctx->stream>>>(n, (const uint32_t*)b.key.p, off, cur, (uint32_t*)b.mem.p);
    IGS_LAUNCHED(ctx);
    lq_own<<<(cells + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, cells, cnt, off, (const uint32_t*)b.mem.p,
                                                         (Sum*)b.own.p);
    IGS_LAUNCHED(ctx);
    for (int lv = 0; lv < L.levels; ++lv) {
        const int m = L.lw[lv] * L.lw[lv];
        lq_subtree<<<(m + 127) / 128, 128, 0, ctx->stream>>>(L, lv, (const Sum*)b.own.p, (Sum*)b.sub.p);
        IGS_LAUNCHED(ctx);
    }
    igs_prof_end(ctx, IGS_PROF_CULL, 0.0);
    b.lq = L;
    b.version = ctx->params_version;
    return IGS_OK;
}

template <int KCAP>
int launch_knn(igs_ctx* ctx, const double* uv, uint32_t npts, int kk, uint32_t* oi, double* oq) {
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    if (!grow(b.hard, (kHardCap + 1) * 4)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
    uint32_t* hard_count = (uint32_t*)b.hard.p;
    uint32_t* hard_list = hard_count + 1;
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    IGS_CUDA(ctx, cudaMemsetAsync(hard_count, 0, 4, ctx->stream));
    const uint64_t threads = (uint64_t)npts * 32;
    knn_points_kernel<KCAP><<<(unsigned)((threads + 127) / 128), 128, 0, ctx->stream>>>(
        ctx->scan, ctx->n, b.lq, (const Sum*)b.own.p, (const Sum*)b.sub.p, (const uint32_t*)b.off.p,
        (const uint32_t*)b.mem.p, uv, npts, kk, oq, oi, igs_prof_counter(ctx, IGS_PROF_SCAN), hard_count,
        hard_list);
    IGS_LAUNCHED(ctx);
    hard_points_kernel<KCAP><<<kHardCap, kHardThreads, 0, ctx->stream>>>(ctx->scan, ctx->n, uv, kk, hard_count, hard_list,
                                                                oq, oi, igs_prof_counter(ctx, IGS_PROF_SCAN));
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
    return IGS_OK;
}

}  // namespace

void igs_knn_free(igs_ctx* ctx) {
    if (!ctx->knn) return;
    KnnBufs* b = static_cast<KnnBufs*>(ctx->knn);
    for (DevBuf* d : {&b->cnt, &b->off, &b->key, &b->mem, &b->own, &b->sub, &b->cub_tmp, &b->hard}) cudaFree(d->p);
    delete b;
    ctx->knn = nullptr;
}

// Exact top-K (q ascending, idx) at device points; kk = min(k, n).
int igs_topk_knn(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32 || npts == 0) return igs_topk_points(ctx, uv, npts, k, oi, oq);
    int e = knn_build(ctx);
    if (e) return e;
    if (kk <= 4) return launch_knn<4>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 8) return launch_knn<8>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 16) return launch_knn<16>(ctx, uv, npts, kk, oi, oq);
    return launch_knn<32>(ctx, uv, npts, kk, oi, oq);
}
