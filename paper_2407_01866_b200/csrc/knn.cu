// knn.cu -- exact top-K at scattered points (training samples, point
// queries) by branch-and-bound over a quadtree of Gaussian-centre bins.
//
// The reference scans all N Gaussians per sample (fit.cpp:65-84 ->
// select_top_k_entries over ps.all_indices(), renderer.cpp:53-74).  Here:
//   build (per set state): Gaussians bucketed into G x G centre cells
//     (count / scan / fill), then a pyramid whose node stores the bbox of its
//     members' centres, the smallest eigenvalue of their Sigma^-1
//     (min(1/s1^2, 1/s2^2)), the largest anisotropy and a member count.
//   query: one warp per point walks the pyramid near-first with an explicit
//     stack.  A node is pruned iff its lower bound lb > tq, the current kk-th
//     best q (strict, so index ties are never pruned).  lb = lambda_min *
//     dist(p, bbox)^2 * (1 - slack): q >= lambda_min |x - mu|^2 in exact
//     arithmetic, and slack covers |fl(q) - q| <= 9u (ia+ib) L1^2 <=
//     18u (1 + aniso) q (forward error of renderer.cpp:17-23) plus the
//     rounding of the bound itself.  Leaves: lanes evaluate 32 members at a
//     time with maha() (the scan's exact op sequence); candidates that beat
//     tq are inserted in lane order into a top-K replicated in every lane,
//     so the kept set is exactly the kk smallest (q, idx) -- the reference's
//     selection -- whatever the visit order.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>

#include "igs_internal.cuh"

using namespace igs_dev;

namespace {

constexpr int kMaxLv = 12;

struct Node {
    double x0, y0, x1, y1;  // bbox of member centres (empty: +inf, -inf)
    double lmin;            // min over members of min(ia, ib)
    float slack;            // multiplicative safety factor for lb (0 = no pruning)
    uint32_t count;         // members in the subtree
};

struct Pyr {
    int G;  // cells per side at level 0
    int levels;
    int lw[kMaxLv], loff[kMaxLv];
};

__device__ __forceinline__ int cell_of(double v, int G) {
    const double f = floor(v * (double)G);
    return isfinite(f) ? (int)fmin(fmax(f, 0.0), (double)(G - 1)) : 0;
}

__global__ void knn_bin_count(const ScanRec* __restrict__ scan, uint32_t n, int G, uint32_t* __restrict__ cnt,
                              uint32_t* __restrict__ bin_of) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = cell_of(scan[i].mu_y, G) * G + cell_of(scan[i].mu_x, G);
    bin_of[i] = (uint32_t)c;
    atomicAdd(cnt + c, 1u);
}

__global__ void knn_bin_fill(uint32_t n, const uint32_t* __restrict__ bin_of, const uint32_t* __restrict__ off,
                             uint32_t* __restrict__ cur, uint32_t* __restrict__ bins) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = bin_of[i];
    bins[off[c] + atomicAdd(cur + c, 1u)] = i;
}

__device__ __forceinline__ float slack_for(double aniso) {
    // 1 - (2^-20 + 256 u (1 + aniso)); no pruning if the bound degrades
    const double s = 1.0 - (9.5367431640625e-07 + 256.0 * 1.1102230246251565e-16 * (1.0 + aniso));
    return s > 0.5 ? (float)(s - 1e-7) : 0.0f;  // round the float down
}

// level-0 nodes: one thread per cell reduces its members
__global__ void knn_leaf_nodes(const ScanRec* __restrict__ scan, int G, const uint32_t* __restrict__ cnt,
                               const uint32_t* __restrict__ off, const uint32_t* __restrict__ bins,
                               Node* __restrict__ nodes) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= G * G) return;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    Node nd;
    nd.x0 = inf; nd.y0 = inf; nd.x1 = -inf; nd.y1 = -inf;
    nd.lmin = inf;
    double aniso = 1.0;
    const uint32_t o = off[c], m = cnt[c];
    for (uint32_t j = 0; j < m; ++j) {
        const ScanRec r = scan[bins[o + j]];
        nd.x0 = fmin(nd.x0, r.mu_x); nd.x1 = fmax(nd.x1, r.mu_x);
        nd.y0 = fmin(nd.y0, r.mu_y); nd.y1 = fmax(nd.y1, r.mu_y);
        const double lo = fmin(r.inv_a, r.inv_b), hi = fmax(r.inv_a, r.inv_b);
        nd.lmin = fmin(nd.lmin, lo);
        aniso = fmax(aniso, hi / lo);
        if (!(lo > 0.0) || !isfinite(hi) || !isfinite(r.mu_x) || !isfinite(r.mu_y)) aniso = inf;
    }
    nd.slack = slack_for(aniso);
    nd.count = m;
    nodes[c] = nd;
}

__global__ void knn_up_nodes(Pyr p, int level, Node* __restrict__ nodes) {
    const int w = p.lw[level];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * w) return;
    const int x = i % w, y = i / w, cw = p.lw[level - 1];
    const Node* ch = nodes + p.loff[level - 1];
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    Node nd;
    nd.x0 = inf; nd.y0 = inf; nd.x1 = -inf; nd.y1 = -inf;
    nd.lmin = inf;
    nd.slack = 1.0f;
    nd.count = 0;
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            const int cx = 2 * x + dx, cy = 2 * y + dy;
            if (cx >= cw || cy >= cw) continue;
            const Node c = ch[cy * cw + cx];
            if (c.count == 0) continue;
            nd.x0 = fmin(nd.x0, c.x0); nd.x1 = fmax(nd.x1, c.x1);
            nd.y0 = fmin(nd.y0, c.y0); nd.y1 = fmax(nd.y1, c.y1);
            nd.lmin = fmin(nd.lmin, c.lmin);
            nd.slack = fminf(nd.slack, c.slack);
            nd.count += c.count;
        }
    nodes[p.loff[level] + i] = nd;
}

// Certified lower bound of fl(q(g, p)) for every member g of the node.
__device__ __forceinline__ double node_lb(const Node& nd, double px, double py) {
    if (nd.count == 0) return __longlong_as_double(0x7ff0000000000000LL);
    const double dx = fmax(fmax(nd.x0 - px, px - nd.x1), 0.0);
    const double dy = fmax(fmax(nd.y0 - py, py - nd.y1), 0.0);
    return nd.lmin * (dx * dx + dy * dy) * (double)nd.slack;
}

// One warp per point.
template <int KCAP>
__global__ void __launch_bounds__(128) knn_points_kernel(const ScanRec* __restrict__ scan, Pyr p,
                                                         const Node* __restrict__ nodes,
                                                         const uint32_t* __restrict__ off,
                                                         const uint32_t* __restrict__ bins,
                                                         const double* __restrict__ uv, uint32_t npts, int kk,
                                                         double* __restrict__ oq, uint32_t* __restrict__ oi,
                                                         unsigned long long* __restrict__ pairs) {
    const uint32_t pt = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (pt >= npts) return;  // warp-uniform
    const double px = uv[2 * (size_t)pt], py = uv[2 * (size_t)pt + 1];
    TopK<KCAP> t;
    t.init(kk);
    unsigned long long evaluated = 0;
    uint32_t stack[3 * kMaxLv + 4];
    int sp = 0;
    stack[sp++] = (uint32_t)(p.levels - 1) << 26;
    while (sp > 0) {
        const uint32_t e = stack[--sp];
        const int l = e >> 26, x = (e >> 13) & 0x1fff, y = e & 0x1fff;
        const int w = p.lw[l];
        const Node nd = nodes[p.loff[l] + y * w + x];
        if (!(node_lb(nd, px, py) <= t.tq())) continue;
        if (l == 0) {
            const uint32_t o = off[y * w + x], m = nd.count;
            for (uint32_t base = 0; base < m; base += 32) {
                const uint32_t j = base + lane;
                double q = 0.0;
                uint32_t gi = kNoIdx;
                bool cand = false;
                if (j < m) {
                    gi = __ldg(bins + o + j);
                    q = maha(scan[gi], px, py);
                    cand = t.beats(q, gi);
                }
                evaluated += min(32u, m - base);
                unsigned msk = __ballot_sync(0xffffffffu, cand);
                while (msk) {
                    const int src = __ffs(msk) - 1;
                    msk &= msk - 1;
                    const double qq = __shfl_sync(0xffffffffu, q, src);
                    const uint32_t ii = __shfl_sync(0xffffffffu, gi, src);
                    t.offer(qq, ii);
                }
            }
            continue;
        }
        // children: lane c < 4 computes child c's bound; push far-first
        const int cw = p.lw[l - 1];
        double lb = __longlong_as_double(0x7ff0000000000000LL);
        uint32_t code = 0;
        if (lane < 4) {
            const int cx = 2 * x + (lane & 1), cy = 2 * y + (lane >> 1);
            if (cx < cw && cy < cw) {
                lb = node_lb(nodes[p.loff[l - 1] + cy * cw + cx], px, py);
                code = ((uint32_t)(l - 1) << 26) | ((uint32_t)cx << 13) | (uint32_t)cy;
            }
        }
        double cl[4];
        uint32_t cc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            cl[c] = __shfl_sync(0xffffffffu, lb, c);
            cc[c] = __shfl_sync(0xffffffffu, code, c);
        }
        // sort 4 descending by bound (uniform across lanes)
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3 - a; ++b)
                if (cl[b] < cl[b + 1]) {
                    const double tl = cl[b]; cl[b] = cl[b + 1]; cl[b + 1] = tl;
                    const uint32_t tc = cc[b]; cc[b] = cc[b + 1]; cc[b + 1] = tc;
                }
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (cl[c] <= t.tq() && sp < 3 * kMaxLv + 4) stack[sp++] = cc[c];
    }
    if (pairs && lane == 0) atomicAdd(pairs, evaluated);
    if (lane == 0) store_topk(t, oq + (size_t)pt * kk, oi + (size_t)pt * kk);
}

struct KnnBufs {
    DevBuf cnt, off, bin_of, bins, nodes, cub_tmp;
    uint64_t version = ~0ull;
    Pyr pyr{};
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
    int G = 16;  // ~4 centres per cell
    while (G < 2048 && (uint64_t)G * G * 4 < n) G *= 2;
    Pyr p{};
    p.G = G;
    int l = 0, w = G, o = 0;
    for (;;) {
        p.lw[l] = w;
        p.loff[l] = o;
        o += w * w;
        ++l;
        if (w == 1) break;
        w /= 2;
    }
    p.levels = l;
    const int cells = G * G;
    if (!grow(b.cnt, (size_t)cells * 8) || !grow(b.off, (size_t)cells * 4) || !grow(b.bin_of, (size_t)n * 4) ||
        !grow(b.bins, (size_t)n * 4) || !grow(b.nodes, (size_t)o * sizeof(Node)))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
    uint32_t* cnt = (uint32_t*)b.cnt.p;
    uint32_t* cur = cnt + cells;
    uint32_t* off = (uint32_t*)b.off.p;
    igs_prof_begin(ctx, IGS_PROF_CULL);
    IGS_CUDA(ctx, cudaMemsetAsync(cnt, 0, (size_t)cells * 8, ctx->stream));
    knn_bin_count<<<(n + 255) / 256, 256, 0, ctx->stream>>>(ctx->scan, n, G, cnt, (uint32_t*)b.bin_of.p);
    IGS_LAUNCHED(ctx);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, cells, ctx->stream);
    if (!grow(b.cub_tmp, tb)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn scan)");
    IGS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(b.cub_tmp.p, tb, cnt, off, cells, ctx->stream));
    ctx->launches += 2;
    knn_bin_fill<<<(n + 255) / 256, 256, 0, ctx->stream>>>(n, (const uint32_t*)b.bin_of.p, off, cur,
                                                           (uint32_t*)b.bins.p);
    IGS_LAUNCHED(ctx);
    Node* nodes = (Node*)b.nodes.p;
    knn_leaf_nodes<<<(cells + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, G, cnt, off, (const uint32_t*)b.bins.p,
                                                                 nodes);
    IGS_LAUNCHED(ctx);
    for (int lv = 1; lv < p.levels; ++lv) {
        const int m = p.lw[lv] * p.lw[lv];
        knn_up_nodes<<<(m + 127) / 128, 128, 0, ctx->stream>>>(p, lv, nodes);
        IGS_LAUNCHED(ctx);
    }
    igs_prof_end(ctx, IGS_PROF_CULL, 0.0);
    b.pyr = p;
    b.version = ctx->params_version;
    return IGS_OK;
}

template <int KCAP>
int launch_knn(igs_ctx* ctx, const double* uv, uint32_t npts, int kk, uint32_t* oi, double* oq) {
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    const uint64_t threads = (uint64_t)npts * 32;
    knn_points_kernel<KCAP><<<(unsigned)((threads + 127) / 128), 128, 0, ctx->stream>>>(
        ctx->scan, b.pyr, (const Node*)b.nodes.p, (const uint32_t*)b.off.p, (const uint32_t*)b.bins.p, uv, npts, kk,
        oq, oi, igs_prof_counter(ctx, IGS_PROF_SCAN));
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
    return IGS_OK;
}

}  // namespace

void igs_knn_free(igs_ctx* ctx) {
    if (!ctx->knn) return;
    KnnBufs* b = static_cast<KnnBufs*>(ctx->knn);
    for (DevBuf* d : {&b->cnt, &b->off, &b->bin_of, &b->bins, &b->nodes, &b->cub_tmp}) cudaFree(d->p);
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
