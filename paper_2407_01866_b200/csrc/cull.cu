// cull.cu -- kernel 2: certified tile binning for the exact global top-K,
// and the culled top-K scans (kernel 3 over tile lists).
//
// Pipeline per (set state, raster grid, kk):
//   1. bin_count / scan / bin_fill : Gaussians bucketed by the tile holding
//      their centre (seeds for the bounds below).
//   2. tau_kernel      : one warp per tile; tau_T = kk-th smallest qmax_ub
//                        over the seeds of the 3x3 (5x5, ...) neighbourhood
//                        (warp-wide register top-K + shared-memory merge).
//   3. pyramid_kernel  : max-pyramid of tau (2x2 blocks per level).
//   4. emit_kernel x2  : per Gaussian, a descent of the pyramid pruned by
//                        qmin_lb(node box) > tau(node); leaves pass iff
//                        qmin_lb(g, T) <= tau_T.  Pass 1 counts per tile
//                        (atomics), a device prefix scan gives the tile
//                        offsets, pass 2 fills the lists.
//   5. consumers       : raster_culled_kernel (CTA per 16x16 tile, list staged
//                        through shared memory) and samples_culled_kernel
//                        (thread per sampled pixel centre).
// List order inside a tile is unspecified (atomic slots); the top-K order is
// a strict total order on (q, idx), so results do not depend on it.  A tile
// whose list exceeded the buffer capacity is detected by its consumer, which
// then scans all N candidates for that tile (exact, just slower); the host
// grows the buffer for the next build.  See cull_math.cuh for the proof.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "cull_math.cuh"
#include "igs_internal.cuh"
#include "scan.cuh"

using namespace igs_dev;
using igs_cull::G;

namespace {

constexpr int kTilePx = 16;
constexpr int kMaxLevels = 16;

struct Grid {
    int W, H;  // raster (pixel mode); unused in points mode
    int T;     // tile edge in pixels
    int TX, TY;
    int pts;   // 1: boxes [tx/TX, (tx+1)/TX] for arbitrary points
    int levels;
    int lw[kMaxLevels], lh[kMaxLevels], loff[kMaxLevels];
};

// Box (closed) covering tiles [tx0, tx1] x [ty0, ty1]: the hull of their
// pixel centres (pixel mode) or of the cells (points mode).
__device__ __forceinline__ void box_of(const Grid& gr, int tx0, int tx1, int ty0, int ty1, double& x0, double& x1,
                                       double& y0, double& y1) {
    if (gr.pts) {
        x0 = (double)tx0 / (double)gr.TX;
        x1 = (double)(tx1 + 1) / (double)gr.TX;
        y0 = (double)ty0 / (double)gr.TY;
        y1 = (double)(ty1 + 1) / (double)gr.TY;
    } else {
        x0 = center(tx0 * gr.T, gr.W);
        x1 = center(min(gr.W, (tx1 + 1) * gr.T) - 1, gr.W);
        y0 = center(ty0 * gr.T, gr.H);
        y1 = center(min(gr.H, (ty1 + 1) * gr.T) - 1, gr.H);
    }
}

__device__ __forceinline__ G load_g(const ScanRec& r) {
    G g;
    g.mx = r.mu_x;
    g.my = r.mu_y;
    g.c = r.cos_t;
    g.s = r.sin_t;
    g.ia = r.inv_a;
    g.ib = r.inv_b;
    igs_cull::conic(g);
    return g;
}

// Tile holding a Gaussian's centre (any assignment is valid; this one keeps
// seeds local).  pixel mode: column floor(mx*W) / T.
__device__ __forceinline__ int center_tile(const Grid& gr, double mx, double my) {
    int tx, ty;
    if (gr.pts) {
        const double fx = floor(mx * (double)gr.TX), fy = floor(my * (double)gr.TY);
        tx = isfinite(fx) ? (int)fmin(fmax(fx, 0.0), (double)(gr.TX - 1)) : 0;
        ty = isfinite(fy) ? (int)fmin(fmax(fy, 0.0), (double)(gr.TY - 1)) : 0;
    } else {
        const double fx = floor(mx * (double)gr.W), fy = floor(my * (double)gr.H);
        const int cx = isfinite(fx) ? (int)fmin(fmax(fx, 0.0), (double)(gr.W - 1)) : 0;
        const int cy = isfinite(fy) ? (int)fmin(fmax(fy, 0.0), (double)(gr.H - 1)) : 0;
        tx = cx / gr.T;
        ty = cy / gr.T;
    }
    return ty * gr.TX + tx;
}

__global__ void bin_count_kernel(const ScanRec* __restrict__ scan, uint32_t n, Grid gr, uint32_t* __restrict__ cnt,
                                 uint32_t* __restrict__ bin_of) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int t = center_tile(gr, scan[i].mu_x, scan[i].mu_y);
    bin_of[i] = (uint32_t)t;
    atomicAdd(cnt + t, 1u);
}

__global__ void bin_fill_kernel(uint32_t n, const uint32_t* __restrict__ bin_of, const uint32_t* __restrict__ off,
                                uint32_t* __restrict__ cur, uint32_t* __restrict__ bins) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = bin_of[i];
    bins[off[t] + atomicAdd(cur + t, 1u)] = i;
}

// One warp per tile: every lane keeps a register top-K of qmax_ub values over
// its share of the seeds; lanes' lists are merged through shared memory by
// kk rounds of a warp-wide min.  tau = the kk-th value popped.
template <int KCAP>
__global__ void __launch_bounds__(128) tau_kernel(const ScanRec* __restrict__ scan, Grid gr, int kk,
                                                  const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                                                  const uint32_t* __restrict__ bins,
                                                  unsigned long long* __restrict__ tau_bits) {
    __shared__ double lists[4][32][KCAP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x * 4 + warp;
    const int ntiles = gr.TX * gr.TY;
    if (tile >= ntiles) return;
    const int tx = tile % gr.TX, ty = tile / gr.TX;
    double x0, x1, y0, y1;
    box_of(gr, tx, tx, ty, ty, x0, x1, y0, y1);
    // smallest neighbourhood holding >= kk seeds (whole grid at worst)
    int r = 1;
    for (;; ++r) {
        const int ax = max(0, tx - r), bx = min(gr.TX - 1, tx + r), ay = max(0, ty - r), by = min(gr.TY - 1, ty + r);
        uint32_t c = 0;
        for (int yy = ay + lane; yy <= by; yy += 32)
            for (int xx = ax; xx <= bx; ++xx) c += cnt[yy * gr.TX + xx];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        const bool whole = ax == 0 && ay == 0 && bx == gr.TX - 1 && by == gr.TY - 1;
        if (c >= (uint32_t)kk || whole) break;
    }
    const int ax = max(0, tx - r), bx = min(gr.TX - 1, tx + r), ay = max(0, ty - r), by = min(gr.TY - 1, ty + r);
    // values only: (qmax, 0) keeps TopK's machinery; kk <= KCAP
    TopK<KCAP> t;
    t.init(kk);
    for (int yy = ay; yy <= by; ++yy)
        for (int xx = ax; xx <= bx; ++xx) {
            const int b = yy * gr.TX + xx;
            const uint32_t o = off[b], c = cnt[b];
            for (uint32_t j = lane; j < c; j += 32) {
                const G g = load_g(scan[bins[o + j]]);
                const double q = igs_cull::qmax_ub(g, x0, x1, y0, y1);
                if (q < t.tq()) t.insert(q, 0u);
            }
        }
    // merge: lane lists (ascending, live slots off..KCAP-1) -> smem
    double* mine = lists[warp][lane];
#pragma unroll
    for (int j = 0; j < KCAP; ++j)
        if (j >= t.off) mine[j - t.off] = t.q[j];
    __syncwarp();
    int head = 0;
    double last = 0.0;
    for (int round = 0; round < kk; ++round) {
        double v = head < kk ? mine[head] : __longlong_as_double(0x7ff0000000000000LL);
        int who = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int ow = __shfl_xor_sync(0xffffffffu, who, o);
            if (ov < v || (ov == v && ow < who)) {
                v = ov;
                who = ow;
            }
        }
        last = v;
        if (lane == who) ++head;
    }
    if (lane == 0) tau_bits[tile] = (unsigned long long)__double_as_longlong(last);
}

// Max-pyramid: level l node = max over its 2x2 children (non-negative
// doubles order like their bit patterns, +inf included).
__global__ void pyramid_kernel(Grid gr, int level, unsigned long long* __restrict__ tau_bits) {
    const int w = gr.lw[level], h = gr.lh[level];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w * h) return;
    const int x = i % w, y = i / w;
    const int cw = gr.lw[level - 1], ch = gr.lh[level - 1];
    const unsigned long long* child = tau_bits + gr.loff[level - 1];
    unsigned long long m = 0;
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            const int cx = 2 * x + dx, cy = 2 * y + dy;
            if (cx < cw && cy < ch) m = max(m, child[cy * cw + cx]);
        }
    tau_bits[gr.loff[level] + i] = m;
}

// Pyramid descent for one Gaussian; calls emit(tile) for every leaf that
// passes the certified test.
template <typename F>
__device__ __forceinline__ void descend(const Grid& gr, const G& g, const unsigned long long* __restrict__ tau_bits,
                                        F emit) {
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = (uint32_t)(gr.levels - 1) << 26;  // root (level top, 0, 0)
    while (sp > 0) {
        const uint32_t e = stack[--sp];
        const int l = e >> 26, x = (e >> 13) & 0x1fff, y = e & 0x1fff;
        const int span = 1 << l;
        const int tx0 = x * span, ty0 = y * span;
        const int tx1 = min(gr.TX, tx0 + span) - 1, ty1 = min(gr.TY, ty0 + span) - 1;
        double x0, x1, y0, y1;
        box_of(gr, tx0, tx1, ty0, ty1, x0, x1, y0, y1);
        const double lb = igs_cull::qmin_lb(g, x0, x1, y0, y1);
        const double tau = __longlong_as_double((long long)tau_bits[gr.loff[l] + y * gr.lw[l] + x]);
        if (l == 0) {
            if (lb <= tau) emit(y * gr.TX + x);
            continue;
        }
        if (lb * igs_cull::kPrune > tau) continue;
        const int cw = gr.lw[l - 1], ch = gr.lh[l - 1];
        for (int dy = 1; dy >= 0; --dy)
            for (int dx = 1; dx >= 0; --dx) {
                const int cx = 2 * x + dx, cy = 2 * y + dy;
                if (cx < cw && cy < ch && sp < 64) stack[sp++] = ((uint32_t)(l - 1) << 26) | ((uint32_t)cx << 13) | cy;
            }
    }
}

__global__ void emit_count_kernel(const ScanRec* __restrict__ scan, uint32_t n, Grid gr,
                                  const unsigned long long* __restrict__ tau_bits, uint32_t* __restrict__ tile_cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const G g = load_g(scan[i]);
    descend(gr, g, tau_bits, [&](int t) { atomicAdd(tile_cnt + t, 1u); });
}

__global__ void emit_fill_kernel(const ScanRec* __restrict__ scan, uint32_t n, Grid gr,
                                 const unsigned long long* __restrict__ tau_bits, const uint32_t* __restrict__ tile_off,
                                 uint32_t* __restrict__ tile_cur, uint32_t* __restrict__ list, uint32_t cap) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const G g = load_g(scan[i]);
    descend(gr, g, tau_bits, [&](int t) {
        const uint32_t pos = tile_off[t] + atomicAdd(tile_cur + t, 1u);
        if (pos < cap) list[pos] = i;
    });
}

__global__ void total_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt, int ntiles,
                             unsigned long long* __restrict__ total) {
    *total = (unsigned long long)off[ntiles - 1] + cnt[ntiles - 1];
}

// ---------------------------------------------------------------------------
// Consumers
// ---------------------------------------------------------------------------
constexpr int kChunk = 256;

// CTA per 16x16 tile, one pixel per thread; the tile's list is gathered into
// shared memory in chunks (records are 48 B, loaded as 3 x 16 B).  An
// overflowed list falls back to every candidate in index order.
template <int KCAP>
__global__ void __launch_bounds__(256) raster_culled_kernel(const ScanRec* __restrict__ scan,
                                                            const ShadeRec* __restrict__ shade, uint32_t n, Grid gr,
                                                            int row0, int row1, int kk,
                                                            const uint32_t* __restrict__ tile_off,
                                                            const uint32_t* __restrict__ tile_cnt,
                                                            const uint32_t* __restrict__ list, uint32_t cap,
                                                            float* __restrict__ out, uint32_t* __restrict__ topk,
                                                            unsigned long long* __restrict__ pairs) {
    __shared__ ScanRec sm[kChunk];
    __shared__ uint32_t sidx[kChunk];
    const int tid = threadIdx.y * kTilePx + threadIdx.x;
    const int tx = blockIdx.x, ty = row0 / kTilePx + blockIdx.y;
    const int px = tx * kTilePx + threadIdx.x;
    const int py = ty * kTilePx + threadIdx.y;
    const bool live = px < gr.W && py < row1 && py >= row0;
    const double x = center(px, gr.W), y = center(py, gr.H);
    const int tile = ty * gr.TX + tx;
    const uint32_t o = tile_off[tile], c = tile_cnt[tile];
    const bool overflow = (uint64_t)o + c > cap;
    const uint32_t total = overflow ? n : c;
    TopK<KCAP> t;
    t.init(kk);
    for (uint32_t base = 0; base < total; base += kChunk) {
        const uint32_t cnt = min((uint32_t)kChunk, total - base);
        __syncthreads();
        if ((uint32_t)tid < cnt) {
            const uint32_t gi = overflow ? base + tid : list[o + base + tid];
            const double2* src = reinterpret_cast<const double2*>(scan + gi);
            double2* dst = reinterpret_cast<double2*>(sm + tid);
            dst[0] = __ldg(src);
            dst[1] = __ldg(src + 1);
            dst[2] = __ldg(src + 2);
            sidx[tid] = gi;
        }
        __syncthreads();
        // every thread runs the loop (warp votes need the full warp); only live
        // threads write results
#pragma unroll 1
            for (uint32_t j = 0; j < cnt; ++j) {
                const double q = maha(sm[j], x, y);
                if (__any_sync(0xffffffffu, q <= t.tq()))
                    if (q <= t.tq()) t.offer(q, sidx[j]);
            }
    }
    if (pairs && tid == 0) atomicAdd(pairs, (unsigned long long)total * (min(gr.W - tx * kTilePx, kTilePx) *
                                                                         min(row1 - ty * kTilePx, kTilePx)));
    if (!live) return;
    double col[3];
    blend_topk(t, shade, col);
    const size_t op = ((size_t)(py - row0) * gr.W + px);
    out[op * 3 + 0] = clamp01f(col[0]);
    out[op * 3 + 1] = clamp01f(col[1]);
    out[op * 3 + 2] = clamp01f(col[2]);
    if (topk) store_topk(t, (double*)nullptr, topk + ((size_t)py * gr.W + px) * kk);
}

// Thread per query point (sampled pixel centre, or arbitrary point in
// points mode); candidates from the point's tile list via the read-only path.
template <int KCAP>
__global__ void __launch_bounds__(128) points_culled_kernel(const ScanRec* __restrict__ scan, uint32_t n, Grid gr,
                                                            const double* __restrict__ uv, uint32_t npts, int kk,
                                                            const uint32_t* __restrict__ tile_off,
                                                            const uint32_t* __restrict__ tile_cnt,
                                                            const uint32_t* __restrict__ list, uint32_t cap,
                                                            double* __restrict__ oq, uint32_t* __restrict__ oi,
                                                            unsigned long long* __restrict__ pairs) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    const double x = uv[2 * (size_t)p], y = uv[2 * (size_t)p + 1];
    int tx, ty;
    bool inside;
    if (gr.pts) {
        tx = (int)floor(x * (double)gr.TX);
        ty = (int)floor(y * (double)gr.TY);
        tx = min(max(tx, 0), gr.TX - 1);
        ty = min(max(ty, 0), gr.TY - 1);
    } else {
        // sampled pixel centres: recover the pixel, then its tile
        tx = min(max((int)floor(x * (double)gr.W), 0), gr.W - 1) / gr.T;
        ty = min(max((int)floor(y * (double)gr.H), 0), gr.H - 1) / gr.T;
    }
    double x0, x1, y0, y1;
    box_of(gr, tx, tx, ty, ty, x0, x1, y0, y1);
    inside = x >= x0 && x <= x1 && y >= y0 && y <= y1;  // else: no certificate -> scan all
    const int tile = ty * gr.TX + tx;
    const uint32_t o = tile_off[tile], c = tile_cnt[tile];
    const bool all = !inside || (uint64_t)o + c > cap;
    const uint32_t total = all ? n : c;
    TopK<KCAP> t;
    t.init(kk);
#pragma unroll 1
    for (uint32_t j = 0; j < total; ++j) {
        const uint32_t gi = all ? j : __ldg(list + o + j);
        const ScanRec r = scan[gi];
        const double q = maha(r, x, y);
        if (q <= t.tq()) t.offer(q, gi);
    }
    if (pairs) atomicAdd(pairs, (unsigned long long)total);
    store_topk(t, oq + (size_t)p * kk, oi + (size_t)p * kk);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct CullBufs {
    DevBuf bin_cnt, bin_off, bin_of, bins, tau, tile_cnt, tile_off, list, cub_tmp, total;
    uint32_t cap = 0;
    unsigned long long* total_pinned = nullptr;  // last build's pair count (read lazily)
    // cache key
    uint64_t version = ~0ull;
    int W = -1, H = -1, pts = -1, kk = -1;
    Grid grid;
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

CullBufs& bufs(igs_ctx* ctx) {
    if (!ctx->cull) ctx->cull = new CullBufs();
    return *static_cast<CullBufs*>(ctx->cull);
}

Grid make_grid(int W, int H, int pts_cells) {
    Grid g{};
    if (pts_cells > 0) {
        g.pts = 1;
        g.W = g.H = 0;
        g.T = 1;
        g.TX = g.TY = pts_cells;
    } else {
        g.pts = 0;
        g.W = W;
        g.H = H;
        g.T = kTilePx;
        g.TX = (W + kTilePx - 1) / kTilePx;
        g.TY = (H + kTilePx - 1) / kTilePx;
    }
    int l = 0, w = g.TX, h = g.TY, off = 0;
    for (;;) {
        g.lw[l] = w;
        g.lh[l] = h;
        g.loff[l] = off;
        off += w * h;
        ++l;
        if (w == 1 && h == 1) break;
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    g.levels = l;
    return g;
}

template <int KCAP>
int launch_tau(igs_ctx* ctx, const Grid& gr, int kk, CullBufs& b) {
    const int ntiles = gr.TX * gr.TY;
    tau_kernel<KCAP><<<(ntiles + 3) / 4, 128, 0, ctx->stream>>>(ctx->scan, gr, kk, (const uint32_t*)b.bin_cnt.p,
                                                                 (const uint32_t*)b.bin_off.p, (const uint32_t*)b.bins.p,
                                                                 (unsigned long long*)b.tau.p);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

// Builds (or reuses) the tile lists for grid (W, H) or points cells.
int build_lists(igs_ctx* ctx, int W, int H, int pts_cells, int kk) {
    CullBufs& b = bufs(ctx);
    if (b.version == ctx->params_version && b.W == W && b.H == H && b.pts == pts_cells && b.kk == kk) return IGS_OK;
    const uint32_t n = ctx->n;
    const Grid gr = make_grid(W, H, pts_cells);
    const int ntiles = gr.TX * gr.TY;
    const int pyr = gr.loff[gr.levels - 1] + 1;
    if (gr.levels > kMaxLevels || gr.TX > 8191 || gr.TY > 8191)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "raster too large for the tile pyramid");
    if (b.cap == 0) b.cap = std::max<uint32_t>(1u << 21, n * 48u);
    // Grow from the previous build's total (copied to pinned memory at the
    // end of that build; the stream has synchronised since in every caller).
    // Tiles that overflowed were still exact (consumers fall back to all N).
    if (b.total_pinned && *b.total_pinned > b.cap) b.cap = (uint32_t)std::min<unsigned long long>(
        0xF0000000ull, *b.total_pinned + *b.total_pinned / 2);
    if (!grow(b.bin_cnt, (size_t)ntiles * 4) || !grow(b.bin_off, (size_t)ntiles * 4) || !grow(b.bin_of, (size_t)n * 4) ||
        !grow(b.bins, (size_t)n * 4) || !grow(b.tau, (size_t)pyr * 8) || !grow(b.tile_cnt, (size_t)ntiles * 8) ||
        !grow(b.tile_off, (size_t)ntiles * 4) || !grow(b.list, (size_t)b.cap * 4) || !grow(b.total, 16))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (tile lists)");
    if (!b.total_pinned) {
        if (cudaMallocHost(&b.total_pinned, 8) != cudaSuccess) return igs_fail(ctx, IGS_E_CUDA, "pinned alloc");
        *b.total_pinned = 0;
    }
    uint32_t* bin_cnt = (uint32_t*)b.bin_cnt.p;
    uint32_t* bin_off = (uint32_t*)b.bin_off.p;
    uint32_t* tile_cnt = (uint32_t*)b.tile_cnt.p;           // [0, ntiles): counts
    uint32_t* tile_cur = tile_cnt + ntiles;                  // [ntiles, 2 ntiles): cursors
    uint32_t* tile_off = (uint32_t*)b.tile_off.p;
    igs_prof_begin(ctx, IGS_PROF_CULL);
    // 1. centre bins
    IGS_CUDA(ctx, cudaMemsetAsync(bin_cnt, 0, (size_t)ntiles * 4, ctx->stream));
    bin_count_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(ctx->scan, n, gr, bin_cnt, (uint32_t*)b.bin_of.p);
    IGS_LAUNCHED(ctx);
    int e;
    if ((e = igs_scan_excl_u32(ctx, bin_cnt, bin_off, (size_t)ntiles))) return e;
    IGS_CUDA(ctx, cudaMemsetAsync(tile_cnt, 0, (size_t)ntiles * 8, ctx->stream));  // reuse as bin cursors
    bin_fill_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(n, (const uint32_t*)b.bin_of.p, bin_off, tile_cnt,
                                                              (uint32_t*)b.bins.p);
    IGS_LAUNCHED(ctx);
    // 2. tau per tile
    if (kk <= 4) e = launch_tau<4>(ctx, gr, kk, b);
    else if (kk <= 8) e = launch_tau<8>(ctx, gr, kk, b);
    else if (kk <= 16) e = launch_tau<16>(ctx, gr, kk, b);
    else e = launch_tau<32>(ctx, gr, kk, b);
    if (e) return e;
    // 3. pyramid
    for (int l = 1; l < gr.levels; ++l) {
        const int cnt = gr.lw[l] * gr.lh[l];
        pyramid_kernel<<<(cnt + 255) / 256, 256, 0, ctx->stream>>>(gr, l, (unsigned long long*)b.tau.p);
        IGS_LAUNCHED(ctx);
    }
    // 4. emit: count, scan, fill
    IGS_CUDA(ctx, cudaMemsetAsync(tile_cnt, 0, (size_t)ntiles * 8, ctx->stream));
    emit_count_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, n, gr, (const unsigned long long*)b.tau.p,
                                                                tile_cnt);
    IGS_LAUNCHED(ctx);
    if ((e = igs_scan_excl_u32(ctx, tile_cnt, tile_off, (size_t)ntiles))) return e;
    emit_fill_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, n, gr, (const unsigned long long*)b.tau.p,
                                                               tile_off, tile_cur, (uint32_t*)b.list.p, b.cap);
    IGS_LAUNCHED(ctx);
    // total pairs = off[last] + cnt[last] -> pinned host word, read at the next build
    total_kernel<<<1, 1, 0, ctx->stream>>>(tile_off, tile_cnt, ntiles, (unsigned long long*)b.total.p);
    IGS_LAUNCHED(ctx);
    IGS_CUDA(ctx, cudaMemcpyAsync(b.total_pinned, b.total.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    igs_prof_end(ctx, IGS_PROF_CULL, 0.0);
    b.version = ctx->params_version;
    b.W = W;
    b.H = H;
    b.pts = pts_cells;
    b.kk = kk;
    b.grid = gr;
    return IGS_OK;
}

// host read of the last build's total pairs (syncs)
uint64_t last_total(igs_ctx* ctx) {
    CullBufs& b = bufs(ctx);
    cudaStreamSynchronize(ctx->stream);
    return *b.total_pinned;
}

template <int KCAP>
int launch_raster_culled(igs_ctx* ctx, int W, int H, int row0, int row1, int kk, float* out, uint32_t* topk) {
    CullBufs& b = bufs(ctx);
    const Grid& gr = b.grid;
    const int tr0 = row0 / kTilePx, tr1 = (row1 + kTilePx - 1) / kTilePx;
    dim3 grid(gr.TX, tr1 - tr0);
    const int ntiles = gr.TX * gr.TY;
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    raster_culled_kernel<KCAP><<<grid, dim3(kTilePx, kTilePx), 0, ctx->stream>>>(
        ctx->scan, ctx->shade, ctx->n, gr, row0, row1, kk, (const uint32_t*)b.tile_off.p,
        (const uint32_t*)b.tile_cnt.p, (const uint32_t*)b.list.p, b.cap, out, topk,
        igs_prof_counter(ctx, IGS_PROF_SCAN));
    IGS_LAUNCHED(ctx);
    (void)ntiles;
    (void)W;
    (void)H;
    igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
    return IGS_OK;
}

template <int KCAP>
int launch_points_culled(igs_ctx* ctx, const double* uv, uint32_t npts, int kk, uint32_t* oi, double* oq) {
    CullBufs& b = bufs(ctx);
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    points_culled_kernel<KCAP><<<(npts + 127) / 128, 128, 0, ctx->stream>>>(
        ctx->scan, ctx->n, b.grid, uv, npts, kk, (const uint32_t*)b.tile_off.p, (const uint32_t*)b.tile_cnt.p,
        (const uint32_t*)b.list.p, b.cap, oq, oi, igs_prof_counter(ctx, IGS_PROF_SCAN));
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
    return IGS_OK;
}

}  // namespace

void igs_cull_free(igs_ctx* ctx) {
    if (!ctx->cull) return;
    CullBufs* b = static_cast<CullBufs*>(ctx->cull);
    for (DevBuf* d : {&b->bin_cnt, &b->bin_off, &b->bin_of, &b->bins, &b->tau, &b->tile_cnt, &b->tile_off, &b->list,
                      &b->cub_tmp, &b->total})
        cudaFree(d->p);
    if (b->total_pinned) cudaFreeHost(b->total_pinned);
    delete b;
    ctx->cull = nullptr;
}

int igs_raster_culled(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out, uint32_t* topk) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32) return igs_raster_global(ctx, W, H, k, row0, row1, out, topk);
    int e = build_lists(ctx, W, H, 0, kk);
    if (e) return e;
    if (kk <= 4) return launch_raster_culled<4>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 8) return launch_raster_culled<8>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 16) return launch_raster_culled<16>(ctx, W, H, row0, row1, kk, out, topk);
    return launch_raster_culled<32>(ctx, W, H, row0, row1, kk, out, topk);
}

// Culled top-K at device points.  Train samples (pixel centres of the target)
// use the target's pixel tiles; arbitrary points use a cells grid.
int igs_topk_culled_grid(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq, int W,
                         int H) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32 || npts == 0) return igs_topk_points(ctx, uv, npts, k, oi, oq);
    int cells = 0;
    if (W <= 0) {
        // ~2 Gaussians per cell on average, 16..1024 cells per side
        cells = 16;
        while (cells < 1024 && (uint64_t)cells * cells * 2 < ctx->n) cells *= 2;
    }
    int e = build_lists(ctx, W, H, cells, kk);
    if (e) return e;
    if (kk <= 4) return launch_points_culled<4>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 8) return launch_points_culled<8>(ctx, uv, npts, kk, oi, oq);
    if (kk <= 16) return launch_points_culled<16>(ctx, uv, npts, kk, oi, oq);
    return launch_points_culled<32>(ctx, uv, npts, kk, oi, oq);
}

int igs_topk_samples_culled(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq) {
    return igs_topk_culled_grid(ctx, uv, npts, k, oi, oq, 0, 0);
}

// Sampled pixel centres of a W x H target: the target's pixel tiles.
int igs_topk_pixels_culled(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq, int W,
                           int H) {
    return igs_topk_culled_grid(ctx, uv, npts, k, oi, oq, W, H);
}

// Debug/parity: CSR of the lists for a W x H raster, members sorted ascending.
int igs_cull_lists(igs_ctx* ctx, int W, int H, int k, uint32_t* ntiles_out, uint64_t* total_out, uint32_t* offsets,
                   uint32_t* members, double* tau) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "tile lists need k <= 32");
    int e = build_lists(ctx, W, H, 0, kk);
    if (e) return e;
    CullBufs& b = bufs(ctx);
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const uint64_t total = last_total(ctx);
    const int ntiles = b.grid.TX * b.grid.TY;
    if (ntiles_out) *ntiles_out = (uint32_t)ntiles;
    if (total_out) *total_out = total;
    if (!offsets && !members && !tau) return IGS_OK;
    if (total > b.cap) {  // rebuild with room, then report
        b.version = ~0ull;
        if ((e = build_lists(ctx, W, H, 0, kk))) return e;
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    std::vector<uint32_t> off(ntiles), cnt(ntiles), list(total);
    std::vector<unsigned long long> tb(ntiles);
    IGS_CUDA(ctx, cudaMemcpy(off.data(), b.tile_off.p, (size_t)ntiles * 4, cudaMemcpyDeviceToHost));
    IGS_CUDA(ctx, cudaMemcpy(cnt.data(), b.tile_cnt.p, (size_t)ntiles * 4, cudaMemcpyDeviceToHost));
    if (total) IGS_CUDA(ctx, cudaMemcpy(list.data(), b.list.p, (size_t)total * 4, cudaMemcpyDeviceToHost));
    IGS_CUDA(ctx, cudaMemcpy(tb.data(), b.tau.p, (size_t)ntiles * 8, cudaMemcpyDeviceToHost));
    for (int t = 0; t < ntiles; ++t) {
        if (offsets) offsets[t] = off[t];
        std::sort(list.begin() + off[t], list.begin() + off[t] + cnt[t]);
        if (tau) std::memcpy(&tau[t], &tb[t], 8);
    }
    if (offsets) offsets[ntiles] = (uint32_t)total;
    if (members && total) std::memcpy(members, list.data(), (size_t)total * 4);
    return IGS_OK;
}
