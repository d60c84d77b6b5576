// bsp.cu -- BSP acceleration (bsp.hpp:70-106): partition build/rebuild,
// kernel 2 in its BSP form (shell binning), locate_block, and kernel 3 over
// shell lists (render_image_blocked, render_topk_blocked).
//
// Reference: bsp.cpp:14-23 shell_of, :27-118 Builder::build, :132-176
// build_partition / collect_shell_members, :178-218 grid locator +
// rebuild_partition, :220-264 locate_block, :268-341 blocked renders.
//
// The split tree is built on the host (a deterministic restatement of the
// recursive alternating-axis median; it needs only the centres, downloaded
// once).  Everything per-pixel or per-(shell, Gaussian) runs on the device:
//   * shell binning: shell_members[b] = {i : mu_i in shell_b (closed)}, in
//     ascending i -- a CTA per shell scans the centres in index order with a
//     block-wide ordered compaction (count pass, exclusive scan, fill pass).
//     This is exactly the set collect_shell_members gathers through the tree
//     (its bbox pruning only skips non-members), and exactly the rectangle
//     test rebuild_partition runs (bsp.cpp:214-216).
//   * locate: the tree descent (c < line ? low : high) or, for partitions
//     rebuilt from corners, the grid locator with its first-containing /
//     nearest-Chebyshev / scan-all fallbacks, op for op.
//   * blocked raster: CTA per 16x16 tile; the tile's pixels usually fall in
//     one or two blocks -- the CTA loops over the distinct blocks present,
//     staging each shell list through shared memory for the pixels of that
//     block (scan order is index order, as the reference's member lists).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "igs_internal.cuh"

using namespace igs_dev;

struct RectD {
    double x1, y1, x2, y2;
};

struct NodeD {
    int axis;
    double line;
    int32_t low, high, block;
};

struct PartitionDev {
    uint32_t nb = 0, source_size = 0;
    int n_max = 0;
    bool tree = false;
    std::vector<RectD> blocks, shells;
    std::vector<NodeD> nodes;
    int32_t root = -1;
    int grid_dim = 0;
    uint64_t shell_total = 0;
    // device
    RectD* d_blocks = nullptr;
    RectD* d_shells = nullptr;
    NodeD* d_nodes = nullptr;
    uint32_t* d_grid_off = nullptr;  // grid_dim^2 + 1
    uint32_t* d_grid_blk = nullptr;
    uint32_t* d_shell_off = nullptr;  // nb + 1
    uint32_t* d_shell_mem = nullptr;
};

namespace {

// bsp.cpp:14-23
RectD shell_of(const RectD& b) {
    const double ex = (b.x2 - b.x1) * 0.25;
    const double ey = (b.y2 - b.y1) * 0.25;
    RectD s{b.x1 - ex, b.y1 - ey, b.x2 + ex, b.y2 + ey};
    s.x1 = std::max(s.x1, 0.0);
    s.y1 = std::max(s.y1, 0.0);
    s.x2 = std::min(s.x2, 1.0);
    s.y2 = std::min(s.y2, 1.0);
    return s;
}

// bsp.cpp:27-118: recursive alternating-axis median split; leaves numbered
// in DFS (low-first) order; the tie-aware split position keeps coincident
// coordinates on one side.
struct Builder {
    const std::vector<double>& mx;
    const std::vector<double>& my;
    int n_max;
    PartitionDev& out;

    int32_t build(RectD rect, std::vector<uint32_t> m, int depth) {
        const int32_t id = (int32_t)out.nodes.size();
        out.nodes.push_back(NodeD{0, 0.0, -1, -1, -1});
        if ((long long)m.size() <= (long long)n_max) {
            out.nodes[id].block = (int32_t)out.blocks.size();
            out.blocks.push_back(rect);
            return id;
        }
        const int axis = depth % 2;
        const std::vector<double>& c = axis == 0 ? mx : my;
        std::sort(m.begin(), m.end(), [&](uint32_t a, uint32_t b) { return c[a] < c[b] || (c[a] == c[b] && a < b); });
        const size_t n = m.size(), half = n / 2;
        size_t pos = 0;
        double line = 0.0;
        bool forced = false;
        if (c[m[half - 1]] < c[m[half]]) {
            pos = half;
        } else {
            size_t lo = 0, hi = 0;
            bool has_lo = false, has_hi = false;
            for (size_t j = half; j-- > 1;)
                if (c[m[j - 1]] < c[m[j]]) {
                    lo = j;
                    has_lo = true;
                    break;
                }
            for (size_t j = half + 1; j < n; ++j)
                if (c[m[j - 1]] < c[m[j]]) {
                    hi = j;
                    has_hi = true;
                    break;
                }
            if (has_lo && (!has_hi || half - lo <= hi - half)) pos = lo;
            else if (has_hi) pos = hi;
            else forced = true;
        }
        if (forced) {
            pos = half;
            line = c[m[0]];
        } else {
            const double lo_c = c[m[pos - 1]], hi_c = c[m[pos]];
            line = 0.5 * (lo_c + hi_c);
            if (!(line > lo_c)) line = hi_c;
        }
        std::vector<uint32_t> lower(m.begin(), m.begin() + pos), upper(m.begin() + pos, m.end());
        m.clear();
        m.shrink_to_fit();
        RectD lr = rect, hr = rect;
        if (axis == 0) {
            lr.x2 = line;
            hr.x1 = line;
        } else {
            lr.y2 = line;
            hr.y1 = line;
        }
        out.nodes[id].axis = axis;
        out.nodes[id].line = line;
        const int32_t l = build(lr, std::move(lower), depth + 1);
        out.nodes[id].low = l;
        const int32_t h = build(hr, std::move(upper), depth + 1);
        out.nodes[id].high = h;
        return id;
    }
};

// --- device helpers ----------------------------------------------------------
__device__ __forceinline__ bool contains_closed(const RectD& r, double x, double y) {
    return x >= r.x1 && x <= r.x2 && y >= r.y1 && y <= r.y2;
}
__device__ __forceinline__ bool contains_half_open(const RectD& r, double x, double y) {
    const bool ix = x >= r.x1 && (x < r.x2 || (r.x2 >= 1.0 && x <= r.x2));
    const bool iy = y >= r.y1 && (y < r.y2 || (r.y2 >= 1.0 && y <= r.y2));
    return ix && iy;
}
__device__ __forceinline__ double cheb(const RectD& r, double x, double y) {
    const double dx = fmax(fmax(r.x1 - x, x - r.x2), 0.0);
    const double dy = fmax(fmax(r.y1 - y, y - r.y2), 0.0);
    return fmax(dx, dy);
}

struct LocView {
    int tree;
    const NodeD* nodes;
    int32_t root;
    int grid_dim;
    const uint32_t* grid_off;
    const uint32_t* grid_blk;
    const RectD* blocks;
    uint32_t nb;
};

// bsp.cpp:220-264 locate_block
__device__ int locate(const LocView& v, double x, double y) {
    if (v.tree) {
        int32_t id = v.root;
        while (v.nodes[id].block < 0) {
            const NodeD nd = v.nodes[id];
            const double c = nd.axis == 0 ? x : y;
            id = c < nd.line ? nd.low : nd.high;
        }
        return v.nodes[id].block;
    }
    const int gd = v.grid_dim;
    int cx = (int)(x * gd), cy = (int)(y * gd);  // C++ truncation, then clamp
    cx = cx < 0 ? 0 : (cx > gd - 1 ? gd - 1 : cx);
    cy = cy < 0 ? 0 : (cy > gd - 1 ? gd - 1 : cy);
    const uint32_t c = (uint32_t)(cy * gd + cx);
    int best = -1;
    double best_d = __longlong_as_double(0x7ff0000000000000LL);
    for (uint32_t j = v.grid_off[c]; j < v.grid_off[c + 1]; ++j) {
        const uint32_t b = v.grid_blk[j];
        const RectD r = v.blocks[b];
        if (contains_half_open(r, x, y)) return (int)b;
        const double d = cheb(r, x, y);
        if (d < best_d) {
            best_d = d;
            best = (int)b;
        }
    }
    if (best >= 0) return best;
    for (uint32_t b = 0; b < v.nb; ++b) {
        const RectD r = v.blocks[b];
        if (contains_half_open(r, x, y)) return (int)b;
        const double d = cheb(r, x, y);
        if (d < best_d) {
            best_d = d;
            best = (int)b;
        }
    }
    return best;
}

// Shell binning, CTA per shell: Gaussians in index order, block-wide ordered
// compaction.  pass 0 counts, pass 1 writes at shell_off[b].
__global__ void __launch_bounds__(256) shell_bin_kernel(const ScanRec* __restrict__ scan, uint32_t n,
                                                        const RectD* __restrict__ shells, int pass,
                                                        uint32_t* __restrict__ counts,
                                                        const uint32_t* __restrict__ off, uint32_t* __restrict__ mem) {
    __shared__ uint32_t warp_tot[8];
    const uint32_t b = blockIdx.x;
    const RectD s = shells[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t written = 0;
    for (uint32_t base = 0; base < n; base += 256) {
        const uint32_t i = base + threadIdx.x;
        const bool in = i < n && contains_closed(s, scan[i].mu_x, scan[i].mu_y);
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (lane == 0) warp_tot[warp] = __popc(m);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < warp) before += warp_tot[w];
            total += warp_tot[w];
        }
        if (pass == 1 && in) mem[off[b] + written + before + __popc(m & ((1u << lane) - 1))] = i;
        written += total;
        __syncthreads();
    }
    if (pass == 0 && threadIdx.x == 0) counts[b] = written;
}

__global__ void locate_kernel(LocView v, const double* __restrict__ uv, uint32_t npts, int32_t* __restrict__ out) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    out[p] = locate(v, uv[2 * (size_t)p], uv[2 * (size_t)p + 1]);
}

constexpr int kTile = 16;
constexpr int kChunk = 256;

// Blocked raster (bsp.cpp:268-317), one pixel per thread.
template <int KCAP>
__global__ void __launch_bounds__(256) blocked_raster_kernel(const ScanRec* __restrict__ scan,
                                                             const ShadeRec* __restrict__ shade, LocView v,
                                                             const uint32_t* __restrict__ shell_off,
                                                             const uint32_t* __restrict__ shell_mem, int W, int H,
                                                             int row0, int row1, int kk, float* __restrict__ out,
                                                             unsigned long long* __restrict__ pairs) {
    __shared__ ScanRec sm[kChunk];
    __shared__ uint32_t sidx[kChunk];
    __shared__ int cur_block;
    const int tid = threadIdx.y * kTile + threadIdx.x;
    // rows [row0, row1) of the W x H raster, written at their place in `out`
    const int px = blockIdx.x * kTile + threadIdx.x, py = row0 + blockIdx.y * kTile + threadIdx.y;
    const bool live = px < W && py < row1;
    const double x = center(px, W), y = center(py, H);
    const int myb = live ? locate(v, x, y) : 0x7fffffff;
    bool done = !live;
    unsigned long long evaluated = 0;
    for (;;) {
        if (tid == 0) cur_block = 0x7fffffff;
        __syncthreads();
        if (!done) atomicMin(&cur_block, myb);
        __syncthreads();
        const int b = cur_block;
        if (b == 0x7fffffff) break;
        const bool mine = !done && myb == b;
        TopK<KCAP> t;
        t.init(kk);
        const uint32_t o = shell_off[b], m = shell_off[b + 1] - o;
        for (uint32_t base = 0; base < m; base += kChunk) {
            const uint32_t cnt = min((uint32_t)kChunk, m - base);
            __syncthreads();
            if ((uint32_t)tid < cnt) {
                const uint32_t gi = shell_mem[o + base + tid];
                const double2* src = reinterpret_cast<const double2*>(scan + gi);
                double2* dst = reinterpret_cast<double2*>(sm + tid);
                dst[0] = __ldg(src);
                dst[1] = __ldg(src + 1);
                dst[2] = __ldg(src + 2);
                sidx[tid] = gi;
            }
            __syncthreads();
            if (__syncthreads_or(mine)) {
                for (uint32_t j = 0; j < cnt; ++j) {
                    const double q = maha(sm[j], x, y);
                    if (__any_sync(0xffffffffu, mine && q <= t.tq()))
                        if (mine && q <= t.tq()) t.offer(q, sidx[j]);
                }
            }
        }
        if (mine) {
            evaluated += m;
            double col[3];
            blend_topk(t, shade, col);  // empty shell: total 0 -> colour 0 (bsp.cpp:274-275)
            const size_t op = (size_t)py * W + px;
            out[op * 3 + 0] = clamp01f(col[0]);
            out[op * 3 + 1] = clamp01f(col[1]);
            out[op * 3 + 2] = clamp01f(col[2]);
            done = true;
        }
        __syncthreads();
    }
    if (pairs && evaluated) atomicAdd(pairs, evaluated);
}

// render_topk_blocked at points (bsp.cpp:321-332), thread per point (shell
// lists are short); unclamped double colour.
template <int KCAP>
__global__ void blocked_points_kernel(const ScanRec* __restrict__ scan, const ShadeRec* __restrict__ shade,
                                      LocView v, const uint32_t* __restrict__ shell_off,
                                      const uint32_t* __restrict__ shell_mem, const double* __restrict__ uv,
                                      uint32_t npts, int kk, double* __restrict__ rgb) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    const double x = uv[2 * (size_t)p], y = uv[2 * (size_t)p + 1];
    const int b = locate(v, x, y);
    TopK<KCAP> t;
    t.init(kk);
    for (uint32_t j = shell_off[b]; j < shell_off[b + 1]; ++j) {
        const uint32_t gi = shell_mem[j];
        const double q = maha(scan[gi], x, y);
        if (q <= t.tq()) t.offer(q, gi);
    }
    double col[3];
    blend_topk(t, shade, col);
    rgb[3 * (size_t)p] = col[0];
    rgb[3 * (size_t)p + 1] = col[1];
    rgb[3 * (size_t)p + 2] = col[2];
}

template <typename T>
T* to_dev(igs_ctx* ctx, const std::vector<T>& v) {
    T* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (!v.empty()) cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream);
    return d;
}

void free_dev(PartitionDev* p) {
    cudaFree(p->d_blocks);
    cudaFree(p->d_shells);
    cudaFree(p->d_nodes);
    cudaFree(p->d_grid_off);
    cudaFree(p->d_grid_blk);
    cudaFree(p->d_shell_off);
    cudaFree(p->d_shell_mem);
}

LocView view_of(const PartitionDev* p) {
    LocView v;
    v.tree = p->tree ? 1 : 0;
    v.nodes = p->d_nodes;
    v.root = p->root;
    v.grid_dim = p->grid_dim;
    v.grid_off = p->d_grid_off;
    v.grid_blk = p->d_grid_blk;
    v.blocks = p->d_blocks;
    v.nb = p->nb;
    return v;
}

// Shells on device, then the two-pass ordered binning.
int finish_partition(igs_ctx* ctx, PartitionDev* p) {
    p->nb = (uint32_t)p->blocks.size();
    p->shells.resize(p->nb);
    for (uint32_t b = 0; b < p->nb; ++b) p->shells[b] = shell_of(p->blocks[b]);
    p->d_blocks = to_dev(ctx, p->blocks);
    p->d_shells = to_dev(ctx, p->shells);
    p->d_nodes = to_dev(ctx, p->nodes);
    if (!p->d_blocks || !p->d_shells || !p->d_nodes) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
    if (!p->tree) {
        // bsp.cpp:178-195 build_grid_locator
        const int nb = (int)p->nb;
        int gd = std::max(1, (int)std::ceil(std::sqrt((double)nb)));
        p->grid_dim = gd;
        std::vector<std::vector<uint32_t>> cells((size_t)gd * gd);
        auto range = [&](double lo, double hi, int& c0, int& c1) {
            c0 = std::clamp((int)std::floor(lo * gd), 0, gd - 1);
            c1 = std::clamp((int)std::ceil(hi * gd) - 1, 0, gd - 1);
            if (c1 < c0) c1 = c0;
        };
        for (int b = 0; b < nb; ++b) {
            int x0, x1, y0, y1;
            range(p->blocks[b].x1, p->blocks[b].x2, x0, x1);
            range(p->blocks[b].y1, p->blocks[b].y2, y0, y1);
            for (int cy = y0; cy <= y1; ++cy)
                for (int cx = x0; cx <= x1; ++cx) cells[(size_t)cy * gd + cx].push_back((uint32_t)b);
        }
        std::vector<uint32_t> off(cells.size() + 1), blk;
        for (size_t c = 0; c < cells.size(); ++c) {
            off[c] = (uint32_t)blk.size();
            blk.insert(blk.end(), cells[c].begin(), cells[c].end());
        }
        off[cells.size()] = (uint32_t)blk.size();
        p->d_grid_off = to_dev(ctx, off);
        p->d_grid_blk = to_dev(ctx, blk);
        if (!p->d_grid_off || !p->d_grid_blk) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
    }
    uint32_t* counts = (uint32_t*)igs_scratch(ctx, 25, (size_t)(p->nb + 1) * 4);
    if (cudaMalloc(&p->d_shell_off, (size_t)(p->nb + 1) * 4) != cudaSuccess || !counts)
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
    igs_prof_begin(ctx, IGS_PROF_BLOCKED);
    IGS_CUDA(ctx, cudaMemsetAsync(counts, 0, (size_t)(p->nb + 1) * 4, ctx->stream));
    shell_bin_kernel<<<p->nb, 256, 0, ctx->stream>>>(ctx->scan, ctx->n, p->d_shells, 0, counts, nullptr, nullptr);
    IGS_LAUNCHED(ctx);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, p->d_shell_off, (int)p->nb + 1, ctx->stream);
    void* temp = igs_scratch(ctx, 26, tb);
    if (!temp) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
    IGS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(temp, tb, counts, p->d_shell_off, (int)p->nb + 1, ctx->stream));
    ctx->launches += 2;
    uint32_t total = 0;
    IGS_CUDA(ctx, cudaMemcpyAsync(&total, p->d_shell_off + p->nb, 4, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    p->shell_total = total;
    if (cudaMalloc(&p->d_shell_mem, std::max<size_t>(total, 1) * 4) != cudaSuccess)
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp shells)");
    shell_bin_kernel<<<p->nb, 256, 0, ctx->stream>>>(ctx->scan, ctx->n, p->d_shells, 1, nullptr, p->d_shell_off,
                                                     p->d_shell_mem);
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_BLOCKED, (double)ctx->n * p->nb);
    return IGS_OK;
}

int check_partition(igs_ctx* ctx) {
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition (igs_partition_build / rebuild)");
    if (ctx->part->nb == 0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "partition has no blocks");
    if (ctx->part->source_size != ctx->n)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "stale partition: Gaussian count changed since construction");
    return IGS_OK;
}

// --- device tree build (bsp.cpp:27-118 on the GPU) --------------------------
// Level-synchronous restatement of Builder::build.  Once: every point's key
// along x and along y, radix-sorted with the index as the stable tie-break
// -- the (coord, idx) order the reference's comparator defines.  Per level:
// a stable radix sort of that global order by the point's current node
// yields every active node's members in (coord, idx) order as one
// contiguous segment; one thread per node applies the tie-aware split rule
// (pos, line); points move to their child.  The host (a few thousand nodes)
// turns the level records into the reference's DFS numbering of nodes and
// blocks and the block rectangles.
__device__ __forceinline__ unsigned long long coord_key(double v) {
    if (v == 0.0) v = 0.0;  // -0 and +0 compare equal in the reference
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__global__ void gb_keys_kernel(const ScanRec* __restrict__ scan, uint32_t n, unsigned long long* __restrict__ kx,
                               unsigned long long* __restrict__ ky, uint32_t* __restrict__ iota,
                               uint32_t* __restrict__ node_of) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    kx[i] = coord_key(scan[i].mu_x);
    ky[i] = coord_key(scan[i].mu_y);
    iota[i] = i;
    node_of[i] = 0;
}

// node key of the j-th point in the global (coord, idx) order
__global__ void gb_gather_kernel(const uint32_t* __restrict__ ord, const uint32_t* __restrict__ node_of, uint32_t n,
                                 uint32_t* __restrict__ key) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) key[j] = node_of[ord[j]];
}

__device__ __forceinline__ double coord_of(const ScanRec* __restrict__ scan, uint32_t i, int axis) {
    return axis == 0 ? scan[i].mu_x : scan[i].mu_y;
}

// bsp.cpp:54-95 for active node k: members seg[start[k] .. start[k]+size[k])
__global__ void gb_split_kernel(const ScanRec* __restrict__ scan, const uint32_t* __restrict__ seg,
                                const uint32_t* __restrict__ start, const uint32_t* __restrict__ size, uint32_t na,
                                int axis, uint32_t* __restrict__ pos_out, double* __restrict__ line_out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= na) return;
    const uint32_t* m = seg + start[k];
    const size_t n = size[k], half = n / 2;
    auto c = [&](size_t j) { return coord_of(scan, m[j], axis); };
    size_t pos = 0;
    double line = 0.0;
    bool forced = false;
    if (c(half - 1) < c(half)) {
        pos = half;
    } else {
        size_t lo = 0, hi = 0;
        bool has_lo = false, has_hi = false;
        for (size_t j = half; j-- > 1;)
            if (c(j - 1) < c(j)) {
                lo = j;
                has_lo = true;
                break;
            }
        for (size_t j = half + 1; j < n; ++j)
            if (c(j - 1) < c(j)) {
                hi = j;
                has_hi = true;
                break;
            }
        if (has_lo && (!has_hi || half - lo <= hi - half)) pos = lo;
        else if (has_hi) pos = hi;
        else forced = true;
    }
    if (forced) {
        pos = half;
        line = c(0);
    } else {
        const double lo_c = c(pos - 1), hi_c = c(pos);
        line = __dmul_rn(0.5, __dadd_rn(lo_c, hi_c));
        if (!(line > lo_c)) line = hi_c;
    }
    pos_out[k] = (uint32_t)pos;
    line_out[k] = line;
}

// Moves the points of active nodes to their children (next-level active
// rank, or `inactive` once the child is a leaf).
__global__ void gb_move_kernel(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ seg_node, uint32_t cnt,
                               const uint32_t* __restrict__ start, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ child, uint32_t* __restrict__ node_of) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cnt) return;
    const uint32_t k = seg_node[j];
    node_of[seg[j]] = child[2 * k + (j - start[k] < pos[k] ? 0 : 1)];
}

struct GbLevelNode {
    uint32_t size;
    bool leaf;
    uint32_t pos = 0;
    double line = 0.0;
    uint32_t low = 0, high = 0;  // indices into the next level
    RectD rect;
};

// Builds p->nodes / p->blocks / p->root exactly like Builder on the device.
int build_tree_device(igs_ctx* ctx, PartitionDev* p, int n_max) {
    const uint32_t n = ctx->n;
    const size_t tb_n = ((size_t)n + 255) / 256;
    // scratch: kx, ky (u64); ordX, ordY, iota, node_of, key, key_sorted, seg (u32)
    // (active nodes hold > n_max >= 1 points each: at most n / 2 of them)
    uint32_t* s32 = (uint32_t*)igs_scratch(ctx, 29, ((size_t)n * 7 + 5 * ((size_t)n / 2 + 1)) * 4);
    unsigned long long* s64 = (unsigned long long*)igs_scratch(ctx, 30, (size_t)n * 8 * 4);
    if (!s32 || !s64) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp build)");
    unsigned long long *kx = s64, *ky = s64 + n, *ks = s64 + 2 * (size_t)n;
    uint32_t *ordX = s32, *ordY = s32 + n, *iota = s32 + 2 * (size_t)n, *node_of = s32 + 3 * (size_t)n,
             *key = s32 + 4 * (size_t)n, *key_sorted = s32 + 5 * (size_t)n, *seg = s32 + 6 * (size_t)n;
    uint32_t* small = s32 + 7 * (size_t)n;  // per-level node arrays (start | size | pos | child...)
    double* line_d = (double*)(s64 + 3 * (size_t)n);
    gb_keys_kernel<<<(unsigned)tb_n, 256, 0, ctx->stream>>>(ctx->scan, n, kx, ky, iota, node_of);
    IGS_LAUNCHED(ctx);
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, kx, ks, iota, ordX, (int)n, 0, 64, ctx->stream);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, key, key_sorted, ordX, seg, (int)n, 0, 32, ctx->stream);
    void* temp = igs_scratch(ctx, 31, std::max(tb, tb2));
    if (!temp) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp build)");
    const size_t tcap = std::max(tb, tb2);
    tb = tcap;
    IGS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(temp, tb, kx, ks, iota, ordX, (int)n, 0, 64, ctx->stream));
    tb = tcap;
    IGS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(temp, tb, ky, ks, iota, ordY, (int)n, 0, 64, ctx->stream));
    ctx->launches += 8;

    std::vector<std::vector<GbLevelNode>> levels(1);
    levels[0].push_back(GbLevelNode{n, (long long)n <= (long long)n_max, 0, 0.0, 0, 0, RectD{0.0, 0.0, 1.0, 1.0}});
    for (int d = 0;; ++d) {
        std::vector<GbLevelNode>& lv = levels[d];
        // active nodes of this level in order, their starts
        std::vector<uint32_t> act;
        for (uint32_t k = 0; k < lv.size(); ++k)
            if (!lv[k].leaf) act.push_back(k);
        const uint32_t na = (uint32_t)act.size();
        if (na == 0) break;
        std::vector<uint32_t> hs(3 * (size_t)na);  // start | size | (pos)
        uint32_t total = 0;
        for (uint32_t a = 0; a < na; ++a) {
            hs[a] = total;
            hs[na + a] = lv[act[a]].size;
            total += lv[act[a]].size;
        }
        uint32_t *d_start = small, *d_size = small + na, *d_pos = small + 2 * (size_t)na,
                 *d_child = small + 3 * (size_t)na;  // 2 na entries
        IGS_CUDA(ctx, cudaMemcpyAsync(d_start, hs.data(), 2 * (size_t)na * 4, cudaMemcpyHostToDevice, ctx->stream));
        const int axis = d % 2;
        const uint32_t* ord = axis == 0 ? ordX : ordY;
        // node key per point in the global order; inactive points sort last
        gb_gather_kernel<<<(unsigned)tb_n, 256, 0, ctx->stream>>>(ord, node_of, n, key);
        IGS_LAUNCHED(ctx);
        int bits = 1;
        while (bits < 32 && (1u << bits) <= na) ++bits;
        tb = tcap;
        IGS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(temp, tb, key, key_sorted, ord, seg, (int)n, 0, bits,
                                                      ctx->stream));
        ctx->launches += 2 * ((bits + 7) / 8) + 1;
        gb_split_kernel<<<(na + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, seg, d_start, d_size, na, axis, d_pos,
                                                                  line_d);
        IGS_LAUNCHED(ctx);
        std::vector<double> hl(na);
        IGS_CUDA(ctx, cudaMemcpyAsync(hs.data() + 2 * (size_t)na, d_pos, (size_t)na * 4, cudaMemcpyDeviceToHost,
                                      ctx->stream));
        IGS_CUDA(ctx, cudaMemcpyAsync(hl.data(), line_d, (size_t)na * 8, cudaMemcpyDeviceToHost, ctx->stream));
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        // children (bsp.cpp:96-117): low = [0, pos), high = [pos, n)
        levels.emplace_back();
        std::vector<GbLevelNode>& nx = levels[d + 1];
        std::vector<GbLevelNode>& cur = levels[d];  // (levels may have reallocated)
        std::vector<uint32_t> child(2 * (size_t)na);
        uint32_t next_active = 0;
        for (uint32_t a = 0; a < na; ++a) {
            GbLevelNode& nd = cur[act[a]];
            nd.pos = hs[2 * (size_t)na + a];
            nd.line = hl[a];
            RectD lr = nd.rect, hr = nd.rect;
            if (axis == 0) {
                lr.x2 = nd.line;
                hr.x1 = nd.line;
            } else {
                lr.y2 = nd.line;
                hr.y1 = nd.line;
            }
            const uint32_t sz[2] = {nd.pos, nd.size - nd.pos};
            const RectD rc[2] = {lr, hr};
            for (int h = 0; h < 2; ++h) {
                const bool leaf = (long long)sz[h] <= (long long)n_max;
                (h == 0 ? nd.low : nd.high) = (uint32_t)nx.size();
                child[2 * (size_t)a + h] = leaf ? 0xFFFFFFFFu : next_active++;
                nx.push_back(GbLevelNode{sz[h], leaf, 0, 0.0, 0, 0, rc[h]});
            }
        }
        IGS_CUDA(ctx, cudaMemcpyAsync(d_child, child.data(), child.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        gb_move_kernel<<<(total + 255) / 256, 256, 0, ctx->stream>>>(seg, key_sorted, total, d_start, d_pos, d_child,
                                                                    node_of);
        IGS_LAUNCHED(ctx);
        // (the next level's host staging reuses `small`; order the copies)
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    // DFS numbering (bsp.cpp:32-118): preorder node ids, leaves in visit order
    const int D = (int)levels.size();
    std::vector<std::vector<uint32_t>> cnt(D), leaves(D);
    for (int d = D - 1; d >= 0; --d) {
        cnt[d].resize(levels[d].size());
        leaves[d].resize(levels[d].size());
        for (size_t k = 0; k < levels[d].size(); ++k) {
            const GbLevelNode& nd = levels[d][k];
            if (nd.leaf) {
                cnt[d][k] = 1;
                leaves[d][k] = 1;
            } else {
                cnt[d][k] = 1 + cnt[d + 1][nd.low] + cnt[d + 1][nd.high];
                leaves[d][k] = leaves[d + 1][nd.low] + leaves[d + 1][nd.high];
            }
        }
    }
    p->nodes.assign(cnt[0][0], NodeD{0, 0.0, -1, -1, -1});
    p->blocks.assign(leaves[0][0], RectD{});
    std::vector<std::vector<int32_t>> id(D), boff(D);
    for (int d = 0; d < D; ++d) {
        id[d].resize(levels[d].size());
        boff[d].resize(levels[d].size());
    }
    id[0][0] = 0;
    boff[0][0] = 0;
    for (int d = 0; d < D; ++d)
        for (size_t k = 0; k < levels[d].size(); ++k) {
            const GbLevelNode& nd = levels[d][k];
            NodeD& out = p->nodes[id[d][k]];
            if (nd.leaf) {
                out.block = boff[d][k];
                p->blocks[boff[d][k]] = nd.rect;
                continue;
            }
            out.axis = d % 2;
            out.line = nd.line;
            id[d + 1][nd.low] = id[d][k] + 1;
            id[d + 1][nd.high] = id[d][k] + 1 + (int32_t)cnt[d + 1][nd.low];
            boff[d + 1][nd.low] = boff[d][k];
            boff[d + 1][nd.high] = boff[d][k] + (int32_t)leaves[d + 1][nd.low];
            out.low = id[d + 1][nd.low];
            out.high = id[d + 1][nd.high];
        }
    p->root = 0;
    return IGS_OK;
}

int download_centres(igs_ctx* ctx, std::vector<double>& mx, std::vector<double>& my) {
    std::vector<double> p((size_t)ctx->n * 8);
    if (ctx->n) {
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        IGS_CUDA(ctx, cudaMemcpy(p.data(), ctx->params, p.size() * 8, cudaMemcpyDeviceToHost));
    }
    mx.resize(ctx->n);
    my.resize(ctx->n);
    for (uint32_t i = 0; i < ctx->n; ++i) {
        mx[i] = p[(size_t)i * 8];
        my[i] = p[(size_t)i * 8 + 1];
    }
    return IGS_OK;
}

}  // namespace

int igs_partition_free(igs_ctx* ctx) {
    if (ctx->part) {
        free_dev(ctx->part);
        delete ctx->part;
        ctx->part = nullptr;
    }
    return IGS_OK;
}

extern "C" {

// bsp.cpp:153-176 build_partition
int igs_partition_build(igs_ctx* ctx, int n_max) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "build_partition requires a non-empty GaussianSet");
    if (n_max < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "n_max must be >= 1");
    auto* p = new PartitionDev();
    p->tree = true;
    p->n_max = n_max;
    p->source_size = ctx->n;
    int e = build_tree_device(ctx, p, n_max);
    if (e) {
        delete p;
        return e;
    }
    igs_partition_free(ctx);
    ctx->part = p;
    if ((e = finish_partition(ctx, p))) {
        igs_partition_free(ctx);
        return e;
    }
    return IGS_OK;
}

// bsp.cpp:197-218 rebuild_partition
int igs_partition_rebuild(igs_ctx* ctx, const double* rects4, uint32_t n_blocks) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (n_blocks == 0 || !rects4)
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "rebuild_partition requires at least one block");
    auto* p = new PartitionDev();
    p->tree = false;
    p->source_size = ctx->n;
    p->blocks.resize(n_blocks);
    std::memcpy(p->blocks.data(), rects4, sizeof(RectD) * n_blocks);
    igs_partition_free(ctx);
    ctx->part = p;
    int e = finish_partition(ctx, p);
    if (e) igs_partition_free(ctx);
    return e;
}

uint32_t igs_partition_source_size(igs_ctx* ctx) { return ctx->part ? ctx->part->source_size : 0; }

int igs_partition_info(igs_ctx* ctx, uint32_t* n_blocks, uint64_t* shell_total) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    if (n_blocks) *n_blocks = ctx->part->nb;
    if (shell_total) *shell_total = ctx->part->shell_total;
    return IGS_OK;
}

int igs_partition_get(igs_ctx* ctx, double* blocks4, double* shells4, uint32_t* shell_offsets,
                      uint32_t* shell_members) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    PartitionDev* p = ctx->part;
    if (blocks4) std::memcpy(blocks4, p->blocks.data(), sizeof(RectD) * p->nb);
    if (shells4) std::memcpy(shells4, p->shells.data(), sizeof(RectD) * p->nb);
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (shell_offsets) IGS_CUDA(ctx, cudaMemcpy(shell_offsets, p->d_shell_off, (size_t)(p->nb + 1) * 4,
                                                cudaMemcpyDeviceToHost));
    if (shell_members && p->shell_total)
        IGS_CUDA(ctx, cudaMemcpy(shell_members, p->d_shell_mem, p->shell_total * 4, cudaMemcpyDeviceToHost));
    return IGS_OK;
}

int igs_locate_blocks(igs_ctx* ctx, const double* uv, uint32_t npts, int32_t* blocks) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (!ctx->part || ctx->part->nb == 0) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    if (npts == 0) return IGS_OK;
    double* duv = (double*)igs_scratch(ctx, 17, (size_t)npts * 16);
    int32_t* dout = (int32_t*)igs_scratch(ctx, 18, (size_t)npts * 4);
    if (!duv || !dout) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    IGS_CUDA(ctx, cudaMemcpyAsync(duv, uv, (size_t)npts * 16, cudaMemcpyHostToDevice, ctx->stream));
    locate_kernel<<<(npts + 127) / 128, 128, 0, ctx->stream>>>(view_of(ctx->part), duv, npts, dout);
    IGS_LAUNCHED(ctx);
    IGS_CUDA(ctx, cudaMemcpyAsync(blocks, dout, (size_t)npts * 4, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

// bsp.cpp:334 render_image_blocked, rows [row0, row1) (tile-row sharding of
// the evaluation / decode render); the rows land at their place in the
// context's W x H image
int igs_blocked_render_rows(igs_ctx* ctx, int width, int height, int k, int row0, int row1) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "render requires a non-empty GaussianSet");
    if (width < 1 || height < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "render target must be at least 1x1");
    if (k < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "k must be >= 1");
    if (row0 < 0 || row1 > height || row0 > row1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bad row range");
    int e;
    if ((e = check_partition(ctx))) return e;
    if ((e = igs_ensure_image(ctx, width, height))) return e;
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "blocked render supports k <= 32");
    if (row1 == row0) return IGS_OK;
    const LocView v = view_of(ctx->part);
    dim3 grid((width + kTile - 1) / kTile, (row1 - row0 + kTile - 1) / kTile), blk(kTile, kTile);
    float* out = (float*)ctx->image.p;
    unsigned long long* pairs = igs_prof_counter(ctx, IGS_PROF_BLOCKED);
    igs_prof_begin(ctx, IGS_PROF_BLOCKED);
#define LAUNCH(KC)                                                                                          \
    blocked_raster_kernel<KC><<<grid, blk, 0, ctx->stream>>>(ctx->scan, ctx->shade, v, ctx->part->d_shell_off, \
                                                             ctx->part->d_shell_mem, width, height, row0, row1, kk, \
                                                             out, pairs)
    if (kk <= 4) LAUNCH(4);
    else if (kk <= 8) LAUNCH(8);
    else if (kk <= 10) LAUNCH(10);
    else if (kk <= 16) LAUNCH(16);
    else LAUNCH(32);
#undef LAUNCH
    IGS_LAUNCHED(ctx);
    igs_prof_end(ctx, IGS_PROF_BLOCKED, 0.0);
    return IGS_OK;
}

int igs_render_image_blocked(igs_ctx* ctx, int width, int height, int k, float* out_rgb) {
    int e = igs_blocked_render_rows(ctx, width, height, k, 0, height);
    if (e) return e;
    if (out_rgb) {
        IGS_CUDA(ctx, cudaMemcpyAsync(out_rgb, ctx->image.p, (size_t)width * height * 12, cudaMemcpyDeviceToHost,
                                      ctx->stream));
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return IGS_OK;
}

int igs_render_image_blocked_rows(igs_ctx* ctx, int width, int height, int k, int row0, int row1, float* out_rgb) {
    int e = igs_blocked_render_rows(ctx, width, height, k, row0, row1);
    if (e) return e;
    if (out_rgb && row1 > row0) {
        IGS_CUDA(ctx, cudaMemcpyAsync(out_rgb, (const float*)ctx->image.p + (size_t)row0 * width * 3,
                                      (size_t)width * (row1 - row0) * 12, cudaMemcpyDeviceToHost, ctx->stream));
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return IGS_OK;
}

}  // extern "C"

// blocked_pixel at npts device points (validated partition, kk <= 32)
int igs_blocked_points_dev(igs_ctx* ctx, const double* duv, uint32_t npts, int kk, double* drgb) {
    const LocView v = view_of(ctx->part);
#define LAUNCH(KC)                                                                                    \
    blocked_points_kernel<KC><<<(npts + 127) / 128, 128, 0, ctx->stream>>>(                          \
        ctx->scan, ctx->shade, v, ctx->part->d_shell_off, ctx->part->d_shell_mem, duv, npts, kk, drgb)
    if (kk <= 4) LAUNCH(4);
    else if (kk <= 8) LAUNCH(8);
    else if (kk <= 10) LAUNCH(10);
    else if (kk <= 16) LAUNCH(16);
    else LAUNCH(32);
#undef LAUNCH
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

extern "C" {

// bsp.cpp:321-332 render_topk_blocked at many points
int igs_render_points_blocked(igs_ctx* ctx, const double* uv, uint32_t npts, int k, double* rgb) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "render requires a non-empty GaussianSet");
    if (k < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "k must be >= 1");
    int e;
    if ((e = check_partition(ctx))) return e;
    if (npts == 0) return IGS_OK;
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "blocked render supports k <= 32");
    double* duv = (double*)igs_scratch(ctx, 17, (size_t)npts * 16);
    double* drgb = (double*)igs_scratch(ctx, 20, (size_t)npts * 24);
    if (!duv || !drgb) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    IGS_CUDA(ctx, cudaMemcpyAsync(duv, uv, (size_t)npts * 16, cudaMemcpyHostToDevice, ctx->stream));
    if ((e = igs_blocked_points_dev(ctx, duv, npts, kk, drgb))) return e;
    if (rgb) {
        IGS_CUDA(ctx, cudaMemcpyAsync(rgb, drgb, (size_t)npts * 24, cudaMemcpyDeviceToHost, ctx->stream));
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return IGS_OK;
}

}  // extern "C"
