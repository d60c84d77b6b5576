// bsp.cu -- BSP acceleration (bsp.hpp:70-106): partition build/rebuild,
// kernel 2 in its BSP form (shell binning), locate_block, and kernel 3 over
// shell lists (render_image_blocked, render_topk_blocked).
//
// Reference: bsp.cpp:14-23 shell_of, :27-118 Builder::build, :132-176
// build_partition / collect_shell_members, :178-218 grid locator +
// rebuild_partition, :220-264 locate_block, :268-341 blocked renders.
//
// Everything runs on the device with the repo's own scan and radix sort
// (scan.cu); the host only turns the per-level node records into the
// reference's DFS numbering at the end:
//   * tree build: a level-synchronous restatement of the recursive
//     alternating-axis median split (build_tree_device below);
//   * shell binning: shell_members[b] = {i : mu_i in shell_b (closed)}, in
//     ascending i -- a uniform cell grid narrows each Gaussian's candidate
//     shells, (shell, index) pairs are emitted in index order and stably
//     radix-sorted by shell.  This is exactly the set collect_shell_members
//     gathers through the tree (its bbox pruning only skips non-members), and
//     exactly the rectangle test rebuild_partition runs (bsp.cpp:214-216).
//   * locate: the tree descent (c < line ? low : high) or, for partitions
//     rebuilt from corners, the grid locator with its first-containing /
//     nearest-Chebyshev / scan-all fallbacks, op for op.
//   * blocked raster: CTA per 16x16 tile; the tile's pixels usually fall in
//     one or two blocks -- the CTA loops over the distinct blocks present,
//     staging each shell list through shared memory for the pixels of that
//     block (scan order is index order, as the reference's member lists).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "igs_internal.cuh"
#include "scan.cuh"

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
    std::vector<uint32_t> grid_off_h, grid_blk_h;  // the grid locator's cells (rebuilt partitions)
    std::vector<int32_t> leaf_block;               // built partitions: pool node -> block (leaves)
    uint32_t* d_leaf_of = nullptr;                 // built partitions: every Gaussian's leaf (pool node)
    // device
    RectD* d_blocks = nullptr;
    RectD* d_shells = nullptr;
    NodeD* d_nodes = nullptr;
    uint32_t* d_grid_off = nullptr;  // grid_dim^2 + 1
    uint32_t* d_grid_blk = nullptr;
    uint32_t* d_shell_off = nullptr;  // nb + 1
    uint32_t* d_shell_mem = nullptr;
    // capacities (bytes) of the device arrays above: a replaced partition's
    // arrays are kept for the next one (ctx->part_spare), so a rebuild at
    // every evaluation allocates nothing
    size_t cap[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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

// Shell binning (kernel 2, count -> scan -> sort): shell_members[b] = {i :
// mu_i in shell_b (closed)} in ascending i -- the set collect_shell_members
// gathers through the tree (bsp.cpp:132-143, its bbox pruning only skips
// non-members) and exactly rebuild_partition's rectangle test
// (bsp.cpp:214-216).  A uniform grid of G x G cells lists the shells that
// overlap each cell (a superset: floor(x G) is monotone in x); every
// Gaussian tests only its cell's shells, counts its memberships, and after
// an exclusive scan emits (shell, index) pairs in index order; a stable
// radix sort by shell then leaves each shell's members ascending.
__device__ __forceinline__ uint32_t grid_cell(double x, double y, int G) {
    int cx = (int)floor(x * G), cy = (int)floor(y * G);
    cx = cx < 0 ? 0 : (cx > G - 1 ? G - 1 : cx);
    cy = cy < 0 ? 0 : (cy > G - 1 ? G - 1 : cy);
    return (uint32_t)(cy * G + cx);
}

// pass 0: memberships per Gaussian into cnt[i]; pass 1: the (shell, i)
// pairs at off[i], and a count per shell
__global__ void shell_pairs_kernel(const ScanRec* __restrict__ scan, uint32_t n, const RectD* __restrict__ shells,
                                   const uint32_t* __restrict__ cell_off, const uint32_t* __restrict__ cell_shell,
                                   int G, int pass, uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                                   unsigned long long* __restrict__ pair_key, uint32_t* __restrict__ pair_val,
                                   uint32_t* __restrict__ shell_cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = scan[i].mu_x, y = scan[i].mu_y;
    const uint32_t c = grid_cell(x, y, G);
    uint32_t k = 0, o = pass ? off[i] : 0u;
    for (uint32_t j = cell_off[c]; j < cell_off[c + 1]; ++j) {
        const uint32_t b = cell_shell[j];
        if (!contains_closed(shells[b], x, y)) continue;
        if (pass) {
            pair_key[o + k] = b;
            pair_val[o + k] = i;
            atomicAdd(shell_cnt + b, 1u);
        }
        ++k;
    }
    if (!pass) cnt[i] = k;
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

// grow-only device array: ptr keeps at least `bytes` (capacity in cap)
template <class T>
bool reserve_dev(T*& ptr, size_t& cap, size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    if (cap >= bytes) return true;
    cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    if (cudaMalloc(&ptr, bytes) != cudaSuccess) {
        cudaGetLastError();
        ptr = nullptr;
        return false;
    }
    cap = bytes;
    return true;
}

template <class T>
bool to_dev(igs_ctx* ctx, T*& ptr, size_t& cap, const std::vector<T>& v) {
    if (!reserve_dev(ptr, cap, v.size() * sizeof(T))) return false;
    if (!v.empty()) cudaMemcpyAsync(ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream);
    return true;
}

void free_dev(PartitionDev* p) {
    cudaFree(p->d_blocks);
    cudaFree(p->d_shells);
    cudaFree(p->d_nodes);
    cudaFree(p->d_grid_off);
    cudaFree(p->d_grid_blk);
    cudaFree(p->d_shell_off);
    cudaFree(p->d_shell_mem);
    cudaFree(p->d_leaf_of);
}

// a new partition, inheriting the device arrays of the last replaced one
PartitionDev* new_partition(igs_ctx* ctx) {
    auto* p = new PartitionDev();
    if (PartitionDev* s = ctx->part_spare) {
        p->d_blocks = s->d_blocks;
        p->d_shells = s->d_shells;
        p->d_nodes = s->d_nodes;
        p->d_grid_off = s->d_grid_off;
        p->d_grid_blk = s->d_grid_blk;
        p->d_shell_off = s->d_shell_off;
        p->d_shell_mem = s->d_shell_mem;
        p->d_leaf_of = s->d_leaf_of;
        std::copy(s->cap, s->cap + 8, p->cap);
        delete s;
        ctx->part_spare = nullptr;
    }
    return p;
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
    if (!to_dev(ctx, p->d_blocks, p->cap[0], p->blocks) || !to_dev(ctx, p->d_shells, p->cap[1], p->shells) ||
        !to_dev(ctx, p->d_nodes, p->cap[2], p->nodes))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
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
        if (!to_dev(ctx, p->d_grid_off, p->cap[3], off) || !to_dev(ctx, p->d_grid_blk, p->cap[4], blk))
            return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
        p->grid_off_h = std::move(off);
        p->grid_blk_h = std::move(blk);
    }
    // shell -> cell lists on the host (a few thousand shells)
    const uint32_t nb = p->nb, n = ctx->n;
    const int G = std::max(1, (int)std::ceil(2.0 * std::sqrt((double)nb)));
    std::vector<std::vector<uint32_t>> cl((size_t)G * G);
    auto cidx = [&](double v) { return std::clamp((int)std::floor(v * G), 0, G - 1); };
    for (uint32_t b = 0; b < nb; ++b) {
        const RectD& r = p->shells[b];
        for (int cy = cidx(r.y1); cy <= cidx(r.y2); ++cy)
            for (int cx = cidx(r.x1); cx <= cidx(r.x2); ++cx) cl[(size_t)cy * G + cx].push_back(b);
    }
    std::vector<uint32_t> coff(cl.size() + 1), cshell;
    for (size_t c = 0; c < cl.size(); ++c) {
        coff[c] = (uint32_t)cshell.size();
        cshell.insert(cshell.end(), cl[c].begin(), cl[c].end());
    }
    coff[cl.size()] = (uint32_t)cshell.size();
    uint32_t* d_coff = (uint32_t*)igs_scratch(ctx, 25, coff.size() * 4);
    uint32_t* d_cshell = (uint32_t*)igs_scratch(ctx, 26, std::max<size_t>(cshell.size(), 1) * 4);
    uint32_t* cnt = (uint32_t*)igs_scratch(ctx, 29, ((size_t)n + 1) * 4);
    if (!reserve_dev(p->d_shell_off, p->cap[5], (size_t)(nb + 1) * 4) || !d_coff || !d_cshell || !cnt)
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp)");
    igs_prof_begin(ctx, IGS_PROF_BLOCKED);
    IGS_CUDA(ctx, cudaMemcpyAsync(d_coff, coff.data(), coff.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    IGS_CUDA(ctx, cudaMemcpyAsync(d_cshell, cshell.data(), cshell.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    const unsigned tb = (n + 255) / 256;
    shell_pairs_kernel<<<tb, 256, 0, ctx->stream>>>(ctx->scan, n, p->d_shells, d_coff, d_cshell, G, 0, cnt, nullptr,
                                                     nullptr, nullptr, nullptr);
    IGS_LAUNCHED(ctx);
    IGS_CUDA(ctx, cudaMemsetAsync(cnt + n, 0, 4, ctx->stream));
    int e;
    if ((e = igs_scan_excl_u32(ctx, cnt, cnt, (size_t)n + 1))) return e;  // cnt[n] = pair total
    uint32_t total = 0;
    IGS_CUDA(ctx, cudaMemcpyAsync(&total, cnt + n, 4, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    p->shell_total = total;
    if (!reserve_dev(p->d_shell_mem, p->cap[6], (size_t)total * 4))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp shells)");
    unsigned long long* pk = (unsigned long long*)igs_scratch(ctx, 30, std::max<size_t>(total, 1) * 8 * 3);
    uint32_t* pv = (uint32_t*)igs_scratch(ctx, 31, std::max<size_t>(total, 1) * 4 * 2);
    if (!pk || !pv) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp shells)");
    IGS_CUDA(ctx, cudaMemsetAsync(p->d_shell_off, 0, (size_t)(nb + 1) * 4, ctx->stream));
    shell_pairs_kernel<<<tb, 256, 0, ctx->stream>>>(ctx->scan, n, p->d_shells, d_coff, d_cshell, G, 1, nullptr, cnt,
                                                     pk, pv, p->d_shell_off);
    IGS_LAUNCHED(ctx);
    if ((e = igs_scan_excl_u32(ctx, p->d_shell_off, p->d_shell_off, (size_t)nb + 1))) return e;
    int bits = 1;
    while (bits < 32 && (1ull << bits) < nb) ++bits;
    if ((e = igs_radix_sort_u64_u32(ctx, pk, pv, pk + total, p->d_shell_mem, pk + 2 * (size_t)total, pv + total,
                                    total, bits)))
        return e;
    igs_prof_end(ctx, IGS_PROF_BLOCKED, (double)total);
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
// Level-synchronous restatement of Builder::build, device-resident.
// Invariant: every active node of the current level owns one contiguous
// segment [start, start + size) of BOTH ordX and ordY, and within it ordX is
// sorted by (x, idx) and ordY by (y, idx) -- the reference comparator's
// order along either axis.  Set up once by two stable radix sorts of the
// coordinate keys (indices in order).  Per level (axis a = depth % 2):
//   1. node flags -> exclusive scan = active index of every node;
//   2. one thread per active node applies the tie-aware split rule
//      (bsp.cpp:54-95) to its ord_a segment -> (pos, line), and writes its
//      two children (sizes pos / size - pos, starts, rects) to the next level
//      at positions 2 a, 2 a + 1 (Builder's low-then-high order);
//   3. the low child is the ord_a segment's first pos points (ord_a needs no
//      change); ord_b is stably partitioned inside each segment by side
//      (a flag scan over all positions gives each point's rank on its side),
//      so both invariants hold for the children.
// Nothing comes back to the host per level: levels run in batches of eight
// (a level past the last active one costs a few empty launches) and one
// readback decides whether another batch is needed.  The host then numbers
// nodes and blocks in DFS order from the downloaded per-level records.
__device__ __forceinline__ unsigned long long coord_key(double v) {
    if (v == 0.0) v = 0.0;  // -0 and +0 compare equal in the reference
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

constexpr uint32_t kInact = 0xFFFFFFFFu;

struct BuildNodes {  // the node pool, all levels (<= 2n - 1 nodes)
    uint32_t* size;
    uint32_t* start;
    uint32_t* act;  // active index within its level, kInact for a leaf
    uint32_t* pos;
    double* line;
    RectD* rect;
};

__global__ void gb_keys_kernel(const ScanRec* __restrict__ scan, uint32_t n, unsigned long long* __restrict__ kx,
                               unsigned long long* __restrict__ ky, uint32_t* __restrict__ iota,
                               uint32_t* __restrict__ node_of, BuildNodes P, uint32_t* __restrict__ lvl) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {  // the root: level 0 = node 0
        P.size[0] = n;
        P.start[0] = 0;
        P.rect[0] = RectD{0.0, 0.0, 1.0, 1.0};
        lvl[0] = 0;  // base of level 0
        lvl[1] = 1;  // its node count
    }
    if (i >= n) return;
    kx[i] = coord_key(scan[i].mu_x);
    ky[i] = coord_key(scan[i].mu_y);
    iota[i] = i;
    node_of[i] = 0;
}

// lvl[2 d] = pool base of level d, lvl[2 d + 1] = its node count
__global__ void gb_flag_kernel(BuildNodes P, const uint32_t* __restrict__ lvl, int d, uint32_t bound, int n_max,
                               uint32_t* __restrict__ flag) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= bound) return;
    const uint32_t cnt = lvl[2 * d + 1];
    flag[j] = j < cnt && (long long)P.size[lvl[2 * d] + j] > (long long)n_max ? 1u : 0u;
}

__device__ __forceinline__ double coord_of(const ScanRec* __restrict__ scan, uint32_t i, int axis) {
    return axis == 0 ? scan[i].mu_x : scan[i].mu_y;
}

// bsp.cpp:54-95 on node j's ord_a segment; children to level d + 1
__global__ void gb_split_kernel(const ScanRec* __restrict__ scan, const uint32_t* __restrict__ ord_a, BuildNodes P,
                                uint32_t* __restrict__ lvl, int d, uint32_t bound, int n_max,
                                const uint32_t* __restrict__ flag, const uint32_t* __restrict__ aidx) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t base = lvl[2 * d], cnt = lvl[2 * d + 1];
    if (cnt == 0) {  // past the last level: keep the (empty) level records defined
        if (j == 0) {
            lvl[2 * d + 2] = base;
            lvl[2 * d + 3] = 0;
        }
        return;
    }
    if (j >= cnt || j >= bound) return;
    const uint32_t g = base + j;
    if (j == cnt - 1) {  // the next level: 2 x (active nodes here)
        lvl[2 * d + 2] = base + cnt;
        lvl[2 * d + 3] = 2 * (aidx[j] + flag[j]);
    }
    if (!flag[j]) {
        P.act[g] = kInact;
        return;
    }
    const uint32_t a = aidx[j];
    P.act[g] = a;
    const int axis = d % 2;
    const uint32_t* m = ord_a + P.start[g];
    const size_t n = P.size[g], half = n / 2;
    auto c = [&](size_t k) { return coord_of(scan, m[k], axis); };
    size_t pos = 0;
    double line = 0.0;
    bool forced = false;
    if (c(half - 1) < c(half)) {
        pos = half;
    } else {
        size_t lo = 0, hi = 0;
        bool has_lo = false, has_hi = false;
        for (size_t k = half; k-- > 1;)
            if (c(k - 1) < c(k)) {
                lo = k;
                has_lo = true;
                break;
            }
        for (size_t k = half + 1; k < n; ++k)
            if (c(k - 1) < c(k)) {
                hi = k;
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
    P.pos[g] = (uint32_t)pos;
    P.line[g] = line;
    const RectD r = P.rect[g];
    RectD lr = r, hr = r;
    if (axis == 0) {
        lr.x2 = line;
        hr.x1 = line;
    } else {
        lr.y2 = line;
        hr.y1 = line;
    }
    const uint32_t c0 = base + cnt + 2 * a;
    P.size[c0] = (uint32_t)pos;
    P.start[c0] = P.start[g];
    P.rect[c0] = lr;
    P.size[c0 + 1] = (uint32_t)(n - pos);
    P.start[c0 + 1] = P.start[g] + (uint32_t)pos;
    P.rect[c0 + 1] = hr;
}

// side of every point of an active node (position in its ord_a segment)
__global__ void gb_side_kernel(const uint32_t* __restrict__ ord_a, uint32_t n, BuildNodes P,
                               const uint32_t* __restrict__ node_of, uint8_t* __restrict__ side) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = ord_a[i], g = node_of[p];
    if (g == kInact || P.act[g] == kInact) return;
    side[p] = i - P.start[g] < P.pos[g] ? 0 : 1;
}

// flag0[i] = the point at ord_b[i] goes to its node's low child
__global__ void gb_lowflag_kernel(const uint32_t* __restrict__ ord_b, uint32_t n, BuildNodes P,
                                  const uint32_t* __restrict__ node_of, const uint8_t* __restrict__ side,
                                  uint32_t* __restrict__ flag0) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = ord_b[i], g = node_of[p];
    flag0[i] = (g != kInact && P.act[g] != kInact && side[p] == 0) ? 1u : 0u;
}

// stable partition of ord_b inside each active segment; points move to
// their child (or out of the build once their node is a leaf)
__global__ void gb_scatter_kernel(const uint32_t* __restrict__ ord_b, uint32_t n, BuildNodes P,
                                  uint32_t* __restrict__ node_of, const uint8_t* __restrict__ side,
                                  const uint32_t* __restrict__ s0, const uint32_t* __restrict__ lvl, int d,
                                  uint32_t* __restrict__ ord_b_out, uint32_t* __restrict__ leaf_of) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = ord_b[i], g = node_of[p];
    if (g == kInact) {
        ord_b_out[i] = p;
        return;
    }
    const uint32_t a = P.act[g];
    if (a == kInact) {  // its node is a leaf: the point stays put for good
        ord_b_out[i] = p;
        node_of[p] = kInact;
        leaf_of[p] = g;  // the block members (Builder's leaf lists)
        return;
    }
    const uint32_t start = P.start[g], pos = P.pos[g];
    const uint32_t r0 = s0[i] - s0[start];  // low-side points before i in the segment
    const uint32_t sd = side[p];
    ord_b_out[sd == 0 ? start + r0 : start + pos + (i - start - r0)] = p;
    node_of[p] = lvl[2 * d] + lvl[2 * d + 1] + 2 * a + sd;
}

// Builds p->nodes / p->blocks / p->root exactly like Builder, on the device.
int build_tree_device(igs_ctx* ctx, PartitionDev* p, int n_max) {
    const uint32_t n = ctx->n;
    const unsigned tb_n = (unsigned)(((size_t)n + 255) / 256);
    const size_t pool = 2 * (size_t)n + 2;  // nodes of all levels
    // scratch: kx, ky, key tmp (u64); ordX, ordY, ord tmp, iota, node_of, flags, scan (u32); side (u8)
    unsigned long long* s64 = (unsigned long long*)igs_scratch(ctx, 30, (size_t)n * 8 * 3);
    uint32_t* s32 = (uint32_t*)igs_scratch(ctx, 29, ((size_t)n * 7 + 4) * 4);
    uint8_t* side = (uint8_t*)igs_scratch(ctx, 31, (size_t)n + 16);
    // node pool: size, start, act, pos (u32) | line (f64) | rect (4 f64) | levels
    char* np = (char*)igs_scratch(ctx, 45, pool * (4 * 4 + 8 + 32) + 64 * 1024);
    if (!s64 || !s32 || !side || !np) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp build)");
    unsigned long long *kx = s64, *ky = s64 + n, *kt = s64 + 2 * (size_t)n;
    uint32_t *ordX = s32, *ordY = s32 + n, *ordT = s32 + 2 * (size_t)n, *iota = s32 + 3 * (size_t)n,
             *node_of = s32 + 4 * (size_t)n, *flag = s32 + 5 * (size_t)n, *scan_o = s32 + 6 * (size_t)n;
    BuildNodes P;
    P.size = (uint32_t*)np;
    P.start = P.size + pool;
    P.act = P.start + pool;
    P.pos = P.act + pool;
    P.line = (double*)(P.pos + pool);
    P.rect = (RectD*)(P.line + pool);
    uint32_t* lvl = (uint32_t*)(P.rect + pool);  // 2 words per level (<= 8192 levels)
    const int kMaxLevels = 8192;
    if (!reserve_dev(p->d_leaf_of, p->cap[7], (size_t)n * 4))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (bsp build)");
    gb_keys_kernel<<<std::max(tb_n, 1u), 256, 0, ctx->stream>>>(ctx->scan, n, kx, ky, iota, node_of, P, lvl);
    IGS_LAUNCHED(ctx);
    int e;
    // the (coord, idx) orders: stable sorts of the coordinate keys, indices in order
    if ((e = igs_radix_sort_u64_u32(ctx, kx, iota, kx, ordX, kt, ordT, n, 64))) return e;
    if ((e = igs_radix_sort_u64_u32(ctx, ky, iota, ky, ordY, kt, ordT, n, 64))) return e;
    uint32_t* ord[2] = {ordX, ordY};
    uint32_t* spare = ordT;
    int d = 0;
    for (;;) {
        for (int batch = 0; batch < 8; ++batch, ++d) {
            if (d + 1 >= kMaxLevels) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "partition deeper than 8192 levels");
            const int axis = d % 2;
            // a level has at most min(2^d, n) nodes
            const uint32_t bound = d < 31 ? std::min<uint32_t>(1u << d, n) : n;
            gb_flag_kernel<<<(bound + 255) / 256, 256, 0, ctx->stream>>>(P, lvl, d, bound, n_max, flag);
            IGS_LAUNCHED(ctx);
            if ((e = igs_scan_excl_u32(ctx, flag, scan_o, bound))) return e;
            gb_split_kernel<<<(bound + 127) / 128, 128, 0, ctx->stream>>>(ctx->scan, ord[axis], P, lvl, d, bound,
                                                                         n_max, flag, scan_o);
            IGS_LAUNCHED(ctx);
            gb_side_kernel<<<tb_n, 256, 0, ctx->stream>>>(ord[axis], n, P, node_of, side);
            IGS_LAUNCHED(ctx);
            uint32_t* ob = ord[axis ^ 1];
            gb_lowflag_kernel<<<tb_n, 256, 0, ctx->stream>>>(ob, n, P, node_of, side, flag);
            IGS_LAUNCHED(ctx);
            if ((e = igs_scan_excl_u32(ctx, flag, scan_o, n))) return e;
            gb_scatter_kernel<<<tb_n, 256, 0, ctx->stream>>>(ob, n, P, node_of, side, scan_o, lvl, d, spare,
                                                             p->d_leaf_of);
            IGS_LAUNCHED(ctx);
            ord[axis ^ 1] = spare;
            spare = ob;
        }
        uint32_t next = 0;
        IGS_CUDA(ctx, cudaMemcpyAsync(&next, lvl + 2 * d + 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (next == 0) break;
    }
    // levels 0 .. D-1 hold nodes (level d's count is 0 once d passed the last)
    std::vector<uint32_t> hl(2 * (size_t)(d + 1));
    IGS_CUDA(ctx, cudaMemcpy(hl.data(), lvl, hl.size() * 4, cudaMemcpyDeviceToHost));
    int D = 0;
    while (D <= d && hl[2 * D + 1] > 0) ++D;
    const uint32_t total = hl[2 * (D - 1)] + hl[2 * (D - 1) + 1];
    std::vector<uint32_t> hsize(total), hact(total), hpos(total);
    std::vector<double> hline(total);
    std::vector<RectD> hrect(total);
    IGS_CUDA(ctx, cudaMemcpy(hsize.data(), P.size, total * 4, cudaMemcpyDeviceToHost));
    IGS_CUDA(ctx, cudaMemcpy(hact.data(), P.act, total * 4, cudaMemcpyDeviceToHost));
    IGS_CUDA(ctx, cudaMemcpy(hpos.data(), P.pos, total * 4, cudaMemcpyDeviceToHost));
    IGS_CUDA(ctx, cudaMemcpy(hline.data(), P.line, total * 8, cudaMemcpyDeviceToHost));
    IGS_CUDA(ctx, cudaMemcpy(hrect.data(), P.rect, total * sizeof(RectD), cudaMemcpyDeviceToHost));
    // DFS numbering (bsp.cpp:32-118): preorder node ids, leaves in visit
    // order.  Node j of level l with active index a has children 2a, 2a+1 of
    // level l + 1.  Subtree node / leaf counts bottom-up, then ids top-down.
    auto base = [&](int l) { return hl[2 * l]; };
    auto count = [&](int l) { return hl[2 * l + 1]; };
    std::vector<uint32_t> cnt(total), leaves(total);
    for (int l = D - 1; l >= 0; --l)
        for (uint32_t j = 0; j < count(l); ++j) {
            const uint32_t g = base(l) + j;
            if (hact[g] == kInact) {
                cnt[g] = leaves[g] = 1;
            } else {
                const uint32_t c0 = base(l + 1) + 2 * hact[g];
                cnt[g] = 1 + cnt[c0] + cnt[c0 + 1];
                leaves[g] = leaves[c0] + leaves[c0 + 1];
            }
        }
    p->nodes.assign(cnt[0], NodeD{0, 0.0, -1, -1, -1});
    p->blocks.assign(leaves[0], RectD{});
    std::vector<int32_t> id(total), boff(total);
    p->leaf_block.assign(total, -1);
    id[0] = 0;
    boff[0] = 0;
    for (int l = 0; l < D; ++l)
        for (uint32_t j = 0; j < count(l); ++j) {
            const uint32_t g = base(l) + j;
            NodeD& out = p->nodes[id[g]];
            if (hact[g] == kInact) {
                out.block = boff[g];
                p->blocks[boff[g]] = hrect[g];
                p->leaf_block[g] = boff[g];
                continue;
            }
            const uint32_t c0 = base(l + 1) + 2 * hact[g];
            out.axis = l % 2;
            out.line = hline[g];
            id[c0] = id[g] + 1;
            id[c0 + 1] = id[g] + 1 + (int32_t)cnt[c0];
            boff[c0] = boff[g];
            boff[c0 + 1] = boff[g] + (int32_t)leaves[c0];
            out.low = id[c0];
            out.high = id[c0 + 1];
        }
    p->root = 0;
    return IGS_OK;
}

}  // namespace

// drops the resident partition; its device arrays are kept for the next one
int igs_partition_free(igs_ctx* ctx) {
    if (ctx->part) {
        if (ctx->part_spare) {
            free_dev(ctx->part_spare);
            delete ctx->part_spare;
        }
        ctx->part_spare = ctx->part;
        ctx->part = nullptr;
    }
    return IGS_OK;
}

void igs_partition_release(igs_ctx* ctx) {
    igs_partition_free(ctx);
    if (ctx->part_spare) {
        free_dev(ctx->part_spare);
        delete ctx->part_spare;
        ctx->part_spare = nullptr;
    }
}

extern "C" {

// bsp.cpp:153-176 build_partition
int igs_partition_build(igs_ctx* ctx, int n_max) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (ctx->n == 0) return igs_fail(ctx, IGS_E_EMPTY_SET, "build_partition requires a non-empty GaussianSet");
    if (n_max < 1) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "n_max must be >= 1");
    auto* p = new_partition(ctx);
    p->tree = true;
    p->n_max = n_max;
    p->source_size = ctx->n;
    int e = build_tree_device(ctx, p, n_max);
    if (e) {
        free_dev(p);
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
    auto* p = new_partition(ctx);
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

// ---- the whole BspPartition (bsp.hpp:44-66) for the C++ drop-in ----------------
int igs_partition_export(igs_ctx* ctx, int* n_max, uint32_t* source_size, int32_t* root, uint32_t* n_nodes,
                         int* grid_dim, uint32_t* grid_total) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    const PartitionDev* p = ctx->part;
    if (n_max) *n_max = p->n_max;
    if (source_size) *source_size = p->source_size;
    if (root) *root = p->tree ? p->root : -1;
    if (n_nodes) *n_nodes = p->tree ? (uint32_t)p->nodes.size() : 0u;
    if (grid_dim) *grid_dim = p->tree ? 0 : p->grid_dim;
    if (grid_total) *grid_total = p->tree ? 0u : (uint32_t)p->grid_blk_h.size();
    return IGS_OK;
}

int igs_partition_get_tree(igs_ctx* ctx, int32_t* nodes4, double* lines) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    const PartitionDev* p = ctx->part;
    if (!p->tree) return IGS_OK;
    for (size_t i = 0; i < p->nodes.size(); ++i) {
        const NodeD& nd = p->nodes[i];
        if (nodes4) {
            nodes4[4 * i] = nd.axis;
            nodes4[4 * i + 1] = nd.low;
            nodes4[4 * i + 2] = nd.high;
            nodes4[4 * i + 3] = nd.block;
        }
        if (lines) lines[i] = nd.line;
    }
    return IGS_OK;
}

int igs_partition_get_grid(igs_ctx* ctx, uint32_t* cell_offsets, uint32_t* cell_blocks) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    const PartitionDev* p = ctx->part;
    if (p->tree) return IGS_OK;
    if (cell_offsets) std::memcpy(cell_offsets, p->grid_off_h.data(), p->grid_off_h.size() * 4);
    if (cell_blocks && !p->grid_blk_h.empty())
        std::memcpy(cell_blocks, p->grid_blk_h.data(), p->grid_blk_h.size() * 4);
    return IGS_OK;
}

// block_members: the split's leaf lists for a built partition (bsp.cpp:32-40),
// locate_block of every resident centre for a rebuilt one (bsp.cpp:208-211);
// ascending within each block
int igs_partition_block_members(igs_ctx* ctx, uint32_t* offsets, uint32_t* members) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (!ctx->part) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "no partition");
    PartitionDev* p = ctx->part;
    const uint32_t n = p->source_size;
    std::vector<int32_t> blk(n);
    if (p->tree && !p->leaf_block.empty() && p->d_leaf_of) {
        std::vector<uint32_t> leaf(n);
        IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (n) IGS_CUDA(ctx, cudaMemcpy(leaf.data(), p->d_leaf_of, (size_t)n * 4, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < n; ++i) blk[i] = p->leaf_block[leaf[i]];
    } else {
        if (n != ctx->n) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "stale partition: Gaussian count changed since construction");
        std::vector<double> uv((size_t)n * 2);
        std::vector<double> scan6((size_t)n * 6);
        int e;
        if ((e = igs_get_prepared(ctx, scan6.data(), n))) return e;
        for (uint32_t i = 0; i < n; ++i) {
            uv[2 * (size_t)i] = scan6[6 * (size_t)i];
            uv[2 * (size_t)i + 1] = scan6[6 * (size_t)i + 1];
        }
        if ((e = igs_locate_blocks(ctx, uv.data(), n, blk.data()))) return e;
    }
    std::vector<uint32_t> off(p->nb + 1, 0);
    for (uint32_t i = 0; i < n; ++i) ++off[blk[i] + 1];
    for (uint32_t b = 0; b < p->nb; ++b) off[b + 1] += off[b];
    if (offsets) std::memcpy(offsets, off.data(), off.size() * 4);
    if (members) {
        std::vector<uint32_t> cur(off.begin(), off.end() - 1);
        for (uint32_t i = 0; i < n; ++i) members[cur[blk[i]]++] = i;
    }
    return IGS_OK;
}

// installs a caller-held partition (a BspPartition from the reference or from
// igs_partition_export): blocks + the split tree (n_nodes > 0) or, without a
// tree, the grid locator; shells and shell members are re-derived from the
// resident set (the rectangle test both builders apply)
int igs_partition_set(igs_ctx* ctx, const double* blocks4, uint32_t n_blocks, const int32_t* nodes4,
                      const double* lines, uint32_t n_nodes, int32_t root, int n_max, uint32_t source_size) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (n_blocks == 0 || !blocks4) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "partition has no blocks");
    if (n_nodes && (!nodes4 || !lines || root < 0 || (uint32_t)root >= n_nodes))
        return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bad partition tree");
    for (uint32_t i = 0; i < n_nodes; ++i) {
        const int32_t lo = nodes4[4 * i + 1], hi = nodes4[4 * i + 2], b = nodes4[4 * i + 3];
        const bool leaf_ok = b >= 0 && (uint32_t)b < n_blocks;
        const bool inner_ok = b < 0 && lo >= 0 && hi >= 0 && (uint32_t)lo < n_nodes && (uint32_t)hi < n_nodes;
        if (!leaf_ok && !inner_ok) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bad partition tree");
    }
    auto* p = new_partition(ctx);
    p->tree = n_nodes > 0;
    p->n_max = n_max;
    p->source_size = source_size;
    p->blocks.resize(n_blocks);
    std::memcpy(p->blocks.data(), blocks4, sizeof(RectD) * n_blocks);
    p->nodes.resize(n_nodes);
    for (uint32_t i = 0; i < n_nodes; ++i)
        p->nodes[i] = NodeD{nodes4[4 * i], lines[i], nodes4[4 * i + 1], nodes4[4 * i + 2], nodes4[4 * i + 3]};
    p->root = p->tree ? root : -1;
    igs_partition_free(ctx);
    ctx->part = p;
    const int e = finish_partition(ctx, p);
    if (e) igs_partition_free(ctx);
    return e;
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
