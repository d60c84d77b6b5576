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
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "igs_internal.cuh"
#include "knn_tree.cuh"
#include "reduce.cuh"
#include "scan.cuh"

using namespace igs_dev;

namespace {

constexpr int kQueue = 512;  // per-warp frontier capacity
constexpr int kSeedRMax = 8;  // widest seed window at the finest level: 17 x 17 cells

// cell it (0 <= it < 8R) of the square ring at Chebyshev radius R
__device__ __forceinline__ int ring_dx(int it, int R) {
    const int side = it / (2 * R), t = it % (2 * R);
    return side == 0 ? -R + t : (side == 1 ? R : (side == 2 ? R - t : -R));
}
__device__ __forceinline__ int ring_dy(int it, int R) {
    const int side = it / (2 * R), t = it % (2 * R);
    return side == 0 ? -R : (side == 1 ? -R + t : (side == 2 ? R : R - t));
}
// Builds between full re-bucketings (in between, the summaries are refit
// from the member-ordered records the Adam kernels keep current; exact either way, only the tightness
// of the bounds drifts as Gaussians move and change scale).
#ifndef IGS_REFIT_PERIOD
#define IGS_REFIT_PERIOD 16
#endif
#ifndef IGS_GROW_SHIFT
#define IGS_GROW_SHIFT 3
#endif
constexpr int kRefitPeriod = IGS_REFIT_PERIOD;
constexpr int kGrowShift = IGS_GROW_SHIFT;  // re-bucket when more than n >> kGrowShift Gaussians grew

// 32 bytes (one sector).  The bbox is rounded outward and lambda_min down
// to float: a box that contains the true one and a smaller eigenvalue only
// lower the (monotonically evaluated) bound, so it stays certified.
struct __align__(32) Sum {
    float x0, y0, x1, y1;  // centre bbox, rounded outward (empty: +inf/-inf)
    float lmin;            // smallest Sigma^-1 eigenvalue, rounded down
    float slack;           // bound safety factor (0 = never prune)
    uint32_t count;
    uint32_t pad;
};



__device__ __forceinline__ float slack_for(double aniso) {
    const double s = 1.0 - (9.5367431640625e-07 + 256.0 * 1.1102230246251565e-16 * (1.0 + aniso));
    return s > 0.5 ? (float)(s - 1e-7) : 0.0f;
}



__global__ void lq_count(const ScanRec* __restrict__ scan, uint32_t n, Lq L, uint32_t* __restrict__ cnt,
                         uint32_t* __restrict__ key, uint32_t* __restrict__ lcount) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    int l = -1;
    if (i < n) {
        const ScanRec r = scan[i];
        l = level_of(L, fmin(r.inv_a, r.inv_b));
        const int G = L.lw[l];
        const uint32_t k = (uint32_t)(L.loff[l] + cell_of(r.mu_y, G) * G + cell_of(r.mu_x, G));
        key[i] = k | ((uint32_t)l << kKeyLevelShift);
        atomicAdd(cnt + k, 1u);
    }
    // per-level population, warp-aggregated (13 addresses would serialise)
    const unsigned same = __match_any_sync(0xffffffffu, l);
    if (l >= 0 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(lcount + l, (unsigned)__popc(same));
}


// One launch clears everything a build accumulates into.
__global__ void lq_clear(uint32_t cells, uint32_t* __restrict__ cnt2, Acc* __restrict__ acc,
                         uint32_t* __restrict__ lcount) {
    pdl_wait();
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x) {
        cnt2[c] = 0;
        cnt2[cells + c] = 0;
        acc[c] = acc_empty();
        if (c < kMaxLv) lcount[c] = 0;
    }
}

__global__ void lq_fill(const ScanRec* __restrict__ scan, uint32_t n, const uint32_t* __restrict__ key,
                        const uint32_t* __restrict__ off, uint32_t* __restrict__ cur, uint32_t* __restrict__ mem,
                        ScanRec* __restrict__ mrec, uint32_t* __restrict__ minv, uint32_t* __restrict__ mcell,
                        Acc* __restrict__ acc) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = key[i] & kKeyCellMask;
    const uint32_t pos = off[k] + atomicAdd(cur + k, 1u);
    const ScanRec r = scan[i];
    mem[pos] = i;
    mrec[pos] = r;  // the records in member order (the searches' evaluation stream)
    minv[i] = pos;
    mcell[pos] = k;
}

// A full re-bucketing in one persistent launch (one CTA per SM, all
// co-resident; grid barriers as offsets_scatter_kernel): clear -> level,
// cell and count per Gaussian (lq_count) -> cell offsets (exclusive scan:
// chunk totals, barrier, chunk base + block scan) -> member lists, the
// member-ordered records and the accumulators (lq_fill).  The summaries
// follow in lq_tree_kernel.  bar[0] arrivals, bar[1] exits, then the chunk
// totals; the last CTA out resets the counters.
constexpr int kBuildThreads = 256;
constexpr int kBuildPer = 4;  // cell counts per thread and scan pass

__global__ void __launch_bounds__(kBuildThreads) lq_build_kernel(
    const ScanRec* __restrict__ scan, uint32_t n, Lq L, uint32_t cells, uint32_t* __restrict__ cnt,
    uint32_t* __restrict__ cur, uint32_t* __restrict__ off, uint32_t* __restrict__ key, uint32_t* __restrict__ mem,
    ScanRec* __restrict__ mrec, uint32_t* __restrict__ minv, uint32_t* __restrict__ mcell, Acc* __restrict__ acc,
    uint32_t* __restrict__ lcount, unsigned* __restrict__ bar) {
    __shared__ uint32_t s_base;
    uint32_t* chunk_sum = bar + 2;
    pdl_wait();
    const uint32_t G = gridDim.x, tid = blockIdx.x * kBuildThreads + threadIdx.x, nth = G * kBuildThreads;
    // 1. clear
    for (uint32_t c = tid; c < cells; c += nth) {
        cnt[c] = 0;
        cur[c] = 0;
        acc[c] = acc_empty();
    }
    if (tid < kMaxLv) lcount[tid] = 0;
    igs_grid_sync(bar, G);
    // 2. level, cell and count (lq_count)
    for (uint32_t base = blockIdx.x * kBuildThreads; base < n; base += nth) {
        const uint32_t i = base + threadIdx.x;
        int l = -1;
        if (i < n) {
            const ScanRec r = scan[i];
            l = level_of(L, fmin(r.inv_a, r.inv_b));
            const int Gl = L.lw[l];
            const uint32_t k = (uint32_t)(L.loff[l] + cell_of(r.mu_y, Gl) * Gl + cell_of(r.mu_x, Gl));
            key[i] = k | ((uint32_t)l << kKeyLevelShift);
            atomicAdd(cnt + k, 1u);
        }
        const unsigned same = __match_any_sync(0xffffffffu, l);
        if (l >= 0 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(lcount + l, (unsigned)__popc(same));
    }
    igs_grid_sync(bar, 2 * G);
    // 3. cell offsets: chunk totals, barrier, chunk base + block scan
    const uint32_t tile = kBuildThreads * kBuildPer;
    const uint32_t per_cta = ((cells + G - 1) / G + tile - 1) / tile * tile;
    const uint32_t c0 = blockIdx.x * per_cta, c1 = min(cells, c0 + per_cta);
    uint32_t total = 0;
    for (uint32_t b = c0; b < c1; b += tile)
#pragma unroll
        for (int j = 0; j < kBuildPer; ++j) {
            const uint32_t c = b + threadIdx.x * kBuildPer + j;
            if (c < c1) total += __ldcg(cnt + c);
        }
    {
        uint32_t agg;
        block_excl_sum<kBuildThreads>(total, &agg);
        if (threadIdx.x == 0) chunk_sum[blockIdx.x] = agg;
    }
    igs_grid_sync(bar, 3 * G);
    uint32_t mine = 0;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += kBuildThreads) mine += __ldcg(chunk_sum + b);
    {
        uint32_t base;
        block_excl_sum<kBuildThreads>(mine, &base);
        if (threadIdx.x == 0) s_base = base;
    }
    __syncthreads();
    uint32_t run = s_base;
    for (uint32_t b = c0; b < c1; b += tile) {
        uint32_t v[kBuildPer], sum = 0;
#pragma unroll
        for (int j = 0; j < kBuildPer; ++j) {
            const uint32_t c = b + threadIdx.x * kBuildPer + j;
            v[j] = c < c1 ? __ldcg(cnt + c) : 0u;
            sum += v[j];
        }
        uint32_t agg;
        const uint32_t excl = block_excl_sum<kBuildThreads>(sum, &agg);
        uint32_t o = run + excl;
#pragma unroll
        for (int j = 0; j < kBuildPer; ++j) {
            const uint32_t c = b + threadIdx.x * kBuildPer + j;
            if (c < c1) off[c] = o;
            o += v[j];
        }
        run += agg;
    }
    igs_grid_sync(bar, 4 * G);
    // 4. member lists, member-ordered records, accumulators (lq_fill)
    for (uint32_t i = tid; i < n; i += nth) {
        const uint32_t k = key[i] & kKeyCellMask;  // (this thread wrote key[i] in step 2)
        const uint32_t pos = __ldcg(off + k) + atomicAdd(cur + k, 1u);
        const ScanRec r = scan[i];
        mem[pos] = i;
        mrec[pos] = r;
        minv[i] = pos;
        mcell[pos] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(bar + 1, 1u) == G - 1) {
        bar[0] = 0;
        bar[1] = 0;
    }
}

__device__ __forceinline__ Sum empty_sum() {
    const float inf = __int_as_float(0x7f800000);
    Sum s;
    s.x0 = inf; s.y0 = inf; s.x1 = -inf; s.y1 = -inf;
    s.lmin = inf;
    s.slack = 1.0f;
    s.count = 0;
    s.pad = 0;
    return s;
}

__device__ __forceinline__ void merge(Sum& a, const Sum& b) {
    if (b.count == 0) return;
    a.x0 = fminf(a.x0, b.x0); a.x1 = fmaxf(a.x1, b.x1);
    a.y0 = fminf(a.y0, b.y0); a.y1 = fmaxf(a.y1, b.y1);
    a.lmin = fminf(a.lmin, b.lmin);
    a.slack = fminf(a.slack, b.slack);
    a.count += b.count;
}

// Own summary of cell c from its accumulator (written by another CTA of
// lq_tree_kernel).
__device__ __forceinline__ Sum own_of(Acc* __restrict__ acc, const uint32_t* __restrict__ cnt, uint32_t c) {
    Sum s = empty_sum();
    const uint32_t m = cnt[c];
    if (m == 0) return s;
    const Acc a = acc_ldcg(acc + c);  // (written by another CTA)
    s.x0 = odec(a.x0);
    s.y0 = odec(a.y0);
    s.x1 = odec(a.x1);
    s.y1 = odec(a.y1);
    s.lmin = odec(a.lmin);
    s.slack = slack_for((double)odec(a.aniso));
    s.count = m;
    return s;
}

// All own + subtree summaries in one launch, from the member-ordered
// records (mrec, kept current by the Adam launches) -- no per-Gaussian
// atomics anywhere.  CTA (bx, by) owns a 16 x 16 block of level-0 cells and
// levels 0..4 above it (341 cells, 31 rows of cells).  A row's members are
// one contiguous range of mrec (members are ordered by cell), so the CTA
// walks the concatenation of its 31 ranges, one member per thread: each
// warp min/max-reduces its runs of equal cells with shuffles (min/max are
// idempotent, so overlapping windows are harmless) and the first lane of a
// run folds it into the cell's shared-memory accumulator (shared atomics:
// runs can span warps).  Then the summaries level by level (subtree = own +
// the four children).  The members of the levels above 4 (large Gaussians)
// are split evenly over all CTAs and folded into global accumulators the
// same way; the last CTA to finish (atomic ticket after a fence) reads them
// (resetting them for the next launch) and builds the levels above.
constexpr int kBlk = 16;
constexpr int kInLv = 5;       // levels 0..4 live inside a block
constexpr int kTileRows = 31;  // 16 + 8 + 4 + 2 + 1
constexpr int kTileCells = 341;
constexpr int kUpCells = 341;  // 16^2 + 8^2 + 4^2 + 2^2 + 1: upper levels kept in shared memory
#ifndef IGS_KWALK
#define IGS_KWALK 1
#endif
constexpr int kWalk = IGS_KWALK;  // member-walk loads in flight per thread
#ifndef IGS_TREE_THREADS
#define IGS_TREE_THREADS 256
#endif
constexpr int kTreeThreads = IGS_TREE_THREADS;  // >= 256 (the level-0 block)
// Sets up to this size refit with 512-thread CTAs: twice the threads on a
// tile's member walk, which evens out tiles of very different populations
// (trained sets: refit 24.2 -> 22.6 us at C2 t = 5,000, fit start equal);
// larger sets keep 256 (C4: 100 -> 147 us at 512, fewer CTAs per SM).
constexpr uint32_t kTreeWideMaxN = 400000;

// own summary from (count, accumulator)
__device__ __forceinline__ Sum own_from(uint32_t m, const Acc& a) {
    Sum s = empty_sum();
    if (m == 0) return s;
    s.x0 = odec(a.x0);
    s.y0 = odec(a.y0);
    s.x1 = odec(a.x1);
    s.y1 = odec(a.y1);
    s.lmin = odec(a.lmin);
    s.slack = slack_for((double)odec(a.aniso));
    s.count = m;
    return s;
}

// Warp step of the member walk: lane holds (key, a) -- key ~0u for no
// member; runs of equal keys are contiguous.  Returns true in the first
// lane of each run, whose a then covers the whole run within the warp.
__device__ __forceinline__ bool warp_runs(uint32_t key, Acc& a) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yk = __shfl_down_sync(0xffffffffu, key, o);
        const unsigned x0 = __shfl_down_sync(0xffffffffu, a.x0, o), y0 = __shfl_down_sync(0xffffffffu, a.y0, o);
        const unsigned x1 = __shfl_down_sync(0xffffffffu, a.x1, o), y1 = __shfl_down_sync(0xffffffffu, a.y1, o);
        const unsigned lm = __shfl_down_sync(0xffffffffu, a.lmin, o);
        const unsigned an = __shfl_down_sync(0xffffffffu, a.aniso, o);
        if (lane + o < 32 && yk == key) {
            a.x0 = min(a.x0, x0);
            a.y0 = min(a.y0, y0);
            a.x1 = max(a.x1, x1);
            a.y1 = max(a.y1, y1);
            a.lmin = min(a.lmin, lm);
            a.aniso = max(a.aniso, an);
        }
    }
    const uint32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
    return key != ~0u && (lane == 0 || pk != key);
}

__device__ __forceinline__ void acc_fold(Acc* d, const Acc& a) {
    atomicMin(&d->x0, a.x0);
    atomicMin(&d->y0, a.y0);
    atomicMax(&d->x1, a.x1);
    atomicMax(&d->y1, a.y1);
    atomicMin(&d->lmin, a.lmin);
    atomicMax(&d->aniso, a.aniso);
}

template <int NT>
__global__ void __launch_bounds__(NT) lq_tree_kernel(const ScanRec* __restrict__ mrec,
                                                      const uint32_t* __restrict__ mcell,
                                                      const uint32_t* __restrict__ off, uint32_t n,
                                                      Acc* __restrict__ acc, Lq L,
                                                      const uint32_t* __restrict__ cnt, Sum* __restrict__ own,
                                                      Sum* __restrict__ sub, unsigned int* __restrict__ ticket,
                                                      L2Prefetch pf, StageJob job, int full) {
    __shared__ Sum sm[2][kBlk * kBlk];
    __shared__ Sum up[kUpCells];
    __shared__ Acc s_acc[kTileCells];
    __shared__ int s_loff[kMaxLv];
    // per tile row: first cell, first member, local index of the first cell,
    // and the row's start in the concatenated walk (s_v0[kTileRows] = total)
    __shared__ uint32_t s_c0[kTileRows], s_p0[kTileRows], s_l0[kTileRows], s_v0[kTileRows + 1];
    const int t = threadIdx.x;
    if (t == 0) {
#pragma unroll
        for (int l = 0; l < kMaxLv; ++l) s_loff[l] = L.loff[l];
    }
    for (int i = t; i < kTileCells; i += NT) s_acc[i] = acc_empty();
    __syncthreads();
    const int nb = L.G0 / kBlk;  // G0 is a power of two >= 16
    const int bx = blockIdx.x % nb, by = blockIdx.x / nb;
    pdl_wait();
    stage_job_run(job, blockIdx.x * NT + t, gridDim.x * NT);  // the iteration's start (StageJob)
    prefetch_l2(pf, blockIdx.x * NT + t, gridDim.x * NT);  // the search's inputs
    // the counts of the cells this thread owns at each in-block level, and
    // (threads < 31) one row's member range -- one round trip
    uint32_t cell[kInLv], m[kInLv];
#pragma unroll
    for (int l = 0; l < kInLv; ++l) {
        const int side = kBlk >> l, G = L.G0 >> l;
        cell[l] = ~0u;
        m[l] = 0;
        if (t < side * side) {
            const int x = bx * side + t % side, y = by * side + t / side;
            cell[l] = (uint32_t)(L.loff[l] + y * G + x);
            m[l] = cnt[cell[l]];
        }
    }
    uint32_t rlen = 0;
    if (t < kTileRows) {
        int l = 0, r = t, lbase = 0;
        while (r >= (kBlk >> l)) {
            r -= kBlk >> l;
            lbase += (kBlk >> l) * (kBlk >> l);
            ++l;
        }
        const int side = kBlk >> l, G = L.G0 >> l;
        const uint32_t c0 = (uint32_t)(s_loff[l] + (by * side + r) * G + bx * side), c1 = c0 + side - 1;
        const uint32_t p0 = off[c0];
        rlen = off[c1] + cnt[c1] - p0;
        s_c0[t] = c0;
        s_p0[t] = p0;
        s_l0[t] = (uint32_t)(lbase + r * side);
    }
    if (t < 32) {  // exclusive scan of the row lengths (warp 0)
        uint32_t x = rlen;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (t >= o) x += y;
        }
        if (t <= kTileRows) s_v0[t] = x - rlen;  // (t == kTileRows: rlen 0, the total)
    }
    __syncthreads();
    // the members, one per thread, kWalk batches of loads in flight (whole
    // warps iterate alike)
    const uint32_t total = s_v0[kTileRows];
    for (uint32_t vb = 0; vb < total; vb += NT * kWalk) {
        uint32_t key[kWalk];
        Acc a[kWalk];
#pragma unroll
        for (int u = 0; u < kWalk; ++u) {
            const uint32_t v = vb + NT * u + t;
            key[u] = ~0u;
            a[u] = acc_empty();
            if (v < total) {
                int r = 0;  // the row holding walk position v (last start <= v)
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (r + step < kTileRows && s_v0[r + step] <= v) r += step;
                const uint32_t p = s_p0[r] + (v - s_v0[r]);
                key[u] = s_l0[r] + (mcell[p] - s_c0[r]);
                acc_add_local(a[u], mrec[p]);
            }
        }
#pragma unroll
        for (int u = 0; u < kWalk; ++u)
            if (vb + NT * u < total && warp_runs(key[u], a[u])) acc_fold(&s_acc[key[u]], a[u]);
    }
    __syncthreads();
    int cur = 0, lbase = 0;
#pragma unroll
    for (int l = 0; l < kInLv; ++l) {
        const int side = kBlk >> l;
        if (t < side * side) {
            // a cell with no members, or a subtree with none, stays empty
            // between builds (membership only changes at a build): after the
            // build's full pass a refit writes only the others
            const Sum o = own_from(m[l], s_acc[lbase + t]);
            if (full || m[l]) own[cell[l]] = o;
            Sum s = o;
            if (l > 0) {
                const int cs = side * 2;
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx) merge(s, sm[cur][(2 * (t / side) + dy) * cs + 2 * (t % side) + dx]);
            }
            if (full || s.count) sub[cell[l]] = s;
            sm[cur ^ 1][t] = s;
        }
        __syncthreads();
        cur ^= 1;
        lbase += side * side;
    }
    if (L.levels <= kInLv) return;  // (exit: counts as the launch trigger)
    // the cells of the levels above (large Gaussians; few cells, possibly
    // many members each): cell by cell over the CTAs, each cell's members
    // reduced by the whole CTA into its global accumulator (plain store)
    {
        __shared__ Acc s_wacc[NT / 32];
        const uint32_t cu0 = (uint32_t)s_loff[kInLv], cu1 = (uint32_t)s_loff[L.levels - 1] + 1;
        for (uint32_t c = cu0 + blockIdx.x; c < cu1; c += gridDim.x) {
            const uint32_t mc = cnt[c];
            if (mc == 0) continue;  // (uniform)
            const uint32_t p0 = off[c];
            Acc a = acc_empty();
            for (uint32_t e = t; e < mc; e += NT) acc_add_local(a, mrec[p0 + e]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a.x0 = min(a.x0, __shfl_xor_sync(0xffffffffu, a.x0, o));
                a.y0 = min(a.y0, __shfl_xor_sync(0xffffffffu, a.y0, o));
                a.x1 = max(a.x1, __shfl_xor_sync(0xffffffffu, a.x1, o));
                a.y1 = max(a.y1, __shfl_xor_sync(0xffffffffu, a.y1, o));
                a.lmin = min(a.lmin, __shfl_xor_sync(0xffffffffu, a.lmin, o));
                a.aniso = max(a.aniso, __shfl_xor_sync(0xffffffffu, a.aniso, o));
            }
            if ((t & 31) == 0) s_wacc[t >> 5] = a;
            __syncthreads();
            if (t == 0) {
                for (int w = 1; w < NT / 32; ++w) {
                    const Acc& b = s_wacc[w];
                    a.x0 = min(a.x0, b.x0);
                    a.y0 = min(a.y0, b.y0);
                    a.x1 = max(a.x1, b.x1);
                    a.y1 = max(a.y1, b.y1);
                    a.lmin = min(a.lmin, b.lmin);
                    a.aniso = max(a.aniso, b.aniso);
                }
                acc[c] = a;
            }
            __syncthreads();
        }
    }
    // upper levels: the first level from which every level fits in shared
    // memory (<= 16 x 16 cells), and the cells from there to the root
    int l0 = kInLv;
    while (l0 < L.levels && (L.G0 >> l0) > kBlk) ++l0;
    int ncell = 0;
    for (int j = l0; j < L.levels; ++j) ncell += (L.G0 >> j) * (L.G0 >> j);
    // speculative prefetch (every CTA; L2 hits after the first): the counts
    // of the shared-memory levels, so the last CTA does not wait for them
    uint32_t um[2] = {0, 0}, uc[2] = {0, 0};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int i = t + NT * r;
        if (i < ncell) {
            uc[r] = (uint32_t)(s_loff[l0] + i);  // levels are contiguous in the cell numbering
            um[r] = cnt[uc[r]];
        }
    }
    __shared__ bool last;
    // the block's stores are ordered before thread 0's fence by the barrier
    // (the cooperative-groups grid-barrier pattern): one fence per block
    __syncthreads();
    if (t == 0) {
        pdl_trigger();  // only the last CTA's upper levels remain
        __threadfence();
        last = atomicAdd(ticket, 1u) == (unsigned)(nb * nb - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // upper levels too large for shared memory (G0 >= 1024): level by level
    // through global memory
    for (int l = kInLv; l < l0; ++l) {
        const int G = L.G0 >> l, cw = G * 2;
        for (int i = t; i < G * G; i += NT) {
            const int x = i % G, y = i / G;
            const uint32_t c = (uint32_t)(s_loff[l] + i);
            Sum s = own_of(acc, cnt, c);
            own[c] = s;
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) merge(s, sub[s_loff[l - 1] + (2 * y + dy) * cw + 2 * x + dx]);
            sub[c] = s;
        }
        __threadfence();
        __syncthreads();
    }
    // the shared-memory levels: own summaries from the accumulators,
    // children of level l0 from global memory, the rest merged in shared
    // memory
    {
        const int G = L.G0 >> l0, cw = G * 2;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int i = t + NT * r;
            if (i >= ncell) continue;
            const Acc ua = um[r] ? acc_ldcg(acc + uc[r]) : acc_empty();
            const Sum o = own_from(um[r], ua);
            own[uc[r]] = o;
            Sum s = o;
            if (i < G * G) {
                const int x = i % G, y = i / G;
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx) merge(s, sub[s_loff[l0 - 1] + (2 * y + dy) * cw + 2 * x + dx]);
                sub[uc[r]] = s;
            }
            up[i] = s;  // level l0: subtree; above: own (merged below)
        }
    }
    __syncthreads();
    for (int j = l0 + 1, b0 = 0; j < L.levels; ++j) {
        const int G = L.G0 >> j, cw = G * 2, b1 = b0 + cw * cw;  // b0: first cell of level j-1 in up[]
        for (int i = t; i < G * G; i += NT) {
            const int x = i % G, y = i / G;
            Sum s = up[b1 + i];
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) merge(s, up[b0 + (2 * y + dy) * cw + 2 * x + dx]);
            up[b1 + i] = s;
            sub[s_loff[j] + i] = s;
        }
        __syncthreads();
        b0 = b1;
    }
    if (t == 0) *ticket = 0;  // ready for the next build
}

// The query point as a float box [xl, xh] x [yl, yh] around (px, py), so
// the pruning bound below runs in fp32.
struct PtBox {
    float xl, xh, yl, yh;
};
__device__ __forceinline__ PtBox pt_box(double px, double py) {
    return PtBox{__double2float_rd(px), __double2float_ru(px), __double2float_rd(py), __double2float_ru(py)};
}

// Lower bound of q over a cell's members: lmin * dist(point, bbox)^2 * slack,
// in fp32 with every step rounded down and the point widened to its float
// box (so never above the exact bound) -- compared against the threshold
// rounded up (tqf).  slack 0
// (a degenerate member) never prunes; an empty cell always does.
__device__ __forceinline__ float sum_lb_f(const Sum& s, const PtBox& b) {
    if (s.count == 0) return __int_as_float(0x7f800000);
    if (!(s.slack > 0.0f)) return 0.0f;
    const float dx = fmaxf(fmaxf(__fsub_rd(s.x0, b.xh), __fsub_rd(b.xl, s.x1)), 0.0f);
    const float dy = fmaxf(fmaxf(__fsub_rd(s.y0, b.yh), __fsub_rd(b.yl, s.y1)), 0.0f);
    return __fmul_rd(__fmul_rd(s.lmin, __fadd_rd(__fmul_rd(dx, dx), __fmul_rd(dy, dy))), s.slack);
}


// Warp-distributed top-K: lane j holds the j-th best (q, idx) for j < kk,
// ascending in the strict (q, idx) order of select_top_k_entries
// (renderer.cpp:53-74); lanes >= kk hold the (inf, kNoIdx) sentinel.  The
// threshold (entry kk-1) is cached in every lane.  Insertion is
// warp-uniform: the first lane whose entry exceeds the candidate takes it
// and the tail shifts up one lane.
struct WarpTopK {
    double q;
    uint32_t i;
    double tq_;
    float tqf_;
    uint32_t ti;
    int kk, lane;

    __device__ __forceinline__ void init(int kk_, int lane_) {
        kk = kk_;
        lane = lane_;
        q = __longlong_as_double(0x7ff0000000000000LL);
        i = kNoIdx;
        tq_ = q;
        tqf_ = __int_as_float(0x7f800000);
        ti = kNoIdx;
    }
    __device__ __forceinline__ double tq() const { return tq_; }
    __device__ __forceinline__ float tqf() const { return tqf_; }  // tq rounded up (fp32 pruning)
    __device__ __forceinline__ bool beats(double cq, uint32_t ci) const {
        return cq < tq_ || (cq == tq_ && ci < ti);
    }
    // warp-uniform (cq, ci); no effect unless it beats the threshold
    __device__ __forceinline__ void offer(double cq, uint32_t ci) {
        if (!beats(cq, ci)) return;
        push(cq, ci);
        refresh();
    }
    // insertion without the threshold broadcast: a candidate that beats no
    // entry (ballot empty) is dropped, so a stale threshold only costs time;
    // call refresh() before tq()/beats() are used again
    __device__ __forceinline__ void push(double cq, uint32_t ci) {
        const bool gt = lane < kk && (cq < q || (cq == q && ci < i));
        const unsigned m = __ballot_sync(0xffffffffu, gt);
        if (m == 0) return;  // warp-uniform
        const int pos = __ffs(m) - 1;
        const double pq = __shfl_up_sync(0xffffffffu, q, 1);
        const uint32_t pi = __shfl_up_sync(0xffffffffu, i, 1);
        if (lane == pos) {
            q = cq;
            i = ci;
        } else if (lane > pos) {  // lanes >= kk never satisfy gt, so their ballot bit is clear
            q = pq;
            i = pi;
        }
    }
    __device__ __forceinline__ void refresh() {
        tq_ = __shfl_sync(0xffffffffu, q, kk - 1);
        tqf_ = __double2float_ru(tq_);
        ti = __shfl_sync(0xffffffffu, i, kk - 1);
    }
    static __device__ __forceinline__ bool lt(double aq, uint32_t ai, double bq, uint32_t bi) {
        return aq < bq || (aq == bq && ai < bi);
    }
    // compare-exchange with lane ^ j; keep_min: this lane keeps the smaller
    static __device__ __forceinline__ void cx(double& cq, uint32_t& ci, int j, bool keep_min) {
        const double oq = __shfl_xor_sync(0xffffffffu, cq, j);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, ci, j);
        if (lt(oq, oi, cq, ci) == keep_min) {
            cq = oq;
            ci = oi;
        }
    }
    // Many candidates at once (each lane one, (inf, kNoIdx) for none): a
    // bitonic sort of the batch, then the first step of a bitonic merge with
    // the kept list (elementwise min against the reversed batch leaves the
    // 32 smallest of the union as a bitonic sequence) and five half-cleaner
    // stages: lane j ends with the j-th smallest, the list's own layout.
    __device__ __forceinline__ void merge(double cq, uint32_t ci) {
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) cx(cq, ci, j, ((lane & j) == 0) == ((lane & k) == 0));
        const double rq = __shfl_sync(0xffffffffu, cq, 31 - lane);
        const uint32_t ri = __shfl_sync(0xffffffffu, ci, 31 - lane);
        double lq = lane < kk ? q : __longlong_as_double(0x7ff0000000000000LL);
        uint32_t li = lane < kk ? i : kNoIdx;
        if (lt(rq, ri, lq, li)) {
            lq = rq;
            li = ri;
        }
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) cx(lq, li, j, (lane & j) == 0);
        q = lq;
        i = li;
        refresh();
    }
};

constexpr int kMergeMin = 8;  // candidates per batch from which merge() beats sequential inserts

// Evaluates the members of up to 32 cells (lane i: range [o_i, o_i + m_i)),
// flattened so that all lanes work on members.
template <class TK>
__device__ __forceinline__ void eval_members(TK& t, uint32_t o_mine, uint32_t m_mine, int lane,
                                             const ScanRec* __restrict__ mrec, const uint32_t* __restrict__ mem,
                                             double px, double py, unsigned long long& evaluated) {
    if (__ballot_sync(0xffffffffu, m_mine != 0) == 0) return;  // nothing to evaluate (common)
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
            const uint32_t p = lo_o + (f - lo_ex);  // records in member order: no dependent gather
            gi = __ldg(mem + p);
            q = maha(mrec[p], px, py);
            cand = t.beats(q, gi);
        }
        unsigned msk = __ballot_sync(0xffffffffu, cand);
        if (__popc(msk) >= kMergeMin) {
            t.merge(cand ? q : __longlong_as_double(0x7ff0000000000000LL), cand ? gi : kNoIdx);
        } else if (msk) {
            do {
                const int src = __ffs(msk) - 1;
                msk &= msk - 1;
                const double qq = __shfl_sync(0xffffffffu, q, src);
                const uint32_t ii = __shfl_sync(0xffffffffu, gi, src);
                t.push(qq, ii);
            } while (msk);
            t.refresh();
        }
    }
}


// One warp per point.
constexpr uint32_t kHardCap = 256;

// What the warp does with its final top-K (lane j < kk holds entry j).
struct Epi {
    int mode;                    // 0 train (target L1), 1 backward (given upstream), 2 query (top-K out)
    const uint32_t* sidx;        // mode 0: flat target pixel per point
    const float* target;         // mode 0
    const double* samples5;      // mode 1: upstream in columns 2..4
    double inv_n;                // mode 0: 1 / (total samples over all ranks)
    const ShadeRec* shade;
    double* losses;              // mode 0: per point
    double* host_losses;         // mode 0: host-mapped copy of losses (the host sums them in sample order) or null
    double* contrib;             // modes 0/1: [pt][kk][8] (deterministic reduction) or null
    uint32_t* keys;              // modes 0/1: [pt][kk] Gaussian index, n for empty slots
    uint32_t* gcnt;              // modes 0/1 (deterministic): contributions per Gaussian
    uint32_t* bucket;            // with gcnt: [n][kBucket] slot ids by arrival (reduce.cuh), or null
    uint32_t* ovf;               // with bucket: [0] overflow entries, [2] long segments (reduce.cuh)
    uint32_t* ovf_list;          // with bucket: (slot, rank) of every overflow entry
    uint32_t* long_list;         // with bucket: the long segments' Gaussians
    uint32_t* ovf_zero;          // the next iteration's counters (3 words), zeroed at the start of the search
    double* grads_atomic;        // modes 0/1: fast mode (fp64 atomics) or null
    long long* status;           // status[2]: first non-finite loss
    double* oq;                  // mode 2
    uint32_t* oi;                // mode 2
    uint32_t n;
    uint32_t* zero_word;         // zeroed at the start of the search (or null)
    int defer_loss_check;        // multi-rank: the non-finite loss check runs on the gathered losses
    L2Prefetch pf;               // what the kernels after the search read (Adam's rows)
};

// Query point: the centre of target pixel sidx[pt] (mode 0; pixel_center,
// image.hpp:18-20 / fit.cpp:67-70), the sample's (u, v) (mode 1), or uv[pt].
__device__ __forceinline__ void point_of(const double* __restrict__ uv, const Epi& E, int W, int H, uint32_t pt,
                                         double& px, double& py) {
    if (E.mode == 0) {
        const int f = (int)E.sidx[pt];
        px = center(f % W, W);
        py = center(f / W, H);
    } else if (E.mode == 1) {
        px = E.samples5[(size_t)pt * 5];
        py = E.samples5[(size_t)pt * 5 + 1];
    } else {
        px = uv[2 * (size_t)pt];
        py = uv[2 * (size_t)pt + 1];
    }
}

__device__ __forceinline__ double sign_of(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// blend_entries (renderer.cpp:76-89) + the L1 loss / upstream (fit.cpp:67-80)
// + sample_gradients (renderer.cpp:91-122), one lane per selected entry.  The
// blend sums run in entry order through a shuffle chain so every lane holds
// the reference's exact sequential totals.
// WIDTH lanes per point (32, or 16 for two points per warp: the shuffles
// stay inside each half); an inactive group (no point, or one handed to the
// hard-point scan) joins the shuffles and writes nothing.
template <int WIDTH>
__device__ __forceinline__ void warp_epilogue(const Epi& E, const ScanRec* __restrict__ scan, uint32_t pt,
                                              bool active, int kk, int lane, double myq, uint32_t myi, double px,
                                              double py) {
    if (E.mode == 2) {
        if (active && lane < kk) {
            E.oq[(size_t)pt * kk + lane] = myq;
            E.oi[(size_t)pt * kk + lane] = myi;
        }
        return;
    }
    const bool live = active && lane < kk && myi != kNoIdx;
    double w = 0.0;
    ShadeRec h{};
    if (live) {
        w = glibc_math::exp(__dmul_rn(-0.5, myq));
        h = E.shade[myi];
    }
    double total = 0.0, ar = 0.0, ag = 0.0, ab = 0.0;
    for (int j = 0; j < kk; ++j) {
        const double wj = __shfl_sync(0xffffffffu, w, j, WIDTH);
        const double rj = __shfl_sync(0xffffffffu, h.r, j, WIDTH);
        const double gj = __shfl_sync(0xffffffffu, h.g, j, WIDTH);
        const double bj = __shfl_sync(0xffffffffu, h.b, j, WIDTH);
        if (__shfl_sync(0xffffffffu, live ? 1 : 0, j, WIDTH)) {
            total = __dadd_rn(total, wj);
            ar = __dadd_rn(ar, __dmul_rn(wj, rj));
            ag = __dadd_rn(ag, __dmul_rn(wj, gj));
            ab = __dadd_rn(ab, __dmul_rn(wj, bj));
        }
    }
    const double inv_denom = __ddiv_rn(1.0, __dadd_rn(kNormEps, total));
    const double c0 = __dmul_rn(ar, inv_denom), c1 = __dmul_rn(ag, inv_denom), c2 = __dmul_rn(ab, inv_denom);
    double up0, up1, up2;
    if (E.mode == 0) {
        float t0 = 0.0f, t1 = 0.0f, t2 = 0.0f;
        if (active) {
            const float* t = E.target + (size_t)E.sidx[pt] * 3;
            t0 = t[0];
            t1 = t[1];
            t2 = t[2];
        }
        const double d0 = __dsub_rn(c0, (double)t0);
        const double d1 = __dsub_rn(c1, (double)t1);
        const double d2 = __dsub_rn(c2, (double)t2);
        if (active && lane == 0) {
            const double l = __dadd_rn(__dadd_rn(fabs(d0), fabs(d1)), fabs(d2));
            E.losses[pt] = l;
            if (E.host_losses) E.host_losses[pt] = l;
            if (!isfinite(l) && !E.defer_loss_check) atomicMin(E.status + 2, (long long)pt);
        }
        up0 = __dmul_rn(sign_of(d0), E.inv_n);
        up1 = __dmul_rn(sign_of(d1), E.inv_n);
        up2 = __dmul_rn(sign_of(d2), E.inv_n);
    } else {
        if (!active) return;  // nothing below is warp-collective
        up0 = E.samples5[(size_t)pt * 5 + 2];
        up1 = E.samples5[(size_t)pt * 5 + 3];
        up2 = E.samples5[(size_t)pt * 5 + 4];
    }
    if (!active || lane >= kk) return;
    const size_t slot = (size_t)pt * kk + lane;
    if (!live) {
        if (E.keys) E.keys[slot] = E.n;  // sorts past every real index
        return;
    }
    const ScanRec g = scan[myi];
    const double dL_dw = __dmul_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(up0, __dsub_rn(h.r, c0)), __dmul_rn(up1, __dsub_rn(h.g, c1))),
                  __dmul_rn(up2, __dsub_rn(h.b, c2))),
        inv_denom);
    const double wc = __dmul_rn(w, inv_denom);
    const double dx = __dsub_rn(px, g.mu_x);
    const double dy = __dsub_rn(py, g.mu_y);
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
    if (E.grads_atomic) {
#pragma unroll
        for (int p = 0; p < 8; ++p) atomicAdd(E.grads_atomic + (size_t)myi * 8 + p, d[p]);
    } else {
        double2* o = reinterpret_cast<double2*>(E.contrib + slot * 8);
        o[0] = make_double2(d[0], d[1]);
        o[1] = make_double2(d[2], d[3]);
        o[2] = make_double2(d[4], d[5]);
        o[3] = make_double2(d[6], d[7]);
        E.keys[slot] = myi;
        if (E.gcnt) {
            const uint32_t pos = atomicAdd(E.gcnt + myi, 1u);
            if (E.bucket) {
                // overflow entries appended with one atomic per warp
                const unsigned act = __activemask();
                const unsigned over = __ballot_sync(act, pos >= kBucket);
                if (pos < kBucket) {
                    E.bucket[(size_t)myi * kBucket + pos] = (uint32_t)slot;
                } else {
                    const int leader = __ffs(over) - 1;
                    uint32_t q0 = 0;
                    if ((int)(threadIdx.x & 31) == leader) q0 = atomicAdd(E.ovf, (unsigned)__popc(over));
                    const uint32_t q = __shfl_sync(over, q0, leader) + __popc(over & ((1u << (threadIdx.x & 31)) - 1));
                    E.ovf_list[2 * q] = (uint32_t)slot;
                    E.ovf_list[2 * q + 1] = pos;
                    if (pos == kBucket) E.long_list[atomicAdd(E.ovf + 2, 1u)] = myi;
                }
            }
        }
    }
}

__global__ void __launch_bounds__(128, 9) knn_points_kernel(const ScanRec* __restrict__ scan, uint32_t n, Lq L,
                                                            const Sum* __restrict__ own, const Sum* __restrict__ sub,
                                                            const uint32_t* __restrict__ off,
                                                            const uint32_t* __restrict__ mem, const ScanRec* __restrict__ mrec,
                                                            const double* __restrict__ uv, int W, int H, uint32_t npts,
                                                            int kk, Epi E, unsigned long long* __restrict__ pairs,
                                                            uint32_t* __restrict__ hard_count,
                                                            uint32_t* __restrict__ hard_list,
                                                            unsigned long long* __restrict__ hard_stat,
                                                            uint32_t* __restrict__ next_point,
                                                            uint32_t* __restrict__ zero_next) {
    __shared__ uint32_t queue[4][2][kQueue];
    __shared__ int s_loff[kMaxLv];  // level tables (a dynamic index into the
    __shared__ int s_lg[kMaxLv];    // kernel parameters would go to local memory)
    if (threadIdx.x == 0) {
#pragma unroll
        for (int l = 0; l < kMaxLv; ++l) {
            s_loff[l] = L.loff[l];
            s_lg[l] = 31 - __clz(max(L.lw[l], 1));
        }
    }
    __syncthreads();
    pdl_wait();
    // the other counter pair (hard count, point cursor) and the caller's
    // word are zeroed for the next search: nothing reads them before it
    if (blockIdx.x == 0 && threadIdx.x < 2) zero_next[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 2 && E.zero_word) *E.zero_word = 0;
    if (blockIdx.x == 0 && threadIdx.x >= 3 && threadIdx.x < 6 && E.ovf_zero) E.ovf_zero[threadIdx.x - 3] = 0;
    prefetch_l2(E.pf, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // per-level population, one bit per level (same for every point)
    unsigned lvmask = 0;
    if (lane < L.levels && L.lcount[lane] > 0) lvmask = 1u;
    lvmask = __ballot_sync(0xffffffffu, lvmask);
    const int npop = __popc(lvmask);
    // lane j < npop: the j-th populated level (seed item it -> level of lane it / 9)
    const int my_pop = lane < npop ? __fns(lvmask, 0, lane + 1) : 0;
    const int lg0 = s_lg[0];
    // persistent warps: pull points until none are left (no wave tail).
    // Each warp's first point is its global warp index; later ones come from
    // the cursor (offset by the warp count), claimed one point ahead so the
    // atomic's latency overlaps the current point's search.
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    uint32_t claim = blockIdx.x * (blockDim.x >> 5) + warp;
    for (;;) {
    const uint32_t pt = __shfl_sync(0xffffffffu, claim, 0);
    if (pt >= npts) return;  // warp-uniform
    if (lane == 0) claim = nwarps + atomicAdd(next_point, 1u);
    double px, py;
    point_of(uv, E, W, H, pt, px, py);
    const PtBox pb = pt_box(px, py);
    WarpTopK t;
    t.init(kk, lane);
    unsigned long long evaluated = 0;

    // (1) seeds: the 3x3 cells around the point at every populated level.
    // Pass 0 evaluates the point's own cell at each level and the whole
    // window at the finest populated level (a tight threshold at once);
    // pass 1 evaluates the other window cells whose own bound survives it.
    const int lfine = __ffs(lvmask) - 1;
    // the point's cell at level 0; at level l it is (cx0 >> l, cy0 >> l)
    // (G_l = G0 >> l, so floor(v G_l) = floor(v G0) >> l)
    const int cx0 = cell_of(px, 1 << lg0), cy0 = cell_of(py, 1 << lg0);
    for (int pass = 0; pass < 2; ++pass) {
        // pass 0: the 9 finest-level cells, then the own cell at each other
        // populated level; pass 1: the 8 other window cells at those levels
        const int nitems = pass == 0 ? 8 + npop : 8 * (npop - 1);
        for (int base = 0; base < nitems; base += 32) {
            const int it = base + lane;
            int k, d;
            if (pass == 0) {
                k = it < 9 ? 0 : it - 8;
                d = it < 9 ? it : 4;
            } else {
                k = 1 + it / 8;
                d = it % 8 + (it % 8 >= 4);
            }
            const int l = __shfl_sync(0xffffffffu, my_pop, min(k, 31));
            uint32_t o = 0, m = 0;
            if (it < nitems) {
                const int lg = s_lg[l], G = 1 << lg;
                const int x = (cx0 >> l) + d % 3 - 1, y = (cy0 >> l) + d / 3 - 1;
                if (x >= 0 && x < G && y >= 0 && y < G) {
                    const uint32_t c = (uint32_t)(s_loff[l] + (y << lg) + x);
                    if (pass == 0) {
                        o = off[c];
                        m = own[c].count;
                    } else {
                        const Sum so = own[c];
                        if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                            o = off[c];
                            m = so.count;
                        }
                    }
                }
            }
            eval_members(t, o, m, lane, mrec, mem, px, py, evaluated);
        }
    }

    // (1b) fewer than kk candidates so far (sparse finest level): widen the
    // window at the finest populated level ring by ring, so the descent
    // starts with a finite threshold
    int R = 1;
    while (!(t.tq() < __longlong_as_double(0x7ff0000000000000LL)) && R < kSeedRMax) {
        ++R;
        const int lg = s_lg[lfine], G = 1 << lg, sx = cx0 >> lfine, sy = cy0 >> lfine;
        for (int b = 0; b < 8 * R; b += 32) {
            const int it = b + lane;
            uint32_t o = 0, m = 0;
            if (it < 8 * R) {
                const int x = sx + ring_dx(it, R), y = sy + ring_dy(it, R);
                if (x >= 0 && x < G && y >= 0 && y < G) {
                    const uint32_t c = (uint32_t)(s_loff[lfine] + (y << lg) + x);
                    o = off[c];
                    m = own[c].count;
                }
            }
            eval_members(t, o, m, lane, mrec, mem, px, py, evaluated);
        }
    }

    bool overflow = false;
    // (2) descent: evaluate own members of frontier nodes, expand children
    // (G_l = G0 >> l is a power of two, so the child grid is exactly 2x).
    // Flat start: the levels above ls (at most 4 x 4 cells, 21 in all) are
    // checked cell by cell -- own members whose own bound survives -- and
    // the frontier at ls (8 x 8) is every cell whose subtree bound does;
    // the same sets a descent from the root reaches (a subtree bound never
    // exceeds an ancestor's), without its chain of dependent loads.
    uint32_t* cur = queue[warp][0];
    uint32_t* nxt = queue[warp][1];
    const int ls = min(L.levels - 1, max(lg0 - 3, 0));
    {
        const uint32_t c0 = ls + 1 < L.levels ? (uint32_t)s_loff[ls + 1] : 0u;
        const uint32_t nup = ls + 1 < L.levels ? (uint32_t)(s_loff[L.levels - 1] + 1) - c0 : 0u;
        for (uint32_t b = 0; b < nup; b += 32) {
            const uint32_t c = c0 + b + lane;
            uint32_t o = 0, m = 0;
            if (b + lane < nup) {
                int l = ls + 1;
                while (l + 1 < L.levels && (uint32_t)s_loff[l + 1] <= c) ++l;
                const int lg = s_lg[l];
                const int node = (int)(c - (uint32_t)s_loff[l]);
                const int x = node & ((1 << lg) - 1), y = node >> lg;
                const int Rl = l == lfine ? R : 1;  // the seed window at this level
                if (abs(x - (cx0 >> l)) > Rl || abs(y - (cy0 >> l)) > Rl) {
                    const Sum so = own[c];
                    if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                        o = off[c];
                        m = so.count;
                    }
                }
            }
            eval_members(t, o, m, lane, mrec, mem, px, py, evaluated);
        }
    }
    // Each visited cell c: its subtree bound decides whether its children
    // are visited (and it joins the frontier), its own bound -- when c lies
    // outside the seed window at its level -- whether its own members are
    // evaluated, in the same pass (a pruned subtree prunes its own members:
    // own bound >= subtree bound).
    int ncur = 0;
    {
        const int lg = s_lg[ls], nls = 1 << (2 * lg);
        const uint32_t lo = (uint32_t)s_loff[ls];
        const int sx = cx0 >> ls, sy = cy0 >> ls, Rl = ls == lfine ? R : 1;
        for (int b = 0; b < nls; b += 32) {
            const int node = b + lane;
            bool keep = false;
            uint32_t o = 0, m = 0;
            if (node < nls) {
                keep = sum_lb_f(sub[lo + node], pb) <= t.tqf();
                const int x = node & ((1 << lg) - 1), y = node >> lg;
                if (keep && (abs(x - sx) > Rl || abs(y - sy) > Rl)) {
                    const Sum so = own[lo + node];
                    if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                        o = off[lo + node];
                        m = so.count;
                    }
                }
            }
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            const int pos = ncur + __popc(msk & ((1u << lane) - 1));
            if (keep) cur[pos] = (uint32_t)node;  // (at most 64 <= kQueue)
            ncur += __popc(msk);
            eval_members(t, o, m, lane, mrec, mem, px, py, evaluated);
        }
        __syncwarp();
    }
    for (int l = ls; l > 0 && ncur > 0; --l) {
        const int lg = s_lg[l];
        const int wmask = (1 << lg) - 1;
        const uint32_t clo = (uint32_t)s_loff[l - 1];
        const int clg = lg + 1;
        const int csx = cx0 >> (l - 1), csy = cy0 >> (l - 1);  // the children's seed window
        const int cR = l - 1 == lfine ? R : 1;
        int nnext = 0;
        for (int base = 0; base < ncur * 4; base += 32) {
            const int item = base + lane;
            bool keep = false;
            uint32_t child = 0, o = 0, m = 0;
            if (item < ncur * 4) {
                const uint32_t node = cur[item >> 2];
                const uint32_t x = node & (uint32_t)wmask, y = node >> lg;
                const uint32_t cx = 2 * x + (item & 1), cy = 2 * y + ((item >> 1) & 1);
                child = (cy << clg) + cx;
                keep = sum_lb_f(sub[clo + child], pb) <= t.tqf();
                if (keep && (abs((int)cx - csx) > cR || abs((int)cy - csy) > cR)) {
                    const Sum so = own[clo + child];
                    if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                        o = off[clo + child];
                        m = so.count;
                    }
                }
            }
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            const int pos = nnext + __popc(msk & ((1u << lane) - 1));
            if (keep && pos < kQueue) nxt[pos] = child;
            nnext += __popc(msk);
            eval_members(t, o, m, lane, mrec, mem, px, py, evaluated);
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
        if (lane == 0 && hard_stat) atomicAdd(hard_stat, 1ull);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot < kHardCap) {
            if (lane == 0) hard_list[slot] = pt;
            continue;
        }
        t.init(kk, lane);
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
    warp_epilogue<32>(E, scan, pt, true, kk, lane, t.q, t.i, px, py);
    }  // persistent loop
}

// ---------------------------------------------------------------------------
// Two points per warp (kk <= 16): each half-warp runs the search above for
// its own point in 16-lane batches.  Every loop runs the larger of the two
// halves' trip counts so the warp-wide votes and shuffles stay converged; a
// half with nothing left feeds no-ops ((inf, kNoIdx) candidates, empty
// cells).  Per point this halves the batch bookkeeping (votes, scans,
// shuffles, the epilogue's blend chain), and a batch merge sorts 16
// candidates instead of 32.  The selection is the same exact (q, idx) top-K.
constexpr int kQueue16 = 256;   // per-half frontier capacity
#ifndef IGS_MERGE_MIN16
#define IGS_MERGE_MIN16 4
#endif
constexpr int kMergeMin16 = IGS_MERGE_MIN16;  // candidates per half-batch from which merge() is used
#ifndef IGS_FLAT_START16
#define IGS_FLAT_START16 2
#endif
constexpr int kFlatStart16 = IGS_FLAT_START16;  // the descent starts flat at level lg0 - this (a 4^this-cell grid)

__device__ __forceinline__ unsigned half_bits(unsigned ballot) { return (ballot >> (threadIdx.x & 16)) & 0xffffu; }
__device__ __forceinline__ int other_half(int v) { return __shfl_xor_sync(0xffffffffu, v, 16); }

// WarpTopK on 16 lanes: lane hl < kk holds entry hl of its half's point
struct HalfTopK {
    double q;
    uint32_t i;
    double tq_;
    float tqf_;
    uint32_t ti;
    int kk, hl;

    __device__ __forceinline__ void init(int kk_, int hl_) {
        kk = kk_;
        hl = hl_;
        q = __longlong_as_double(0x7ff0000000000000LL);
        i = kNoIdx;
        tq_ = q;
        tqf_ = __int_as_float(0x7f800000);
        ti = kNoIdx;
    }
    __device__ __forceinline__ double tq() const { return tq_; }
    __device__ __forceinline__ float tqf() const { return tqf_; }  // tq rounded up (fp32 pruning)
    __device__ __forceinline__ bool beats(double cq, uint32_t ci) const {
        return cq < tq_ || (cq == tq_ && ci < ti);
    }
    // (cq, ci) uniform within the half; one that beats no entry (including
    // (inf, kNoIdx)) changes nothing; refresh() before tq()/beats()
    __device__ __forceinline__ void push(double cq, uint32_t ci) {
        const bool gt = hl < kk && (cq < q || (cq == q && ci < i));
        const unsigned m = half_bits(__ballot_sync(0xffffffffu, gt));
        const int pos = m ? __ffs(m) - 1 : 16;
        const double pq = __shfl_up_sync(0xffffffffu, q, 1, 16);
        const uint32_t pi = __shfl_up_sync(0xffffffffu, i, 1, 16);
        if (hl == pos) {
            q = cq;
            i = ci;
        } else if (hl > pos) {
            q = pq;
            i = pi;
        }
    }
    __device__ __forceinline__ void refresh() {
        tq_ = __shfl_sync(0xffffffffu, q, kk - 1, 16);
        tqf_ = __double2float_ru(tq_);
        ti = __shfl_sync(0xffffffffu, i, kk - 1, 16);
    }
    // a half-batch (one candidate per lane, (inf, kNoIdx) for none): bitonic
    // sort of 16, elementwise min against the reversed batch, four
    // half-cleaner stages (WarpTopK::merge on 16 lanes)
    __device__ __forceinline__ void merge(double cq, uint32_t ci) {
#pragma unroll
        for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) WarpTopK::cx(cq, ci, j, ((hl & j) == 0) == ((hl & k) == 0));
        const double rq = __shfl_sync(0xffffffffu, cq, 15 - hl, 16);
        const uint32_t ri = __shfl_sync(0xffffffffu, ci, 15 - hl, 16);
        double lq = hl < kk ? q : __longlong_as_double(0x7ff0000000000000LL);
        uint32_t li = hl < kk ? i : kNoIdx;
        if (WarpTopK::lt(rq, ri, lq, li)) {
            lq = rq;
            li = ri;
        }
#pragma unroll
        for (int j = 8; j > 0; j >>= 1) WarpTopK::cx(lq, li, j, (hl & j) == 0);
        q = lq;
        i = li;
        refresh();
    }
};

// eval_members on 16 lanes per point (lane hl: cell range [o, o + m))
__device__ __forceinline__ void eval_members16(HalfTopK& t, uint32_t o_mine, uint32_t m_mine, int hl,
                                               const ScanRec* __restrict__ mrec, const uint32_t* __restrict__ mem,
                                               double px, double py, unsigned long long& evaluated) {
    if (__ballot_sync(0xffffffffu, m_mine != 0) == 0) return;  // nothing in either half (common)
    uint32_t incl = m_mine;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d, 16);
        if (hl >= d) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 15, 16);
    const uint32_t excl = incl - m_mine;
    evaluated += total;
    const uint32_t tmax = max(total, (uint32_t)other_half((int)total));
    for (uint32_t base = 0; base < tmax; base += 16) {
        const uint32_t f = base + hl;
        int lo = 0;
#pragma unroll
        for (int step = 8; step > 0; step >>= 1) {
            const uint32_t ex = __shfl_sync(0xffffffffu, excl, lo + step, 16);
            if (ex <= f) lo += step;
        }
        const uint32_t lo_ex = __shfl_sync(0xffffffffu, excl, lo, 16);
        const uint32_t lo_o = __shfl_sync(0xffffffffu, o_mine, lo, 16);
        double q = __longlong_as_double(0x7ff0000000000000LL);
        uint32_t gi = kNoIdx;
        bool cand = false;
        if (f < total) {
            const uint32_t p = lo_o + (f - lo_ex);  // records in member order: no dependent gather
            gi = __ldg(mem + p);
            q = maha(mrec[p], px, py);
            cand = t.beats(q, gi);
        }
        unsigned mh = half_bits(__ballot_sync(0xffffffffu, cand));
        const int np = __popc(mh), npmax = max(np, other_half(np));
        if (npmax >= kMergeMin16) {
            t.merge(cand ? q : __longlong_as_double(0x7ff0000000000000LL), cand ? gi : kNoIdx);
        } else if (npmax) {
            for (int r = 0; r < npmax; ++r) {
                const int src = mh ? __ffs(mh) - 1 : 0;
                mh &= mh - 1;
                double qq = __shfl_sync(0xffffffffu, q, src, 16);
                uint32_t ii = __shfl_sync(0xffffffffu, gi, src, 16);
                if (r >= np) {
                    qq = __longlong_as_double(0x7ff0000000000000LL);
                    ii = kNoIdx;
                }
                t.push(qq, ii);
            }
            t.refresh();
        }
    }
}

#ifndef IGS_KNN16_MINB
#define IGS_KNN16_MINB 9
#endif
__global__ void __launch_bounds__(128, IGS_KNN16_MINB) knn_points16_kernel(const ScanRec* __restrict__ scan, uint32_t n, Lq L,
                                                              const Sum* __restrict__ own,
                                                              const Sum* __restrict__ sub,
                                                              const uint32_t* __restrict__ off,
                                                              const uint32_t* __restrict__ mem, const ScanRec* __restrict__ mrec,
                                                              const double* __restrict__ uv, int W, int H,
                                                              uint32_t npts, int kk, Epi E,
                                                              unsigned long long* __restrict__ pairs,
                                                              uint32_t* __restrict__ hard_count,
                                                              uint32_t* __restrict__ hard_list,
                                                              unsigned long long* __restrict__ hard_stat,
                                                              uint32_t* __restrict__ next_point,
                                                              uint32_t* __restrict__ zero_next, int hand_off) {
    __shared__ uint32_t queue[4][2][2][kQueue16];
    __shared__ int s_loff[kMaxLv];
    __shared__ int s_lg[kMaxLv];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int l = 0; l < kMaxLv; ++l) {
            s_loff[l] = L.loff[l];
            s_lg[l] = 31 - __clz(max(L.lw[l], 1));
        }
    }
    __syncthreads();
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x < 2) zero_next[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 2 && E.zero_word) *E.zero_word = 0;
    if (blockIdx.x == 0 && threadIdx.x >= 3 && threadIdx.x < 6 && E.ovf_zero) E.ovf_zero[threadIdx.x - 3] = 0;
    prefetch_l2(E.pf, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int hl = lane & 15, hh = lane >> 4;
    unsigned lvmask = 0;
    if (lane < L.levels && L.lcount[lane] > 0) lvmask = 1u;
    lvmask = __ballot_sync(0xffffffffu, lvmask);
    const int npop = __popc(lvmask);
    const int my_pop = hl < npop ? __fns(lvmask, 0, hl + 1) : 0;
    const int lg0 = s_lg[0];
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    // persistent warps over point pairs (2c, 2c + 1), claimed as in
    // knn_points_kernel
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    uint32_t claim = blockIdx.x * (blockDim.x >> 5) + warp;
    for (;;) {
    const uint32_t pair = __shfl_sync(0xffffffffu, claim, 0);
    if (pair >= (npts + 1) / 2) return;  // warp-uniform
    if (lane == 0) claim = nwarps + atomicAdd(next_point, 1u);
    const uint32_t pt = 2 * pair + hh;
    const bool active = pt < npts;  // the second half of an odd tail searches a dummy point
    double px = 0.5, py = 0.5;
    if (active) point_of(uv, E, W, H, pt, px, py);
    const PtBox pb = pt_box(px, py);
    if (active && E.mode == 0) {  // the target pixel the epilogue reads
        const float* tp = E.target + (size_t)E.sidx[pt] * 3;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
    }
    HalfTopK t;
    t.init(kk, hl);
    unsigned long long evaluated = 0;

    // (1) seeds, as knn_points_kernel
    const int lfine = __ffs(lvmask) - 1;
    const int cx0 = cell_of(px, 1 << lg0), cy0 = cell_of(py, 1 << lg0);
    for (int pass = 0; pass < 2; ++pass) {
        const int nitems = pass == 0 ? 8 + npop : 8 * (npop - 1);
        for (int base = 0; base < nitems; base += 16) {
            const int it = base + hl;
            int k, d;
            if (pass == 0) {
                k = it < 9 ? 0 : it - 8;
                d = it < 9 ? it : 4;
            } else {
                k = 1 + it / 8;
                d = it % 8 + (it % 8 >= 4);
            }
            const int l = __shfl_sync(0xffffffffu, my_pop, min(k, 15), 16);
            uint32_t o = 0, m = 0;
            if (it < nitems) {
                const int lg = s_lg[l], G = 1 << lg;
                const int x = (cx0 >> l) + d % 3 - 1, y = (cy0 >> l) + d / 3 - 1;
                if (x >= 0 && x < G && y >= 0 && y < G) {
                    const uint32_t c = (uint32_t)(s_loff[l] + (y << lg) + x);
                    if (pass == 0) {
                        o = off[c];
                        m = own[c].count;
                    } else {
                        const Sum so = own[c];
                        if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                            o = off[c];
                            m = so.count;
                        }
                    }
                }
            }
            eval_members16(t, o, m, hl, mrec, mem, px, py, evaluated);
        }
    }

    // (1b) ring widening at the finest level while a half has no threshold
    int R = 1;
    for (;;) {
        const bool need = !(t.tq() < inf) && R < kSeedRMax;
        if (__ballot_sync(0xffffffffu, need) == 0) break;
        if (need) ++R;
        const int nring = need ? 8 * R : 0;
        const int nmax = max(nring, other_half(nring));
        const int lg = s_lg[lfine], G = 1 << lg, sx = cx0 >> lfine, sy = cy0 >> lfine;
        for (int b = 0; b < nmax; b += 16) {
            const int it = b + hl;
            uint32_t o = 0, m = 0;
            if (it < nring) {
                const int x = sx + ring_dx(it, R), y = sy + ring_dy(it, R);
                if (x >= 0 && x < G && y >= 0 && y < G) {
                    const uint32_t c = (uint32_t)(s_loff[lfine] + (y << lg) + x);
                    o = off[c];
                    m = own[c].count;
                }
            }
            eval_members16(t, o, m, hl, mrec, mem, px, py, evaluated);
        }
    }

    // (2) descent, as knn_points_kernel (flat start at ls, one pass per level)
    bool overflow = false;
    uint32_t* cur = queue[warp][hh][0];
    uint32_t* nxt = queue[warp][hh][1];
    const int ls = min(L.levels - 1, max(lg0 - kFlatStart16, 0));
    {
        const uint32_t c0 = ls + 1 < L.levels ? (uint32_t)s_loff[ls + 1] : 0u;
        const uint32_t nup = ls + 1 < L.levels ? (uint32_t)(s_loff[L.levels - 1] + 1) - c0 : 0u;
        for (uint32_t b = 0; b < nup; b += 16) {
            const uint32_t c = c0 + b + hl;
            uint32_t o = 0, m = 0;
            if (b + hl < nup) {
                int l = ls + 1;
                while (l + 1 < L.levels && (uint32_t)s_loff[l + 1] <= c) ++l;
                const int lg = s_lg[l];
                const int node = (int)(c - (uint32_t)s_loff[l]);
                const int x = node & ((1 << lg) - 1), y = node >> lg;
                const int Rl = l == lfine ? R : 1;
                if (abs(x - (cx0 >> l)) > Rl || abs(y - (cy0 >> l)) > Rl) {
                    const Sum so = own[c];
                    if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                        o = off[c];
                        m = so.count;
                    }
                }
            }
            eval_members16(t, o, m, hl, mrec, mem, px, py, evaluated);
        }
    }
    int ncur = 0;
    {
        const int lg = s_lg[ls], nls = 1 << (2 * lg);
        const uint32_t lo = (uint32_t)s_loff[ls];
        const int sx = cx0 >> ls, sy = cy0 >> ls, Rl = ls == lfine ? R : 1;
        for (int b = 0; b < nls; b += 16) {
            const int node = b + hl;
            bool keep = false;
            uint32_t o = 0, m = 0;
            if (node < nls) {
                keep = sum_lb_f(sub[lo + node], pb) <= t.tqf();
                const int x = node & ((1 << lg) - 1), y = node >> lg;
                if (keep && (abs(x - sx) > Rl || abs(y - sy) > Rl)) {
                    const Sum so = own[lo + node];
                    if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                        o = off[lo + node];
                        m = so.count;
                    }
                }
            }
            const unsigned mh = half_bits(__ballot_sync(0xffffffffu, keep));
            const int pos = ncur + __popc(mh & ((1u << hl) - 1));
            if (keep) cur[pos] = (uint32_t)node;  // (at most 16 <= kQueue16)
            ncur += __popc(mh);
            eval_members16(t, o, m, hl, mrec, mem, px, py, evaluated);
        }
        __syncwarp();
    }
    // one level per pass (two per pass -- a kept node's 16 grandchildren on
    // the 16 lanes -- halves the dependent rounds but measured 20 % slower:
    // the search is issue-bound, and it tests more nodes).  Own lists of
    // levels with no members (lvmask) are not read.
    for (int l = ls; l > 0; --l) {
        if (__ballot_sync(0xffffffffu, ncur > 0) == 0) break;
        const int lg = s_lg[l];
        const int wmask = (1 << lg) - 1;
        const uint32_t clo = (uint32_t)s_loff[l - 1];
        const int clg = lg + 1;
        const int csx = cx0 >> (l - 1), csy = cy0 >> (l - 1);
        const int cR = l - 1 == lfine ? R : 1;
        const bool cpop = (lvmask >> (l - 1)) & 1u;
        int nnext = 0;
        const int items = ncur * 4, imax = max(items, other_half(items));
        for (int base = 0; base < imax; base += 16) {
            const int item = base + hl;
            bool keep = false;
            uint32_t child = 0, o = 0, m = 0;
            if (item < items) {
                const uint32_t node = cur[item >> 2];
                const uint32_t x = node & (uint32_t)wmask, y = node >> lg;
                const uint32_t cx = 2 * x + (item & 1), cy = 2 * y + ((item >> 1) & 1);
                child = (cy << clg) + cx;
                keep = sum_lb_f(sub[clo + child], pb) <= t.tqf();
                if (keep && cpop && (abs((int)cx - csx) > cR || abs((int)cy - csy) > cR)) {
                    const Sum so = own[clo + child];
                    if (so.count && sum_lb_f(so, pb) <= t.tqf()) {
                        o = off[clo + child];
                        m = so.count;
                    }
                }
            }
            const unsigned mh = half_bits(__ballot_sync(0xffffffffu, keep));
            const int pos = nnext + __popc(mh & ((1u << hl) - 1));
            if (keep && pos < kQueue16) nxt[pos] = child;
            nnext += __popc(mh);
            eval_members16(t, o, m, hl, mrec, mem, px, py, evaluated);
        }
        __syncwarp();
        if (nnext > kQueue16) {  // this half stops; the other goes on
            overflow = true;
            nnext = 0;
        }
        uint32_t* tmp = cur;
        cur = nxt;
        nxt = tmp;
        ncur = nnext;
    }

    // frontier overflow (rare: the first steps from an initial set): handed
    // to the split hard-point scan up to its capacity (hand_off), else all N
    // scanned here by this half-warp
    bool handed = false;
    if (__ballot_sync(0xffffffffu, overflow && active)) {
        const bool mine = overflow && active;
        uint32_t slot = 0;
        if (mine && hl == 0) {
            slot = atomicAdd(hard_count, 1u);
            if (hard_stat) atomicAdd(hard_stat, 1ull);
        }
        slot = __shfl_sync(0xffffffffu, slot, 0, 16);
        bool brute = false;
        if (mine) {
            if (hand_off && slot < kHardCap) {
                if (hl == 0) hard_list[slot] = pt;
                handed = true;
            } else {
                brute = true;
                t.init(kk, hl);
            }
        }
        if (__ballot_sync(0xffffffffu, brute)) {
            for (uint32_t base = 0; base < n; base += 16) {
                const uint32_t gi = base + hl;
                double q = inf;
                bool cand = false;
                if (brute && gi < n) {
                    q = maha(scan[gi], px, py);
                    cand = t.beats(q, gi);
                }
                unsigned mh = half_bits(__ballot_sync(0xffffffffu, cand));
                const int np = __popc(mh), npmax = max(np, other_half(np));
                for (int r = 0; r < npmax; ++r) {
                    const int src = mh ? __ffs(mh) - 1 : 0;
                    mh &= mh - 1;
                    double qq = __shfl_sync(0xffffffffu, q, src, 16);
                    uint32_t ii = base + src;
                    if (r >= np || !t.beats(qq, ii)) {
                        qq = inf;
                        ii = kNoIdx;
                    }
                    t.push(qq, ii);
                    t.refresh();
                }
            }
            if (brute) evaluated += n;
        }
    }
    if (pairs && active && hl == 0) atomicAdd(pairs, evaluated);
    warp_epilogue<16>(E, scan, pt, active && !handed, kk, hl, t.q, t.i, px, py);
    }  // persistent loop
}

// Hard points (frontier overflow) are resolved by an exact split scan:
// hard_scan_kernel -- a persistent grid walks (point, split) items; each CTA
// scans a contiguous 1/kHardSplit of the set with per-thread top-K lists and
// folds them (warp 0) into one partial list; the CTA completing a point's
// last split then offers the kHardSplit partial lists to a warp top-K (any
// order: (q, idx) is a strict total order) and runs the epilogue.
constexpr int kHardThreads = 128;
constexpr int kHardSplit = 32;

// The point of hard slot `slot`: merge its kHardSplit partial lists (any
// order: (q, idx) is a strict total order) and run the epilogue -- one warp.
__device__ __forceinline__ void hard_merge_point(const ScanRec* __restrict__ scan, uint32_t n,
                                                 const double* __restrict__ uv, int W, int H, int kk,
                                                 const uint32_t* __restrict__ hard_list, const Epi& E,
                                                 const double* __restrict__ part_q,
                                                 const uint32_t* __restrict__ part_i, uint32_t slot, int lane,
                                                 unsigned long long* __restrict__ pairs) {
    const uint32_t pt = hard_list[slot];
    double px, py;
    point_of(uv, E, W, H, pt, px, py);
    const PtBox pb = pt_box(px, py);
    WarpTopK t;
    t.init(kk, lane);
    for (int sp = 0; sp < kHardSplit; ++sp) {
        const size_t o = ((size_t)slot * kHardSplit + sp) * kk;
        const double q = lane < kk ? part_q[o + lane] : 0.0;
        const uint32_t i = lane < kk ? part_i[o + lane] : kNoIdx;
        for (int j = 0; j < kk; ++j) {
            const uint32_t ij = __shfl_sync(0xffffffffu, i, j);
            const double qj = __shfl_sync(0xffffffffu, q, j);
            if (ij == kNoIdx) break;
            t.offer(qj, ij);
        }
    }
    if (pairs && lane == 0) atomicAdd(pairs, (unsigned long long)n);
    warp_epilogue<32>(E, scan, pt, true, kk, lane, t.q, t.i, px, py);
}

// The (point, split) items of the hard points (cnt of them) for a CTA of
// at least kHardThreads threads: items first, first + stride, ...; sq / si:
// kHardThreads * KCAP entries of the caller's shared memory.
template <int KCAP>
__device__ __forceinline__ void hard_scan_items(const ScanRec* __restrict__ scan, uint32_t n,
                                                const double* __restrict__ uv, int W, int H, int kk, uint32_t cnt,
                                                const uint32_t* __restrict__ hard_list, const Epi& E,
                                                double* __restrict__ part_q, uint32_t* __restrict__ part_i,
                                                unsigned int* __restrict__ point_done,
                                                unsigned long long* __restrict__ pairs, uint32_t first,
                                                uint32_t stride, double* sq /* kHardThreads * KCAP */,
                                                uint32_t* si /* kHardThreads * KCAP */) {
    const uint32_t per = (n + kHardSplit - 1) / kHardSplit;
    for (uint32_t item = first; item < cnt * kHardSplit; item += stride) {
        const uint32_t slot = item / kHardSplit, split = item % kHardSplit;
        const uint32_t pt = hard_list[slot];
        double px, py;
        point_of(uv, E, W, H, pt, px, py);
    const PtBox pb = pt_box(px, py);
        const uint32_t g0 = split * per, g1 = min(n, g0 + per);
        TopK<KCAP> t;
        t.init(kk);
        // 4 independent records in flight per thread; the (rare) insertion
        // sits behind a warp vote so it stays a branch, not predicated code
        // (threads past kHardThreads, in a wider CTA, only join the barriers)
        for (uint32_t base = g0 + (threadIdx.x < kHardThreads ? 0u : g1 - g0); base < g1; base += 4 * kHardThreads) {
            double q[4];
            uint32_t gi[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                gi[j] = base + j * kHardThreads + threadIdx.x;
                q[j] = gi[j] < g1 ? maha(scan[gi[j]], px, py) : __longlong_as_double(0x7ff0000000000000LL);
            }
            const double qm = fmin(fmin(q[0], q[1]), fmin(q[2], q[3]));
            if (__any_sync(0xffffffffu, qm <= t.tq())) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (gi[j] < g1 && q[j] <= t.tq()) t.offer(q[j], gi[j]);
            }
        }
        __syncthreads();
        if (threadIdx.x < kHardThreads) store_topk(t, sq + threadIdx.x * KCAP, si + threadIdx.x * KCAP);
        __syncthreads();
        if (threadIdx.x < 32) {
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
                    part_q[(size_t)item * kk + r] = v;
                    part_i[(size_t)item * kk + r] = vi;
                }
            }
            // the CTA finishing a point's last split merges it (the partial
            // writes are made visible before the count that publishes them)
            unsigned last = 0;
            if (lane == 0) {
                __threadfence();
                last = atomicAdd(point_done + slot, 1u) == (unsigned)(kHardSplit - 1);
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
                hard_merge_point(scan, n, uv, W, H, kk, hard_list, E, part_q, part_i, slot, lane, pairs);
                if (lane == 0) point_done[slot] = 0;  // ready for the next search
            }
        }
    }
}

template <int KCAP>
__global__ void __launch_bounds__(kHardThreads) hard_scan_kernel(const ScanRec* __restrict__ scan, uint32_t n,
                                                                 const double* __restrict__ uv, int W, int H, int kk,
                                                                 const uint32_t* __restrict__ hard_count,
                                                                 const uint32_t* __restrict__ hard_list, Epi E,
                                                                 double* __restrict__ part_q,
                                                                 uint32_t* __restrict__ part_i,
                                                                 unsigned int* __restrict__ point_done,
                                                                 unsigned long long* __restrict__ pairs) {
    __shared__ double sq[kHardThreads * KCAP];
    __shared__ uint32_t si[kHardThreads * KCAP];
    pdl_wait();
    hard_scan_items<KCAP>(scan, n, uv, W, H, kk, min(*hard_count, kHardCap), hard_list, E, part_q, part_i, point_done,
                          pairs, blockIdx.x, gridDim.x, sq, si);
}

// The hard-point scan and the reduction's offsets + scatter in one persistent
// launch (one CTA per SM): the hard points' contributions (when there are
// any) land before a grid barrier, then offsets_scatter_body.  Saves the
// hard-point scan's own launch, which the chain pays even when it is empty.
// With fuse_long (bucket mode) the loss (CTAs 0..kLossCtas-1, first) and the
// long segments (after one more barrier, only when there are any) ride here
// too, and the separate long-segment launch is skipped.
template <int KCAP>
__global__ void __launch_bounds__(kOffThreads) hard_offsets_kernel(const ScanRec* __restrict__ scan, uint32_t n,
                                                                   const double* __restrict__ uv, int W, int H, int kk,
                                                                   const uint32_t* __restrict__ hard_count,
                                                                   const uint32_t* __restrict__ hard_list, Epi E,
                                                                   double* __restrict__ part_q,
                                                                   uint32_t* __restrict__ part_i,
                                                                   unsigned int* __restrict__ point_done,
                                                                   unsigned long long* __restrict__ pairs,
                                                                   OffArgs A, LongArgs LA, int fuse_long) {
    __shared__ __align__(16) unsigned char s_raw[kLongSmemBytes > kHardThreads * KCAP * 12 ? kLongSmemBytes
                                                                                         : kHardThreads * KCAP * 12];
    pdl_wait();
    if (fuse_long && LA.dloss && blockIdx.x < kLossCtas)
        loss_chunk<kOffThreads>(LA, blockIdx.x, reinterpret_cast<double*>(s_raw));
    const uint32_t cnt = min(*hard_count, kHardCap);
    unsigned base = 0;
    if (cnt) {  // (uniform: every CTA read the same count)
        hard_scan_items<KCAP>(scan, n, uv, W, H, kk, cnt, hard_list, E, part_q, part_i, point_done, pairs, blockIdx.x,
                              gridDim.x, reinterpret_cast<double*>(s_raw),
                              reinterpret_cast<uint32_t*>(s_raw + kHardThreads * KCAP * 8));
        igs_grid_sync(A.bar, gridDim.x);
        base = gridDim.x;
    }
    base = offsets_scatter_body(A, base);
    // bucket mode: the long-segment queue was complete before the launch
    // (search epilogue) or the barrier above (hard points) -- uniform
    if (fuse_long && *(volatile const uint32_t*)LA.long_count) {
        base += gridDim.x;
        igs_grid_sync(A.bar, base);  // the overflow entries scattered
        long_segments<kOffThreads>(LA, blockIdx.x, gridDim.x, reinterpret_cast<uint32_t*>(s_raw),
                                   reinterpret_cast<uint32_t*>(s_raw) + kLongCap,
                                   reinterpret_cast<double(*)[8]>(s_raw + (kLongCap + kLongRank) * 4));
    }
    if (base) grid_exit(A.bar);  // (no barrier used -- the common case -- nothing to reset; uniform)
}


struct KnnBufs {
    DevBuf cnt, off, key, mem, own, sub, cub_tmp, hard, ticket, part, lcount, acc, mcell;
    DevBuf mrec, minv;  // records in member order, and each Gaussian's position there
    DevBuf bctl;        // lq_build_kernel: barrier counters + chunk totals
    int hard_phase = 0;  // which (hard count, cursor) pair the next search uses
    int knn_blocks[2] = {0, 0};  // resident CTAs for the persistent query kernels (full warp, halves)
    uint64_t version = ~0ull;  // params_version the summaries describe
    // refit chain: Adam launches accumulated every Gaussian into acc (by its
    // cell at the last rebuild) for each params version up to `chain`
    bool acc_ok = false;
    uint64_t chain = ~0ull;
    uint32_t built_n = 0;
    int since_build = 0;
    uint64_t builds = 0, refits = 0;
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

// What knn_points_kernel reads besides the tree: the scan records and the
// member lists.
L2Prefetch search_inputs(igs_ctx* ctx, const KnnBufs& b) {
    L2Prefetch pf{};
    l2pf_add(pf, ctx->scan, (size_t)ctx->n * sizeof(ScanRec));
    l2pf_add(pf, b.mem.p, (size_t)ctx->n * 4);
    l2pf_add(pf, b.mrec.p, (size_t)ctx->n * sizeof(ScanRec));
    return pf;
}

int knn_build(igs_ctx* ctx) {
    if (!ctx->knn) ctx->knn = new KnnBufs();
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    const StageJob job = ctx->stage_job;  // run by lq_tree_kernel below, or standalone
    ctx->stage_job = StageJob{};
    if (b.version == ctx->params_version) return igs_stage_launch(ctx, job);
    // ctx->knn_grown: the last Adam's count of Gaussians grown past their
    // level, read back with the step's status (-1: unknown)
    if (b.acc_ok && b.chain == ctx->params_version && b.built_n == ctx->n && b.since_build < kRefitPeriod &&
        ctx->knn_grown >= 0 && ctx->knn_grown <= (long long)(ctx->n >> kGrowShift)) {
        b.refits++;
        // every Gaussian was accumulated into its (old) cell by the Adam
        // launches since the last build: re-derive the summaries only
        const int nb = (b.lq.G0 + kBlk - 1) / kBlk;
        igs_prof_begin(ctx, IGS_PROF_CULL);
        if (ctx->n <= kTreeWideMaxN)
            IGS_PDL(ctx, lq_tree_kernel<2 * kTreeThreads>, nb * nb, 2 * kTreeThreads, 0, (const ScanRec*)b.mrec.p,
                    (const uint32_t*)b.mcell.p, (const uint32_t*)b.off.p, ctx->n, (Acc*)b.acc.p, b.lq,
                    (const uint32_t*)b.cnt.p, (Sum*)b.own.p, (Sum*)b.sub.p, (unsigned int*)b.ticket.p,
                    search_inputs(ctx, b), job, 0);
        else
            IGS_PDL(ctx, lq_tree_kernel<kTreeThreads>, nb * nb, kTreeThreads, 0, (const ScanRec*)b.mrec.p,
                    (const uint32_t*)b.mcell.p, (const uint32_t*)b.off.p, ctx->n, (Acc*)b.acc.p, b.lq,
                    (const uint32_t*)b.cnt.p, (Sum*)b.own.p, (Sum*)b.sub.p, (unsigned int*)b.ticket.p,
                    search_inputs(ctx, b), job, 0);
        igs_prof_end(ctx, IGS_PROF_CULL, 0.0);
        b.since_build++;
        b.version = b.chain = ctx->params_version;
        return IGS_OK;
    }
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
        !grow(b.mem, (size_t)n * 4) || !grow(b.mrec, (size_t)n * sizeof(ScanRec)) || !grow(b.minv, (size_t)n * 4) ||
        !grow(b.mcell, (size_t)n * 4) || !grow(b.own, (size_t)cells * sizeof(Sum)) ||
        !grow(b.sub, (size_t)cells * sizeof(Sum)))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
    if (!b.ticket.p) {
        if (!grow(b.ticket, 16)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
        IGS_CUDA(ctx, cudaMemsetAsync(b.ticket.p, 0, 16, ctx->stream));
    }
    if (!grow(b.lcount, kMaxLv * 4) || !grow(b.acc, (size_t)cells * sizeof(Acc)))
        return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
    L.lcount = (const uint32_t*)b.lcount.p;
    uint32_t* cnt = (uint32_t*)b.cnt.p;
    uint32_t* cur = cnt + cells;
    uint32_t* off = (uint32_t*)b.off.p;
    igs_prof_begin(ctx, IGS_PROF_CULL);
    if (!getenv("IGS_KNN_BUILD_LAUNCHES")) {
        // one persistent launch (lq_build_kernel): [0, 2) barrier counters, then chunk totals
        if (!b.bctl.p) {
            if (!grow(b.bctl, (2 + (size_t)ctx->sm_count) * 4))
                return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
            IGS_CUDA(ctx, cudaMemsetAsync(b.bctl.p, 0, 8, ctx->stream));
        }
        IGS_PDL_COOP(ctx, lq_build_kernel, ctx->sm_count, kBuildThreads, 0, (const ScanRec*)ctx->scan, n, L, cells, cnt,
                cur, off, (uint32_t*)b.key.p, (uint32_t*)b.mem.p, (ScanRec*)b.mrec.p, (uint32_t*)b.minv.p,
                (uint32_t*)b.mcell.p, (Acc*)b.acc.p, (uint32_t*)b.lcount.p, (unsigned*)b.bctl.p);
    } else {
        IGS_PDL(ctx, lq_clear, 2 * ctx->sm_count, 256, 0, cells, cnt, (Acc*)b.acc.p, (uint32_t*)b.lcount.p);
        IGS_PDL(ctx, lq_count, (n + 255) / 256, 256, 0, (const ScanRec*)ctx->scan, n, L, cnt, (uint32_t*)b.key.p,
                (uint32_t*)b.lcount.p);
        const int es = igs_scan_excl_u32(ctx, cnt, off, (size_t)cells);
        if (es) return es;
        IGS_PDL(ctx, lq_fill, (n + 255) / 256, 256, 0, (const ScanRec*)ctx->scan, n, (const uint32_t*)b.key.p,
                (const uint32_t*)off, cur, (uint32_t*)b.mem.p, (ScanRec*)b.mrec.p, (uint32_t*)b.minv.p,
                (uint32_t*)b.mcell.p, (Acc*)b.acc.p);
    }
    const int nb = (G0 + kBlk - 1) / kBlk;
    if (n <= kTreeWideMaxN)
        IGS_PDL(ctx, lq_tree_kernel<2 * kTreeThreads>, nb * nb, 2 * kTreeThreads, 0, (const ScanRec*)b.mrec.p,
                (const uint32_t*)b.mcell.p, (const uint32_t*)off, n, (Acc*)b.acc.p, L, (const uint32_t*)cnt,
                (Sum*)b.own.p, (Sum*)b.sub.p, (unsigned int*)b.ticket.p, search_inputs(ctx, b), job, 1);
    else
        IGS_PDL(ctx, lq_tree_kernel<kTreeThreads>, nb * nb, kTreeThreads, 0, (const ScanRec*)b.mrec.p,
                (const uint32_t*)b.mcell.p, (const uint32_t*)off, n, (Acc*)b.acc.p, L, (const uint32_t*)cnt,
                (Sum*)b.own.p, (Sum*)b.sub.p, (unsigned int*)b.ticket.p, search_inputs(ctx, b), job, 1);
    igs_prof_end(ctx, IGS_PROF_CULL, 0.0);
    b.lq = L;
    b.builds++;
    b.version = b.chain = ctx->params_version;
    b.acc_ok = true;
    b.built_n = n;
    b.since_build = 0;
    return IGS_OK;
}

template <int KCAP>
int launch_knn(igs_ctx* ctx, const double* uv, int W, int H, uint32_t npts, int kk, const Epi& E) {
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    if (!b.hard.p) {
        // [0..3] counter pairs, [4..] hard list, [4 + kHardCap..] per-slot split counts
        if (!grow(b.hard, (2 * kHardCap + 4) * 4)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
        IGS_CUDA(ctx, cudaMemsetAsync(b.hard.p, 0, (2 * kHardCap + 4) * 4, ctx->stream));
    }
    // [0,1] and [2,3]: two (hard-point count, point cursor) pairs used by
    // alternate searches -- each search zeroes the other pair; [4..] list
    uint32_t* hard_count = (uint32_t*)b.hard.p + 2 * b.hard_phase;
    uint32_t* cursor = hard_count + 1;
    uint32_t* zero_next = (uint32_t*)b.hard.p + 2 * (b.hard_phase ^ 1);
    uint32_t* hard_list = (uint32_t*)b.hard.p + 4;
    b.hard_phase ^= 1;
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    // kk <= 16: two points per warp (knn_points16_kernel)
    const bool halves = kk <= 16 && !getenv("IGS_KNN_FULLWARP");  // (A/B switch for tests and profiling)
    if (b.knn_blocks[halves] == 0) {
        int per_sm = 0;
        if (halves)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, knn_points16_kernel, 128, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, knn_points_kernel, 128, 0);
        b.knn_blocks[halves] = std::max(1, per_sm) * ctx->sm_count;
    }
    const uint64_t per_block = halves ? 8 : 4;
    const unsigned blocks =
        (unsigned)std::min<uint64_t>(b.knn_blocks[halves], ((uint64_t)npts + per_block - 1) / per_block);
    // frontier overflows go to the split hard-point scan (a launch of its
    // own, ~1.4 us per step even when empty); IGS_KNN_HARD_INWARP: the
    // half-warp search scans an overflowing point's whole set itself and the
    // launch is skipped -- cheaper when nothing overflows, but a half-warp
    // scanning all N serially takes milliseconds when something does
    const bool hand_off = !halves || getenv("IGS_KNN_HARD_INWARP") == nullptr;
    if (halves)
        IGS_PDL(ctx, knn_points16_kernel, blocks, 128, 0, (const ScanRec*)ctx->scan, ctx->n,
                b.lq, (const Sum*)b.own.p, (const Sum*)b.sub.p, (const uint32_t*)b.off.p, (const uint32_t*)b.mem.p,
            (const ScanRec*)b.mrec.p, uv,
            W, H, npts, kk, E, igs_prof_counter(ctx, IGS_PROF_SCAN), hard_count, hard_list,
            igs_prof_counter(ctx, IGS_PROF_KNN_HARD), cursor, zero_next, (int)hand_off);
    else
        IGS_PDL(ctx, knn_points_kernel, blocks, 128, 0, (const ScanRec*)ctx->scan, ctx->n,
            b.lq, (const Sum*)b.own.p, (const Sum*)b.sub.p, (const uint32_t*)b.off.p, (const uint32_t*)b.mem.p,
            (const ScanRec*)b.mrec.p, uv,
            W, H, npts, kk, E, igs_prof_counter(ctx, IGS_PROF_SCAN), hard_count, hard_list,
            igs_prof_counter(ctx, IGS_PROF_KNN_HARD), cursor, zero_next);
    const size_t pitems = (size_t)kHardCap * kHardSplit * kk;
    if (!grow(b.part, pitems * 12)) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (knn)");
    double* part_q = (double*)b.part.p;
    uint32_t* part_i = (uint32_t*)(part_q + pitems);
    bool fused_off = false;
    if constexpr (KCAP <= 16) {
        if (hand_off && ctx->fuse_off.ready) {
            // the reduction's offsets + scatter ride in the same launch
            ctx->fuse_off.ready = false;
            ctx->fuse_off.done = true;
            fused_off = true;
            // (profiled with the reduction: mostly its offsets + scatter)
            igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
            igs_prof_begin(ctx, IGS_PROF_REDUCE);
            // up to kOffCtasPerSm co-resident CTAs per SM (the long segments
            // take one CTA each)
            static int per_sm = 0;
            if (!per_sm) {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hard_offsets_kernel<KCAP>, kOffThreads, 0);
                per_sm = std::max(1, std::min(per_sm, kOffCtasPerSm));
            }
            IGS_PDL_COOP(ctx, hard_offsets_kernel<KCAP>, per_sm * ctx->sm_count, kOffThreads, 0,
                         (const ScanRec*)ctx->scan, ctx->n, uv, W, H, kk, (const uint32_t*)hard_count,
                         (const uint32_t*)hard_list, E, part_q, part_i,
                         (unsigned int*)((uint32_t*)b.hard.p + 4 + kHardCap), igs_prof_counter(ctx, IGS_PROF_SCAN),
                         ctx->fuse_off.args, ctx->fuse_off.long_args, (int)ctx->fuse_off.fuse_long);
            igs_prof_end(ctx, IGS_PROF_REDUCE, 0.0);
            return IGS_OK;
        }
    }
    if (hand_off && !fused_off) {
        IGS_PDL(ctx, hard_scan_kernel<KCAP>, ctx->sm_count, kHardThreads, 0, (const ScanRec*)ctx->scan, ctx->n, uv,
                W, H, kk, (const uint32_t*)hard_count, (const uint32_t*)hard_list, E, part_q, part_i,
                (unsigned int*)((uint32_t*)b.hard.p + 4 + kHardCap), igs_prof_counter(ctx, IGS_PROF_SCAN));
    }
    igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
    return IGS_OK;
}

int run_knn(igs_ctx* ctx, const double* uv, int W, int H, uint32_t npts, int kk, const Epi& E) {
    int e = knn_build(ctx);
    if (e) return e;
    if (kk <= 4) return launch_knn<4>(ctx, uv, W, H, npts, kk, E);
    if (kk <= 8) return launch_knn<8>(ctx, uv, W, H, npts, kk, E);
    if (kk <= 10) return launch_knn<10>(ctx, uv, W, H, npts, kk, E);
    if (kk <= 16) return launch_knn<16>(ctx, uv, W, H, npts, kk, E);
    return launch_knn<32>(ctx, uv, W, H, npts, kk, E);
}

// ---------------------------------------------------------------------------
// Global render through the loose quadtree (renderer.cpp:161-191): one warp
// per 8 x 4 pixel patch, lane = pixel, a register top-K per lane (the
// reference's per-pixel selection), one shared candidate search per patch.
// A tree node or cell is skipped only when its certified bound over the
// patch's pixel-centre box, lambda_min * dist(box, bbox)^2 * slack, exceeds
// T = the largest kk-th best q over the lanes -- then none of its members
// can enter any lane's top-K (strictly, so index ties are never pruned).
// Members are staged 32 at a time in shared memory and every lane scans
// them; the epilogue is raster_global_kernel's (blend, clamp, float32).
// ---------------------------------------------------------------------------
constexpr int kPatchW = 8, kPatchH = 4;

__device__ __forceinline__ double box_lb(const Sum& s, double bx0, double by0, double bx1, double by1) {
    if (s.count == 0) return __longlong_as_double(0x7ff0000000000000LL);
    const double dx = fmax(fmax((double)s.x0 - bx1, bx0 - (double)s.x1), 0.0);
    const double dy = fmax(fmax((double)s.y0 - by1, by0 - (double)s.y1), 0.0);
    return (double)s.lmin * (dx * dx + dy * dy) * (double)s.slack;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// Every lane offers the members of up to 32 cells (lane i: [o_i, o_i + m_i))
// for its own pixel; returns the refreshed warp threshold.
template <int KCAP>
__device__ __forceinline__ double raster_members(TopK<KCAP>& t, uint32_t o_mine, uint32_t m_mine, int lane,
                                                 const ScanRec* __restrict__ mrec, const uint32_t* __restrict__ mem,
                                                 ScanRec* stage, uint32_t* stage_i, double px, double py,
                                                 double T, unsigned long long& evaluated) {
    if (__ballot_sync(0xffffffffu, m_mine != 0) == 0) return T;
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
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t ex = __shfl_sync(0xffffffffu, excl, lo + step);
            if (ex <= f) lo += step;
        }
        const uint32_t lo_ex = __shfl_sync(0xffffffffu, excl, lo);
        const uint32_t lo_o = __shfl_sync(0xffffffffu, o_mine, lo);
        __syncwarp();
        if (f < total) {
            const uint32_t p = lo_o + (f - lo_ex);
            const uint32_t gi = __ldg(mem + p);
            stage[lane] = mrec[p];
            stage_i[lane] = gi;
        }
        __syncwarp();
        const uint32_t cnt = min(32u, total - base);
#pragma unroll 1
        for (uint32_t c = 0; c < cnt; ++c) {
            const double q = maha(stage[c], px, py);
            if (__any_sync(0xffffffffu, q <= t.tq()))
                if (q <= t.tq()) t.offer(q, stage_i[c]);
        }
        T = warp_max(t.tq());
    }
    return T;
}

template <int KCAP>
__global__ void __launch_bounds__(128, KCAP <= 16 ? 5 : 2) knn_raster_kernel(const ScanRec* __restrict__ scan,
                                                            const ShadeRec* __restrict__ shade, uint32_t n, Lq L,
                                                            const Sum* __restrict__ own, const Sum* __restrict__ sub,
                                                            const uint32_t* __restrict__ off,
                                                            const uint32_t* __restrict__ mem,
                                                            const ScanRec* __restrict__ mrec, int W, int H, int row0,
                                                            int row1, int kk, float* __restrict__ out,
                                                            uint32_t* __restrict__ topk, uint32_t npx_patch,
                                                            uint32_t npatch, uint32_t* __restrict__ next_patch,
                                                            unsigned long long* __restrict__ pairs) {
    __shared__ uint32_t queue[4][2][kQueue];
    __shared__ ScanRec stage[4][32];
    __shared__ uint32_t stage_i[4][32];
    __shared__ int s_loff[kMaxLv];
    __shared__ int s_lg[kMaxLv];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int l = 0; l < kMaxLv; ++l) {
            s_loff[l] = L.loff[l];
            s_lg[l] = 31 - __clz(max(L.lw[l], 1));
        }
    }
    __syncthreads();
    pdl_wait();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned lvmask = 0;
    if (lane < L.levels && L.lcount[lane] > 0) lvmask = 1u;
    lvmask = __ballot_sync(0xffffffffu, lvmask);
    const int npop = __popc(lvmask);
    const int my_pop = lane < npop ? __fns(lvmask, 0, lane + 1) : 0;
    const int lg0 = s_lg[0];
    for (;;) {
        uint32_t patch = 0;
        if (lane == 0) patch = atomicAdd(next_patch, 1u);
        patch = __shfl_sync(0xffffffffu, patch, 0);
        if (patch >= npatch) return;
        const int x0 = (int)(patch % npx_patch) * kPatchW, y0 = row0 + (int)(patch / npx_patch) * kPatchH;
        const int x1 = min(x0 + kPatchW, W) - 1, y1 = min(y0 + kPatchH, row1) - 1;
        const int xi = x0 + (lane % kPatchW), yi = y0 + (lane / kPatchW);
        const bool live = xi <= x1 && yi <= y1;
        // lanes past the edge work on a copy of an edge pixel (so the
        // warp threshold stays finite) and write nothing
        const double px = center(min(xi, x1), W), py = center(min(yi, y1), H);
        const double bx0 = center(x0, W), bx1 = center(x1, W), by0 = center(y0, H), by1 = center(y1, H);
        TopK<KCAP> t;
        t.init(kk);
        double T = __longlong_as_double(0x7ff0000000000000LL);
        unsigned long long evaluated = 0;
        const double cx = __dmul_rn(0.5, __dadd_rn(bx0, bx1)), cy = __dmul_rn(0.5, __dadd_rn(by0, by1));
        const int cx0 = cell_of(cx, 1 << lg0), cy0 = cell_of(cy, 1 << lg0);

        // (1) seeds around the patch centre's cell (see knn_points_kernel)
        const int nseed = npop * 9;
        const int lfine = __ffs(lvmask) - 1;
        for (int pass = 0; pass < 2; ++pass) {
            for (int b = 0; b < nseed; b += 32) {
                const int it = b + lane;
                const int l = __shfl_sync(0xffffffffu, my_pop, min(it / 9, 31));
                uint32_t o = 0, m = 0;
                if (it < nseed) {
                    const int d = it % 9, lg = s_lg[l], G = 1 << lg;
                    const int x = (cx0 >> l) + d % 3 - 1, y = (cy0 >> l) + d / 3 - 1;
                    const bool primary = d == 4 || l == lfine;
                    if (x >= 0 && x < G && y >= 0 && y < G && primary == (pass == 0)) {
                        const uint32_t c = (uint32_t)(s_loff[l] + (y << lg) + x);
                        const Sum so = own[c];
                        if (so.count && (primary || box_lb(so, bx0, by0, bx1, by1) <= T)) {
                            o = off[c];
                            m = so.count;
                        }
                    }
                }
                T = raster_members(t, o, m, lane, mrec, mem, stage[warp], stage_i[warp], px, py, T, evaluated);
            }
        }

        // (1b) widen the finest-level window while some lane has < kk
        int R = 1;
        while (!(T < __longlong_as_double(0x7ff0000000000000LL)) && R < kSeedRMax) {
            ++R;
            const int lg = s_lg[lfine], G = 1 << lg, sx = cx0 >> lfine, sy = cy0 >> lfine;
            for (int b = 0; b < 8 * R; b += 32) {
                const int it = b + lane;
                uint32_t o = 0, m = 0;
                if (it < 8 * R) {
                    const int x = sx + ring_dx(it, R), y = sy + ring_dy(it, R);
                    if (x >= 0 && x < G && y >= 0 && y < G) {
                        const uint32_t c = (uint32_t)(s_loff[lfine] + (y << lg) + x);
                        o = off[c];
                        m = own[c].count;
                    }
                }
                T = raster_members(t, o, m, lane, mrec, mem, stage[warp], stage_i[warp], px, py, T, evaluated);
            }
        }

        // (2) descent from the root with box bounds
        bool overflow = false;
        uint32_t* cur = queue[warp][0];
        uint32_t* nxt = queue[warp][1];
        int ncur = 1;
        if (lane == 0) cur[0] = 0;
        __syncwarp();
        for (int l = L.levels - 1; l >= 0 && ncur > 0; --l) {
            const int lg = s_lg[l];
            const int wmask = (1 << lg) - 1;
            const int sx = cx0 >> l, sy = cy0 >> l;
            const uint32_t lo = (uint32_t)s_loff[l];
            for (int b = 0; b < ncur; b += 32) {
                const int i = b + lane;
                uint32_t o = 0, m = 0;
                if (i < ncur) {
                    const uint32_t node = cur[i];
                    const int x = (int)node & wmask, y = (int)(node >> lg);
                    const int Rl = l == lfine ? R : 1;  // the seed window at this level
                    if (abs(x - sx) > Rl || abs(y - sy) > Rl) {
                        const uint32_t c = lo + node;
                        const Sum so = own[c];
                        if (so.count && box_lb(so, bx0, by0, bx1, by1) <= T) {
                            o = off[c];
                            m = so.count;
                        }
                    }
                }
                T = raster_members(t, o, m, lane, mrec, mem, stage[warp], stage_i[warp], px, py, T, evaluated);
            }
            if (l == 0) break;
            const uint32_t clo = (uint32_t)s_loff[l - 1];
            const int clg = lg + 1;
            int nnext = 0;
            for (int b = 0; b < ncur * 4; b += 32) {
                const int item = b + lane;
                bool keep = false;
                uint32_t child = 0;
                if (item < ncur * 4) {
                    const uint32_t node = cur[item >> 2];
                    const uint32_t x = node & (uint32_t)wmask, y = node >> lg;
                    child = ((2 * y + ((item >> 1) & 1)) << clg) + 2 * x + (item & 1);
                    keep = box_lb(sub[clo + child], bx0, by0, bx1, by1) <= T;
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
            // the frontier outgrew the queue: every lane scans all N (exact)
            t.init(kk);
            for (uint32_t b = 0; b < n; b += 32) {
                __syncwarp();
                const uint32_t gi = b + lane;
                if (gi < n) {
                    stage[warp][lane] = scan[gi];
                    stage_i[warp][lane] = gi;
                }
                __syncwarp();
                const uint32_t cnt = min(32u, n - b);
#pragma unroll 1
                for (uint32_t c = 0; c < cnt; ++c) {
                    const double q = maha(stage[warp][c], px, py);
                    if (__any_sync(0xffffffffu, q <= t.tq()))
                        if (q <= t.tq()) t.offer(q, stage_i[warp][c]);
                }
            }
            evaluated += n;
        }
        if (pairs && lane == 0) atomicAdd(pairs, evaluated * 32ull);
        if (!live) continue;
        double col[3];
        blend_topk(t, shade, col);
        const size_t o = (size_t)(yi - row0) * W + xi;
        out[o * 3 + 0] = clamp01f(col[0]);
        out[o * 3 + 1] = clamp01f(col[1]);
        out[o * 3 + 2] = clamp01f(col[2]);
        if (topk) store_topk(t, (double*)nullptr, topk + ((size_t)yi * W + xi) * kk);
    }
}

template <int KCAP>
int launch_knn_raster(igs_ctx* ctx, int W, int H, int row0, int row1, int kk, float* out, uint32_t* topk) {
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    uint32_t* cursor = (uint32_t*)igs_scratch(ctx, 27, 16);
    if (!cursor) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (raster)");
    IGS_CUDA(ctx, cudaMemsetAsync(cursor, 0, 4, ctx->stream));
    const uint32_t npx = (uint32_t)((W + kPatchW - 1) / kPatchW);
    const uint32_t npy = (uint32_t)((row1 - row0 + kPatchH - 1) / kPatchH);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, knn_raster_kernel<KCAP>, 128, 0);
    const unsigned blocks = (unsigned)std::min<uint64_t>((uint64_t)std::max(1, per_sm) * ctx->sm_count,
                                                         ((uint64_t)npx * npy + 3) / 4);
    igs_prof_begin(ctx, IGS_PROF_SCAN);
    IGS_PDL(ctx, knn_raster_kernel<KCAP>, blocks, 128, 0, (const ScanRec*)ctx->scan, (const ShadeRec*)ctx->shade,
            ctx->n, b.lq, (const Sum*)b.own.p, (const Sum*)b.sub.p, (const uint32_t*)b.off.p,
            (const uint32_t*)b.mem.p, (const ScanRec*)b.mrec.p, W, H, row0, row1, kk, out, topk, npx, npx * npy, cursor,
            igs_prof_counter(ctx, IGS_PROF_SCAN));
    igs_prof_end(ctx, IGS_PROF_SCAN, 0.0);
    return IGS_OK;
}

}  // namespace

// The refit's inputs (member records, cells, offsets and counts), for the step's first
// kernel to prefetch; empty unless the next search can refit.
L2Prefetch igs_knn_tree_inputs(igs_ctx* ctx) {
    L2Prefetch pf{};
    if (!ctx->knn) return pf;
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    if (!b.acc_ok || b.version == ctx->params_version) return pf;
    const size_t cells = (size_t)b.lq.loff[b.lq.levels - 1] + 1;
    l2pf_add(pf, b.mrec.p, (size_t)b.built_n * sizeof(ScanRec));
    l2pf_add(pf, b.mcell.p, (size_t)b.built_n * 4);
    l2pf_add(pf, b.off.p, cells * 4);
    l2pf_add(pf, b.cnt.p, cells * 4);
    return pf;
}

// Called by an Adam launch right before it bumps params_version by one.
TreeAcc igs_knn_tree_acc(igs_ctx* ctx) {
    if (!ctx->knn) return TreeAcc{nullptr, nullptr};
    KnnBufs& b = *static_cast<KnnBufs*>(ctx->knn);
    TreeAcc ta{};
    if (b.acc_ok && b.chain == ctx->params_version && b.built_n == ctx->n) {
        b.chain = ctx->params_version + 1;
        ta.acc = (Acc*)b.acc.p;
        ta.key = (const uint32_t*)b.key.p;
        ta.mrec = (ScanRec*)b.mrec.p;
        ta.minv = (const uint32_t*)b.minv.p;
        ta.grown = (unsigned long long*)(ctx->status + 3);
        ta.L = b.lq;
        return ta;
    }
    b.acc_ok = false;
    return ta;
}

void igs_knn_free(igs_ctx* ctx) {
    if (!ctx->knn) return;
    KnnBufs* b = static_cast<KnnBufs*>(ctx->knn);
    // IGS_KNN_STATS=1: how often the tree was re-bucketed vs refit (diagnostics)
    if (getenv("IGS_KNN_STATS"))
        fprintf(stderr, "knn tree: %llu builds, %llu refits\n", (unsigned long long)b->builds,
                (unsigned long long)b->refits);
    for (DevBuf* d : {&b->bctl, &b->mrec, &b->minv, &b->cnt, &b->off, &b->key, &b->mem, &b->own, &b->sub, &b->cub_tmp,
                      &b->hard, &b->ticket,
                      &b->part, &b->lcount, &b->acc, &b->mcell})
        cudaFree(d->p);
    delete b;
    ctx->knn = nullptr;
}

// Global render (kk <= 32) through the loose quadtree; rows [row0, row1).
int igs_raster_knn(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out, uint32_t* topk) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    int e = knn_build(ctx);
    if (e) return e;
    if (kk <= 4) return launch_knn_raster<4>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 8) return launch_knn_raster<8>(ctx, W, H, row0, row1, kk, out, topk);
    if (kk <= 10) return launch_knn_raster<10>(ctx, W, H, row0, row1, kk, out, topk);  // (the default K)
    if (kk <= 16) return launch_knn_raster<16>(ctx, W, H, row0, row1, kk, out, topk);
    return launch_knn_raster<32>(ctx, W, H, row0, row1, kk, out, topk);
}

// Exact top-K (q ascending, idx) at device points; kk = min(k, n).
int igs_topk_knn(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq) {
    const int kk = (int)std::min<uint32_t>((uint32_t)k, ctx->n);
    if (kk > 32 || npts == 0) return igs_topk_points(ctx, uv, npts, k, oi, oq);
    Epi E{};
    E.mode = 2;
    E.oq = oq;
    E.oi = oi;
    E.n = ctx->n;
    return run_knn(ctx, uv, 0, 0, npts, kk, E);
}

// Fused forward + backward at points (kk <= 32): the top-K search with the
// blend / loss / gradient epilogue.  mode 0: sampled target pixels (sidx),
// mode 1: samples5 (u, v, upstream).  Writes losses and either the
// contribution records + sort keys (contrib != null) or fp64 atomics into
// grads_atomic.
int igs_knn_forward_backward(igs_ctx* ctx, int mode, const uint32_t* sidx, const double* samples5, uint32_t npts,
                             int kk, double inv_n, double* losses, double* contrib, uint32_t* keys, uint32_t* gcnt,
                             double* grads_atomic, uint32_t* zero_word, const L2Prefetch* pf,
                             int defer_loss_check) {
    Epi E{};
    E.defer_loss_check = defer_loss_check;
    E.zero_word = zero_word;
    if (pf) E.pf = *pf;
    E.gcnt = gcnt;
    if (gcnt && ctx->fuse_off.ready && ctx->fuse_off.bucket) {
        E.bucket = ctx->fuse_off.bucket;
        E.ovf = ctx->fuse_off.ovf;
        E.ovf_list = ctx->fuse_off.ovf_list;
        E.long_list = ctx->fuse_off.long_list;
        E.ovf_zero = ctx->fuse_off.ovf_zero;
    }
    E.mode = mode;
    E.sidx = sidx;
    E.target = (const float*)ctx->target.p;
    E.samples5 = samples5;
    E.inv_n = inv_n;
    E.shade = ctx->shade;
    E.losses = losses;
    E.host_losses = mode == 0 && !defer_loss_check ? ctx->loss_mirror : nullptr;
    ctx->loss_mirrored = E.host_losses != nullptr;
    E.contrib = contrib;
    E.keys = keys;
    E.grads_atomic = grads_atomic;
    E.status = ctx->status;
    E.n = ctx->n;
    return run_knn(ctx, nullptr, ctx->tgt_w, ctx->tgt_h, npts, kk, E);
}
