// reduce.cuh -- the deterministic reduction's offsets + slot scatter as a
// device body, shared by offsets_scatter_kernel (train.cu) and the fused
// hard-point scan + offsets launch (knn.cu).
#pragma once

#include "igs_internal.cuh"
#include "scan.cuh"

namespace igs_dev {

constexpr uint32_t kShortSeg = 128;  // longer segments go to long_segment_kernel
// Segment buckets: the search epilogue files each slot id at
// bucket[g][arrival rank] while the rank is below kBucket = 128 (every short
// segment is then complete in its bucket: Adam sorts and sums it there, no
// offsets, no scatter).  Later arrivals are overflow entries -- (slot, rank)
// appended to a list -- and a Gaussian's first one queues it as a long
// segment.  The offsets body then gives each long segment a region of
// perm (bump allocation: regions in any order, ranks inside), a grid
// barrier, and drops the overflow entries at region + rank; the long
// kernel reads ranks < kBucket from the bucket and the rest from perm.
constexpr uint32_t kBucket = kShortSeg;
constexpr int kOffThreads = 256;
constexpr int kOffPer = 4;  // counts per thread and chunk pass
constexpr int kOffCtasPerSm = 2;  // persistent offsets launches: at most this many CTAs per SM (chunk_sum sizing)

// (OffArgs: igs_internal.cuh)

// Segment offsets (exclusive scan of the per-Gaussian counts) and the slot
// scatter for a persistent, co-resident grid of kOffThreads-thread CTAs:
// every CTA scans its chunk of the counts, a grid barrier publishes the
// chunk totals, each CTA adds its base and writes the offsets, a second
// barrier, then the scatter (slot ids at offset + arrival rank; every
// Gaussian with more than kShortSeg contributions queued once); in bucket
// mode only the overflow entries (see kBucket).  Barrier targets start at
// bar_base (arrivals already counted by the caller); returns the target
// reached.  The launch ends with grid_exit, which resets the counters.
__device__ __forceinline__ unsigned offsets_scatter_body(const OffArgs& A, unsigned bar_base) {
    __shared__ uint32_t s_base;
    const uint32_t* __restrict__ gcnt = A.gcnt;
    const uint32_t n = A.n;
    uint32_t* __restrict__ goff = A.goff;
    uint32_t* __restrict__ chunk_sum = A.chunk_sum;
    const uint32_t* __restrict__ keys = A.keys;
    const uint32_t items = A.items;
    uint32_t* __restrict__ gcur = A.gcur;
    uint32_t* __restrict__ perm = A.perm;
    uint32_t* __restrict__ long_count = A.long_count;
    uint32_t* __restrict__ long_list = A.long_list;
    const uint32_t G = gridDim.x;
    if (A.ovf) {
        const uint32_t no = *(volatile const uint32_t*)A.ovf;  // (uniform)
        if (no) {
            const uint32_t nl = *(volatile const uint32_t*)long_count;
            for (uint32_t i = blockIdx.x * kOffThreads + threadIdx.x; i < nl; i += G * kOffThreads) {
                const uint32_t g = long_list[i];
                goff[g] = atomicAdd(A.ovf + 1, gcnt[g]);  // (ranks < kBucket of the region stay unused)
            }
            igs_grid_sync(A.bar, bar_base + G);
            for (uint32_t i = blockIdx.x * kOffThreads + threadIdx.x; i < no; i += G * kOffThreads) {
                const uint32_t slot = A.ovf_list[2 * i], pos = A.ovf_list[2 * i + 1];
                perm[__ldcg(goff + keys[slot]) + pos] = slot;
            }
        }
        return no ? bar_base + G : bar_base;
    }
    // chunk of CTA b: [b * per_cta, (b + 1) * per_cta), per_cta a multiple of kOffThreads * kOffPer
    const uint32_t tile = kOffThreads * kOffPer;
    const uint32_t per_cta = ((n + G - 1) / G + tile - 1) / tile * tile;
    const uint32_t c0 = blockIdx.x * per_cta, c1 = min(n, c0 + per_cta);
    // pass 1: chunk total
    uint32_t total = 0;
    for (uint32_t b = c0; b < c1; b += tile) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < kOffPer; ++j) {
            const uint32_t i = b + threadIdx.x * kOffPer + j;
            if (i < c1) v += gcnt[i];
        }
        total += v;
    }
    {
        uint32_t agg;
        block_excl_sum<kOffThreads>(total, &agg);
        if (threadIdx.x == 0) chunk_sum[blockIdx.x] = agg;
    }
    igs_grid_sync(A.bar, bar_base + G);
    // the chunk's base: the totals of the chunks before it
    uint32_t mine = 0;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += kOffThreads) mine += *(volatile uint32_t*)(chunk_sum + b);
    {
        uint32_t base;
        block_excl_sum<kOffThreads>(mine, &base);
        if (threadIdx.x == 0) s_base = base;
    }
    __syncthreads();
    uint32_t run = s_base;
    // pass 2: offsets
    for (uint32_t b = c0; b < c1; b += tile) {
        uint32_t v[kOffPer], sum = 0;
#pragma unroll
        for (int j = 0; j < kOffPer; ++j) {
            const uint32_t i = b + threadIdx.x * kOffPer + j;
            v[j] = i < c1 ? gcnt[i] : 0u;
            sum += v[j];
        }
        uint32_t agg;
        const uint32_t excl = block_excl_sum<kOffThreads>(sum, &agg);
        uint32_t o = run + excl;
#pragma unroll
        for (int j = 0; j < kOffPer; ++j) {
            const uint32_t i = b + threadIdx.x * kOffPer + j;
            if (i < c1) goff[i] = o;
            o += v[j];
        }
        run += agg;
    }
    igs_grid_sync(A.bar, bar_base + 2 * G);
    // scatter (scatter_slots_kernel)
    for (uint32_t slot = blockIdx.x * kOffThreads + threadIdx.x; slot < items; slot += G * kOffThreads) {
        const uint32_t g = keys[slot];
        if (g >= n) continue;
        const uint32_t pos = atomicAdd(gcur + g, 1u);
        perm[__ldcg(goff + g) + pos] = slot;  // (written by other CTAs: read through L2)
        if (pos == 0 && gcnt[g] > kShortSeg) long_list[atomicAdd(long_count, 1u)] = g;
    }
    return bar_base + 2 * G;
}

// The end of a persistent launch that used grid barriers on bar: the last
// CTA out resets the counters for the next launch.
__device__ __forceinline__ void grid_exit(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(bar + 1, 1u) == gridDim.x - 1) {
        bar[0] = 0;
        bar[1] = 0;
    }
}

// Long segments: one CTA (NT threads) per queued Gaussian, CTAs first,
// first + stride, ...  The slot ids are put in slot (= sample) order in
// shared memory: up to kLongRank by counting ranks (rank = number of
// smaller ids; ids are distinct), up to kLongCap by a bitonic sort, and
// beyond shared memory by ranks straight from global memory into `big`;
// then 8 threads, one per parameter, accumulate the contribution rows in
// that order, kLongRows rows gathered ahead of the dependent adds.  After a
// Gaussian's gradient is stored the whole CTA calls fin(g).  Shared memory
// (the caller's): keys[kLongCap], sorted[kLongRank], rows[kLongRows][8].
constexpr uint32_t kLongCap = 2048;
constexpr uint32_t kLongRank = 256;  // up to here: rank by counting; above: bitonic sort
constexpr int kLongThreads = 256;
constexpr int kLongRows = 128;
constexpr uint32_t kLossCtas = 8;    // CTAs that form the loss
constexpr size_t kLongSmemBytes = kLongCap * 4 + kLongRank * 4 + kLongRows * 8 * sizeof(double);

struct NoFin {
    __device__ void operator()(uint32_t) const {}
};

template <int NT, class Fin = NoFin>
__device__ __forceinline__ void long_segments(const LongArgs& A, uint32_t first, uint32_t stride, uint32_t* keys,
                                              uint32_t* sorted, double (*rows)[8], Fin fin = Fin{}) {
    const uint32_t total = *(volatile const uint32_t*)A.long_count;
    const int t = threadIdx.x;
    for (uint32_t it = first; it < total; it += stride) {
        const uint32_t g = A.long_list[it];
        const uint32_t m = A.gcnt[g], o = A.goff[g];
        // slot id of rank e: bucket mode keeps ranks < kBucket in the bucket
        auto slot_at = [&](uint32_t e) {
            return A.bucket && e < kBucket ? A.bucket[(size_t)g * kBucket + e] : A.perm[o + e];
        };
        const uint32_t* out = sorted;
        __syncthreads();
        if (m <= kLongRank) {
            for (uint32_t e = t; e < m; e += NT) keys[e] = slot_at(e);
            __syncthreads();
            for (uint32_t e = t; e < m; e += NT) {
                const uint32_t v = keys[e];
                uint32_t r = 0;
                for (uint32_t j = 0; j < m; ++j) r += keys[j] < v;
                sorted[r] = v;
            }
        } else if (m <= kLongCap) {
            // bitonic sort in shared memory, padded to a power of two
            uint32_t pow2 = 1;
            while (pow2 < m) pow2 <<= 1;
            for (uint32_t e = t; e < pow2; e += NT) keys[e] = e < m ? slot_at(e) : 0xFFFFFFFFu;
            __syncthreads();
            for (uint32_t size = 2; size <= pow2; size <<= 1)
                for (uint32_t stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
                    for (uint32_t e = t; e < pow2; e += NT) {
                        const uint32_t partner = e ^ stride2;
                        if (partner > e) {
                            const bool up = (e & size) == 0;
                            const uint32_t a = keys[e], b = keys[partner];
                            if ((a > b) == up) {
                                keys[e] = b;
                                keys[partner] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            out = keys;
        } else {
            // beyond shared memory (degenerate sets): rank from global
            // memory into the same range of a second slot array
            for (uint32_t e = t; e < m; e += NT) {
                const uint32_t v = slot_at(e);
                uint32_t r = 0;
                for (uint32_t j = 0; j < m; ++j) r += slot_at(j) < v;
                A.big[o + r] = v;
            }
            out = A.big + o;
        }
        __syncthreads();
        double acc = 0.0;
        for (uint32_t base = 0; base < m; base += kLongRows) {
            const uint32_t cnt = min((uint32_t)kLongRows, m - base);
            for (uint32_t r = t; r < cnt; r += NT) {
                const double2* c = reinterpret_cast<const double2*>(A.contrib + (size_t)out[base + r] * 8);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const double2 v = c[h];
                    rows[r][2 * h] = v.x;
                    rows[r][2 * h + 1] = v.y;
                }
            }
            __syncthreads();
            if (t < 8)
                for (uint32_t r = 0; r < cnt; ++r) acc = __dadd_rn(acc, rows[r][t]);
            __syncthreads();
        }
        if (t < 8) {
            A.grads[(size_t)g * 8 + t] = acc;
            if (!isfinite(acc)) atomicMin(A.status, (long long)g * 8 + t);  // adam.cpp:29-31 (first (i, p))
        }
        __syncthreads();
        fin(g);
    }
}

// The loss (fit.cpp:87-89: mean of the per-sample L1 losses): chunk c of
// kLossCtas summed by one CTA (NT threads, a fixed tree), the
// chunks combined in order by whichever CTA finishes last.
template <int NT>
__device__ __forceinline__ void loss_chunk(const LongArgs& A, uint32_t c, double* red /* NT */) {
    const int t = threadIdx.x;
    const uint32_t per = (A.ns + kLossCtas - 1) / kLossCtas, l0 = c * per, l1 = min(A.ns, l0 + per);
    double acc = 0.0;
    for (uint32_t i = l0 + t; i < l1; i += NT) acc = __dadd_rn(acc, A.losses[i]);
    red[t] = acc;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (t < s) red[t] = __dadd_rn(red[t], red[t + s]);
        __syncthreads();
    }
    if (t == 0) {
        A.loss_part[c] = red[0];
        __threadfence();
        if (atomicAdd(A.loss_ticket, 1u) == kLossCtas - 1) {
            __threadfence();
            double l = 0.0;
            for (uint32_t k = 0; k < kLossCtas; ++k) l = __dadd_rn(l, __ldcg(A.loss_part + k));
            *A.dloss = __dmul_rn(l, A.inv_n);
            *A.loss_ticket = 0;
        }
    }
}

}  // namespace igs_dev
