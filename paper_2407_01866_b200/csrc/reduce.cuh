// reduce.cuh -- the deterministic reduction's offsets + slot scatter as a
// device body, shared by offsets_scatter_kernel (train.cu) and the fused
// hard-point scan + offsets launch (knn.cu).
#pragma once

#include "igs_internal.cuh"
#include "scan.cuh"

namespace igs_dev {

constexpr uint32_t kShortSeg = 32;  // longer segments go to long_segment_kernel
// Segment buckets: the search epilogue files each slot id at
// bucket[g][arrival rank] while the rank is below kBucket (every short
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

// (OffArgs: igs_internal.cuh)

// Segment offsets (exclusive scan of the per-Gaussian counts) and the slot
// scatter for a persistent, co-resident grid of kOffThreads-thread CTAs:
// every CTA scans its chunk of the counts, a grid barrier publishes the
// chunk totals, each CTA adds its base and writes the offsets, a second
// barrier, then the scatter (slot ids at offset + arrival rank; every
// Gaussian with more than kShortSeg contributions queued once).  Barrier
// targets start at bar_base (arrivals already counted by the caller); the
// last CTA out resets the counters for the next launch.
__device__ __forceinline__ void offsets_scatter_body(const OffArgs& A, unsigned bar_base) {
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
    unsigned* __restrict__ bar = A.bar;
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
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(bar + 1, 1u) == G - 1) {
            bar[0] = 0;
            bar[1] = 0;
        }
        return;
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
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(bar + 1, 1u) == G - 1) {
        bar[0] = 0;
        bar[1] = 0;
    }
}

}  // namespace igs_dev
