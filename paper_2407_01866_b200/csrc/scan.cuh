// scan.cuh -- the repo's own block/device scan and stable key/index radix
// sort (north-star kernel 2: count -> prefix-scan -> radix sort), sm_100a.
//
// * block_excl_sum: exclusive sum over a CTA (warp shuffles + one smem pass).
// * igs_scan_excl_u32: device-wide exclusive sum in ONE pass (decoupled
//   look-back: each tile publishes its aggregate, then its inclusive prefix,
//   and later tiles read back through their predecessors' flags); tiles are
//   claimed in order from an atomic ticket, so a tile only waits on tiles
//   that are already running.
// * igs_radix_sort_u64_u32: stable LSD radix sort of (u64 key, u32 value)
//   pairs, 8 bits per pass: per-tile digit histogram -> exclusive scan of the
//   digit-major (digit, tile) count matrix (the scan above) -> scatter with a
//   stable in-tile rank (warp match_any + per-warp digit counts).  Stability
//   makes it the reference comparator's (coord, idx) order when the values
//   arrive in index order.
#pragma once

#include <stdint.h>

#include "igs_internal.cuh"

namespace igs_dev {

constexpr int kScanThreads = 256;

// Exclusive sum of v over the CTA (blockDim.x == NT, NT % 32 == 0); *total
// receives the CTA's sum.  Uses NT/32 words of shared memory.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_tot[NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    uint32_t base = 0, sum = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        const uint32_t t = warp_tot[i];
        if (i < w) base += t;
        sum += t;
    }
    __syncthreads();  // warp_tot may be reused by the next call
    if (total) *total = sum;
    return base + x - v;
}

// Decoupled look-back for tile `tile` of a single-pass scan, run by one
// whole warp (all 32 lanes call it; all get the result): publishes the
// tile's aggregate, then reads 32 predecessors at once -- lane j the tile
// j + 1 back -- waits until each is published, adds them up to the nearest
// one that carries an inclusive prefix (or all 32 and moves on), publishes
// the tile's inclusive prefix and returns the exclusive one.  Status words
// carry an epoch (one per launch) so they never need clearing.  Tiles must
// be claimed in order (a ticket) so a tile only waits on running tiles.
__device__ __forceinline__ uint32_t tile_lookback(unsigned long long* status, uint32_t tile, uint32_t agg,
                                                  uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    auto pack = [&](uint32_t flag, uint32_t v) {
        return ((unsigned long long)epoch << 34) | ((unsigned long long)flag << 32) | v;
    };
    auto st = [](unsigned long long* p, unsigned long long v) {
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    };
    if (tile == 0) {
        if (lane == 0) st(status, pack(2, agg));
        return 0;
    }
    if (lane == 0) st(status + tile, pack(1, agg));
    uint32_t prefix = 0;
    for (int p = (int)tile - 1;; p -= 32) {
        const int idx = p - lane;
        uint32_t flag = 2, val = 0;  // before tile 0: nothing (tile 0 is always inclusive anyway)
        if (idx >= 0) {
            unsigned long long v;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(status + idx) : "memory");
                flag = (uint32_t)(v >> 32) & 3u;
            } while ((uint32_t)(v >> 34) != epoch || flag == 0);
            val = (uint32_t)v;
        }
        const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
        const int first = incl ? __ffs(incl) - 1 : 31;
        uint32_t x = lane <= first ? val : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        prefix += x;
        if (incl) break;
    }
    if (lane == 0) st(status + tile, pack(2, prefix + agg));
    return prefix;
}

}  // namespace igs_dev

// Device-wide exclusive sum of n u32 (in and out may alias).  Enqueued on
// ctx->stream; no host synchronisation.
int igs_scan_excl_u32(igs_ctx* ctx, const uint32_t* in, uint32_t* out, size_t n);
// Stable ascending sort of (keys, vals) by the low `bits` bits of the keys;
// the sorted pairs end in keys_out / vals_out.  keys_tmp / vals_tmp: n-entry
// scratch (ping-pong).  in may equal tmp.
int igs_radix_sort_u64_u32(igs_ctx* ctx, const unsigned long long* keys_in, const uint32_t* vals_in,
                           unsigned long long* keys_out, uint32_t* vals_out, unsigned long long* keys_tmp,
                           uint32_t* vals_tmp, size_t n, int bits);
