// scan.cu -- device-wide exclusive scan (single pass, decoupled look-back)
// and stable LSD radix sort of (u64 key, u32 value) pairs.  See scan.cuh.
#include <cuda_runtime.h>

#include <algorithm>

#include "scan.cuh"

using namespace igs_dev;

namespace {

constexpr int kScanPer = 8;                            // items per thread
constexpr uint32_t kScanTile = kScanThreads * kScanPer;  // 2048 per tile
constexpr int kSortThreads = 256;
constexpr int kSortRounds = 4;                          // 1024 items per tile
constexpr uint32_t kSortTile = kSortThreads * kSortRounds;
constexpr int kRadix = 256;

// One pass; tiles claimed in order from ctl[0]; ctl[1] counts finished
// tiles (the last one re-arms both for the next call on the stream).
__global__ void __launch_bounds__(kScanThreads) scan_lookback_kernel(const uint32_t* in, uint32_t* out, size_t n,
                                                                     unsigned long long* __restrict__ status,
                                                                     uint32_t* __restrict__ ctl, uint32_t epoch,
                                                                     uint32_t ntiles) {
    __shared__ uint32_t s_tile, s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(ctl, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const size_t base = (size_t)tile * kScanTile + (size_t)threadIdx.x * kScanPer;
    uint32_t v[kScanPer], local = 0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        v[j] = base + j < n ? in[base + j] : 0u;
        local += v[j];
    }
    uint32_t agg;
    const uint32_t excl = block_excl_sum<kScanThreads>(local, &agg);
    if (threadIdx.x < 32) {
        const uint32_t pre = tile_lookback(status, tile, agg, epoch);
        if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    uint32_t run = s_prefix + excl;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        if (base + j < n) out[base + j] = run;
        run += v[j];
    }
    if (threadIdx.x == 0 && atomicAdd(ctl + 1, 1u) == ntiles - 1) {
        ctl[0] = 0;
        ctl[1] = 0;
    }
}

// digit histogram of one tile, digit-major into hist[d * ntiles + tile]
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const unsigned long long* __restrict__ keys,
                                                                  size_t n, int shift, uint32_t ntiles,
                                                                  uint32_t* __restrict__ hist) {
    __shared__ uint32_t cnt[kRadix];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = (size_t)blockIdx.x * kSortTile;
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const size_t i = base + (size_t)r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(uint32_t)(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

// stable scatter: item i of the tile goes to the scanned (digit, tile) base
// plus its rank among the tile's items with the same digit before it
__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals, size_t n, int shift,
    uint32_t ntiles, const uint32_t* __restrict__ offs, unsigned long long* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out) {
    constexpr int NW = kSortThreads / 32;
    __shared__ uint32_t base_d[kRadix];
    __shared__ uint32_t wcnt[NW][kRadix];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    base_d[threadIdx.x] = offs[(size_t)threadIdx.x * ntiles + blockIdx.x];
    const size_t tile0 = (size_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
#pragma unroll
        for (int j = 0; j < NW; ++j) wcnt[j][threadIdx.x] = 0;
        __syncthreads();
        const size_t i = tile0 + (size_t)r * kSortThreads + threadIdx.x;
        const bool live = i < n;
        unsigned long long k = 0;
        uint32_t val = 0, d = 0xFFFFFFFFu;
        if (live) {
            k = keys[i];
            val = vals[i];
            d = (uint32_t)(k >> shift) & 255u;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        if (live && rank == 0) wcnt[w][d] = __popc(peers);
        __syncthreads();
        if (live) {
            uint32_t before = 0;
            for (int j = 0; j < w; ++j) before += wcnt[j][d];
            const uint32_t pos = base_d[d] + before + rank;
            keys_out[pos] = k;
            vals_out[pos] = val;
        }
        __syncthreads();
        uint32_t add = 0;
#pragma unroll
        for (int j = 0; j < NW; ++j) add += wcnt[j][threadIdx.x];
        base_d[threadIdx.x] += add;
        __syncthreads();
    }
}

}  // namespace

// per-context look-back state (contexts are externally synchronised)
struct igs_scan_state {
    unsigned long long* status = nullptr;
    uint32_t* ctl = nullptr;
    size_t tiles = 0;
    uint32_t epoch = 0;
};
using ScanState = igs_scan_state;

static ScanState& scan_state(igs_ctx* ctx) {
    if (!ctx->scan_st) ctx->scan_st = new igs_scan_state;
    return *ctx->scan_st;
}

int igs_scan_excl_u32(igs_ctx* ctx, const uint32_t* in, uint32_t* out, size_t n) {
    if (n == 0) return IGS_OK;
    ScanState& S = scan_state(ctx);
    const size_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles > 0xFFFFFFFFull) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "scan too large");
    if (tiles > S.tiles) {
        cudaFree(S.status);
        S.status = nullptr;
        S.tiles = 0;
        if (cudaMalloc(&S.status, tiles * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            return igs_fail(ctx, IGS_E_CUDA, "out of device memory (scan)");
        }
        // fresh words carry epoch 0, which no call uses
        IGS_CUDA(ctx, cudaMemsetAsync(S.status, 0, tiles * sizeof(unsigned long long), ctx->stream));
        S.tiles = tiles;
    }
    if (!S.ctl) {
        if (cudaMalloc(&S.ctl, 2 * sizeof(uint32_t)) != cudaSuccess) {
            cudaGetLastError();
            return igs_fail(ctx, IGS_E_CUDA, "out of device memory (scan)");
        }
        IGS_CUDA(ctx, cudaMemsetAsync(S.ctl, 0, 2 * sizeof(uint32_t), ctx->stream));
    }
    S.epoch = S.epoch % 0x3FFFFFFFu + 1;  // 1 .. 2^30 - 1
    scan_lookback_kernel<<<(unsigned)tiles, kScanThreads, 0, ctx->stream>>>(in, out, n, S.status, S.ctl, S.epoch,
                                                                             (uint32_t)tiles);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

void igs_scan_free(igs_ctx* ctx) {
    if (!ctx->scan_st) return;
    cudaFree(ctx->scan_st->status);
    cudaFree(ctx->scan_st->ctl);
    delete ctx->scan_st;
    ctx->scan_st = nullptr;
}

int igs_radix_sort_u64_u32(igs_ctx* ctx, const unsigned long long* keys_in, const uint32_t* vals_in,
                           unsigned long long* keys_out, uint32_t* vals_out, unsigned long long* keys_tmp,
                           uint32_t* vals_tmp, size_t n, int bits) {
    if (n == 0) return IGS_OK;
    const int passes = std::max(1, (bits + 7) / 8);
    const size_t tiles = (n + kSortTile - 1) / kSortTile;
    uint32_t* hist = (uint32_t*)igs_scratch(ctx, 41, tiles * kRadix * sizeof(uint32_t));
    if (!hist) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (sort)");
    const unsigned long long* ks = keys_in;
    const uint32_t* vs = vals_in;
    for (int p = 0; p < passes; ++p) {
        // the last pass lands in *_out; earlier ones alternate so that holds
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        unsigned long long* kd = to_out ? keys_out : keys_tmp;
        uint32_t* vd = to_out ? vals_out : vals_tmp;
        radix_hist_kernel<<<(unsigned)tiles, kSortThreads, 0, ctx->stream>>>(ks, n, 8 * p, (uint32_t)tiles, hist);
        IGS_LAUNCHED(ctx);
        int e;
        if ((e = igs_scan_excl_u32(ctx, hist, hist, tiles * kRadix))) return e;
        radix_scatter_kernel<<<(unsigned)tiles, kSortThreads, 0, ctx->stream>>>(ks, vs, n, 8 * p, (uint32_t)tiles,
                                                                                hist, kd, vd);
        IGS_LAUNCHED(ctx);
        ks = kd;
        vs = vd;
    }
    return IGS_OK;
}

extern "C" {

// diagnostics for the tests: the device scan and sort on host arrays
int igs_debug_scan(igs_ctx* ctx, const uint32_t* in, uint32_t n, uint32_t* out) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (n == 0) return IGS_OK;
    uint32_t* d = (uint32_t*)igs_scratch(ctx, 42, (size_t)n * 4);
    if (!d) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    IGS_CUDA(ctx, cudaMemcpyAsync(d, in, (size_t)n * 4, cudaMemcpyHostToDevice, ctx->stream));
    int e;
    if ((e = igs_scan_excl_u32(ctx, d, d, n))) return e;
    IGS_CUDA(ctx, cudaMemcpyAsync(out, d, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

int igs_debug_sort_pairs(igs_ctx* ctx, const uint64_t* keys, const uint32_t* vals, uint32_t n, int bits,
                         uint64_t* keys_out, uint32_t* vals_out) {
    if (!ctx || bits < 1 || bits > 64) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (n == 0) return IGS_OK;
    unsigned long long* dk = (unsigned long long*)igs_scratch(ctx, 43, (size_t)n * 8 * 3);
    uint32_t* dv = (uint32_t*)igs_scratch(ctx, 44, (size_t)n * 4 * 3);
    if (!dk || !dv) return igs_fail(ctx, IGS_E_CUDA, "out of device memory");
    IGS_CUDA(ctx, cudaMemcpyAsync(dk, keys, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    IGS_CUDA(ctx, cudaMemcpyAsync(dv, vals, (size_t)n * 4, cudaMemcpyHostToDevice, ctx->stream));
    int e;
    if ((e = igs_radix_sort_u64_u32(ctx, dk, dv, dk + n, dv + n, dk + 2 * (size_t)n, dv + 2 * (size_t)n, n, bits)))
        return e;
    IGS_CUDA(ctx, cudaMemcpyAsync(keys_out, dk + n, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaMemcpyAsync(vals_out, dv + n, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    IGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

}  // extern "C"
