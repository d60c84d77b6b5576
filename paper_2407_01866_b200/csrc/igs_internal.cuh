// igs_internal.cuh -- shared device records, context and helpers.
//
// Data layout in HBM (all device-resident across calls, grow-only):
//   params   double[n][8]   the reference's Gaussian2D records (64 B/G)
//   scan     ScanRec[n]     48 B: the ScanGaussian fields the top-K scan reads
//                           (renderer.hpp:31-34), 16-B aligned for LDG.128
//   shade    ShadeRec[n]    48 B: color + 1/s for blend and gradients
//   grads    double[n][8]   GaussianGrad records (renderer.hpp:95-100)
//   m, v     double[n][8]   Adam moments in record order (adam.hpp:20-31)
//   image    float[H][W][3] last render; target float[H][W][3]
// Compiled with -fmad=false: every double operation on a parity path rounds
// like the reference's SSE2 code; FMAs only where written explicitly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cstdlib>

#include <string>
#include <vector>

#include "../../include/igs_b200.h"
#include "igs_math.cuh"
#include "glibc_math.cuh"

#ifndef IGS_NO_NCCL
#include <nccl.h>
#endif

namespace igs_dev {

constexpr double kNormEps = 1e-8;   // renderer.hpp:14
constexpr double kScaleMin = 1e-4;  // gaussian.hpp:12
constexpr double kScaleMax = 2.0;   // gaussian.hpp:13
constexpr double kPi = 3.141592653589793;
constexpr uint32_t kNoIdx = 0xFFFFFFFFu;

struct __align__(16) ScanRec {
    double mu_x, mu_y, cos_t, sin_t, inv_a, inv_b;
};
struct __align__(16) ShadeRec {
    double r, g, b, inv_s1, inv_s2, pad;
};
static_assert(sizeof(ScanRec) == 48, "ScanRec");
static_assert(sizeof(ShadeRec) == 48, "ShadeRec");

// PreparedSet entry of Gaussian i (renderer.cpp:37-50): glibc's sincos
// (glibc_math.cuh, bit-identical to the reference's std::cos/std::sin), IEEE
// reciprocals; writes both records and returns the scan one.
__device__ __forceinline__ ScanRec prepare_one(const double* __restrict__ params, uint32_t i,
                                               ScanRec* __restrict__ scan, ShadeRec* __restrict__ shade) {
    const double2* p2 = reinterpret_cast<const double2*>(params + (size_t)i * 8);
    const double2 a = p2[0], b = p2[1], c = p2[2], d = p2[3];
    double s, co;
    glibc_math::sincos(b.x, &s, &co);
    const double inv_s1 = __ddiv_rn(1.0, b.y);
    const double inv_s2 = __ddiv_rn(1.0, c.x);
    ScanRec r;
    r.mu_x = a.x;
    r.mu_y = a.y;
    r.cos_t = co;
    r.sin_t = s;
    r.inv_a = __dmul_rn(inv_s1, inv_s1);
    r.inv_b = __dmul_rn(inv_s2, inv_s2);
    scan[i] = r;
    ShadeRec h;
    h.r = c.y;
    h.g = d.x;
    h.b = d.y;
    h.inv_s1 = inv_s1;
    h.inv_s2 = inv_s2;
    h.pad = 0.0;
    shade[i] = h;
    return r;
}

// renderer.cpp:17-23 mahalanobis_sq, each op rounded separately (no FMA).
__device__ __forceinline__ double maha(const ScanRec& g, double x, double y) {
    const double dx = __dsub_rn(x, g.mu_x);
    const double dy = __dsub_rn(y, g.mu_y);
    const double e1 = __dadd_rn(__dmul_rn(g.cos_t, dx), __dmul_rn(g.sin_t, dy));
    const double e2 = __dadd_rn(__dmul_rn(-g.sin_t, dx), __dmul_rn(g.cos_t, dy));
    return __dadd_rn(__dmul_rn(__dmul_rn(e1, e1), g.inv_a), __dmul_rn(__dmul_rn(e2, e2), g.inv_b));
}

// Register-resident top-K, sorted ascending by (q, idx) -- the strict total
// order of select_top_k_entries (renderer.cpp:53-74).  Because the order is
// total, the kept set and its order do not depend on scan order, so any
// candidate order (tile lists, split scans) yields the reference's result.
//
// Layout: the kk live slots are the LAST kk of KCAP registers; the first
// KCAP-kk hold a (-inf, 0) sentinel that compares below every candidate and
// therefore never moves.  The current worst kept entry is always slot
// KCAP-1, a static register index (a runtime "slot kk-1" would force the
// array into local memory).  Unfilled live slots hold (+inf, kNoIdx).
template <int KCAP>
struct TopK {
    double q[KCAP];
    uint32_t i[KCAP];
    int off;  // = KCAP - kk: first live slot

    __device__ __forceinline__ void init(int kk) {
        off = KCAP - kk;
#pragma unroll
        for (int j = 0; j < KCAP; ++j) {
            const bool dead = j < off;
            q[j] = __longlong_as_double(dead ? (long long)0xfff0000000000000ULL : 0x7ff0000000000000LL);
            i[j] = dead ? 0u : kNoIdx;
        }
    }
    __device__ __forceinline__ double tq() const { return q[KCAP - 1]; }
    __device__ __forceinline__ bool beats(double cq, uint32_t ci) const {
        return cq < q[KCAP - 1] || (cq == q[KCAP - 1] && ci < i[KCAP - 1]);
    }
    // The list is ascending in the (q, idx) order, so lt[j] = (cand < slot j)
    // is monotone in j: slot j takes slot j-1 if the candidate went above it,
    // else the candidate if it goes here, else keeps its own.  All compares
    // read the old list and the slots update in place from the top down, so
    // there is no carried value (no branches, no register rotation).
    __device__ __forceinline__ void insert(double cq, uint32_t ci) {
        bool lt[KCAP];
#pragma unroll
        for (int j = 0; j < KCAP; ++j) lt[j] = (cq < q[j]) | ((cq == q[j]) & (ci < i[j]));
#pragma unroll
        for (int j = KCAP - 1; j > 0; --j) {
            q[j] = lt[j - 1] ? q[j - 1] : (lt[j] ? cq : q[j]);
            i[j] = lt[j - 1] ? i[j - 1] : (lt[j] ? ci : i[j]);
        }
        q[0] = lt[0] ? cq : q[0];
        i[0] = lt[0] ? ci : i[0];
    }
    __device__ __forceinline__ void offer(double cq, uint32_t ci) {
        if (beats(cq, ci)) insert(cq, ci);
    }
    // j-th best (0-based) lives in slot off + j.
    __device__ __forceinline__ bool live(int slot) const { return slot >= off && i[slot] != kNoIdx; }
};

// blend_entries (renderer.cpp:76-89) over the kept entries, best first.
template <int KCAP>
__device__ __forceinline__ double blend_topk(const TopK<KCAP>& t, const ShadeRec* __restrict__ shade, double* c) {
    double total = 0.0, ar = 0.0, ag = 0.0, ab = 0.0;
#pragma unroll
    for (int j = 0; j < KCAP; ++j) {
        if (t.live(j)) {
            const double w = glibc_math::exp(__dmul_rn(-0.5, t.q[j]));
            const ShadeRec s = shade[t.i[j]];
            total = __dadd_rn(total, w);
            ar = __dadd_rn(ar, __dmul_rn(w, s.r));
            ag = __dadd_rn(ag, __dmul_rn(w, s.g));
            ab = __dadd_rn(ab, __dmul_rn(w, s.b));
        }
    }
    const double inv = __ddiv_rn(1.0, __dadd_rn(kNormEps, total));
    c[0] = __dmul_rn(ar, inv);
    c[1] = __dmul_rn(ag, inv);
    c[2] = __dmul_rn(ab, inv);
    return total;
}

// Writes the kk kept entries best-first to dq/di (either nullable).
template <int KCAP>
__device__ __forceinline__ void store_topk(const TopK<KCAP>& t, double* dq, uint32_t* di) {
#pragma unroll
    for (int j = 0; j < KCAP; ++j)
        if (j >= t.off) {
            if (dq) dq[j - t.off] = t.q[j];
            if (di) di[j - t.off] = t.i[j];
        }
}

__device__ __forceinline__ float clamp01f(double v) { return (float)(v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v)); }

// pixel_center (image.hpp:18-20)
__device__ __forceinline__ double center(int i, int n) { return __ddiv_rn(__dadd_rn((double)i, 0.5), (double)n); }

// Arguments of the deterministic reduction's offsets + slot scatter (reduce.cuh).
struct OffArgs {
    const uint32_t* gcnt;  // per-Gaussian counts | [n, 2n) cursors
    uint32_t n;
    uint32_t* goff;
    uint32_t* chunk_sum;   // gridDim.x entries
    const uint32_t* keys;
    uint32_t items;
    uint32_t* gcur;
    uint32_t* perm;
    uint32_t* long_count;
    uint32_t* long_list;
    unsigned* bar;         // [0] arrivals, [1] exits
    // bucket mode (reduce.cuh; null: CSR of every segment): this
    // iteration's [0] overflow entries, [1] allocation cursor, and the
    // (slot, rank) pairs of the overflow entries
    uint32_t* ovf;
    const uint32_t* ovf_list;
};

// Long segments (more than kShortSeg contributions) and the loss (reduce.cuh:
// long_segments, loss_chunk).
struct LongArgs {
    const uint32_t* gcnt;
    const uint32_t* goff;
    const uint32_t* perm;
    const double* contrib;
    double* grads;
    const uint32_t* long_count;
    const uint32_t* long_list;
    long long* status;
    uint32_t* big;            // scratch beyond shared memory (items entries)
    const double* losses;
    uint32_t ns;
    double inv_n;
    double* dloss;            // null: no loss
    double* loss_part;        // kLossCtas partials, then the combining ticket
    unsigned* loss_ticket;
    const uint32_t* bucket;   // bucket mode: ranks < kBucket live there
};

}  // namespace igs_dev

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct PartitionDev;  // bsp.cu

// The start of a training iteration -- status reset, plus the sample
// indices copied from pinned host memory or drawn from raw engine outputs --
// run by the first kernel of the step (the kNN tree refit) instead of a
// launch of its own; igs_stage_launch runs it standalone when no such kernel
// follows.
struct StageJob {
    int kind = 0;  // 0 none, 1 status reset, 2 + copy host indices, 3 + draw from host raw outputs
    long long* status = nullptr;
    const void* host = nullptr;
    uint32_t* dsidx = nullptr;
    uint32_t ns = 0;
    const double* prob = nullptr;
    const uint32_t* alias = nullptr;
    unsigned long long table_n = 0;
};

#ifdef __CUDACC__
__device__ __forceinline__ void stage_job_run(const StageJob& J, uint32_t tid, uint32_t nthr) {
    if (J.kind == 0) return;
    if (tid < 4) J.status[tid] = tid == 3 ? 0 : LLONG_MAX;  // status[3]: a count (kNN tree growth)
    if (J.kind == 1) return;
    for (uint32_t i = tid; i < J.ns; i += nthr) {
        uint32_t v;
        if (J.kind == 2) {
            v = static_cast<const uint32_t*>(J.host)[i];
        } else {
            // AliasTable::sample (sampling.cpp:126-133), as draw_stage_kernel
            const unsigned long long* raw = static_cast<const unsigned long long*>(J.host);
            const unsigned long long r0 = raw[2 * (size_t)i], r1 = raw[2 * (size_t)i + 1];
            const unsigned long long j = r0 % J.table_n;
            const double coin = (double)(r1 >> 11) * 0x1.0p-53;
            v = coin < J.prob[j] ? (uint32_t)j : J.alias[j];
        }
        J.dsidx[i] = v;
    }
}
#endif

struct igs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;                   // off-critical-path work (loss sum)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;
    uint64_t launches = 0;
    int sm_count = 148;

    // options
    int opt_cull = 1;
    int opt_deterministic = 1;
    int opt_shard_adam = 1;  // multi-rank exchange: each rank updates its slice of the set, then an all-gather
    int opt_tile = 16;
    int opt_raster = 0;  // IGS_OPT_RASTER

    // set
    uint32_t n = 0;
    uint32_t cap = 0;
    double* params = nullptr;
    double* grads = nullptr;
    double* adam_m = nullptr;
    double* adam_v = nullptr;
    igs_dev::ScanRec* scan = nullptr;
    igs_dev::ShadeRec* shade = nullptr;
    bool grads_valid = false;
    bool grads_checked = false;  // the reduction already flagged non-finite gradients

    // images
    DevBuf image;
    int img_w = 0, img_h = 0;
    DevBuf target;
    int tgt_w = 0, tgt_h = 0;

    // per-call scratch (grow-only), indexed by purpose
    DevBuf scratch[48];
    // pinned host staging
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    // device status word block: [0] error code flag, [1] first bad slot
    long long* status = nullptr;

    // pinned staging of the async iteration (igs_train_iteration_async)
    // (two slots: [slot] samples, [2 + slot] result block, [4 + slot] the
    // per-sample losses, and a completion event per slot)
    DevBuf async_pin[6];
    uint32_t async_ns[2] = {0, 0};  // samples (all ranks) of the iteration in each slot
    // host-mapped buffer the search epilogue mirrors the per-sample losses
    // into (set around one igs_forward_backward call; loss_mirrored reports
    // whether that call's search wrote it)
    double* loss_mirror = nullptr;
    bool loss_mirrored = false;
    cudaEvent_t async_ev[2] = {nullptr, nullptr};
    StageJob stage_job;          // handed from igs_forward_backward to knn_build (see StageJob)
    struct {
        igs_dev::OffArgs args;   // reduce.cuh: offsets + scatter the kNN launch may take over
        bool ready = false, done = false;
        uint32_t* bucket = nullptr;    // [n][kBucket] slot ids per Gaussian (search epilogue)
        uint32_t* ovf = nullptr;       // this iteration's counters: overflow entries, allocation, long segments
        uint32_t* ovf_list = nullptr;  // (slot, rank) of every overflow entry
        uint32_t* long_list = nullptr; // Gaussians with more than kBucket contributions
        uint32_t* ovf_zero = nullptr;  // the next iteration's counters, zeroed by the search
        igs_dev::LongArgs long_args;   // bucket mode: the long segments + loss ride in the same launch
        bool fuse_long = false;
    } fuse_off;
    bool ovf_ready = false;  // the counter pair (scratch 47) zeroed
    int ovf_phase = 0;
    bool off_ctl_ready = false;  // its barrier counters zeroed (scratch 34)
    bool loss_ticket_ready = false;  // long_segment_kernel's loss ticket zeroed (scratch 35)
    int async_head = 0, async_count = 0;

    // the fit driver's sampling distribution (alias table) on the device
    DevBuf alias_prob, alias_idx;
    uint64_t alias_n = 0;

    // uploaded samples for device-resident training
    DevBuf samples;
    uint32_t samples_ns = 0, samples_steps = 0;

    PartitionDev* part = nullptr;
    PartitionDev* part_spare = nullptr;  // a replaced partition's device arrays, reused by the next
    void* cull = nullptr;            // CullBufs (cull.cu)
    void* knn = nullptr;             // KnnBufs (knn.cu)
    uint64_t params_version = 0;     // bumped on every change of the set
    long long knn_grown = -1;        // status[3] of the last step read back (-1: unknown)
    bool exchanged = false;          // the last forward/backward gathered every rank's contributions
    const void* gcnt_clean = nullptr;  // deterministic-reduction counters left zeroed (for this n)
    uint32_t gcnt_clean_n = 0;

    // profiling (igs_profile_*)
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_ev[IGS_PROF_FAMILIES];  // begin/end pairs
    double prof_work[IGS_PROF_FAMILIES] = {};
    unsigned long long* prof_dev_work = nullptr;  // device work counters (pairs) per family
    cudaEvent_t timer[2] = {nullptr, nullptr};
    bool timer_armed = false;     // igs_timer_begin called, stop not yet recorded
    bool timer_stopped = false;   // stop event already recorded by a device loop
    DevBuf flush;
    int flush_salt = 0;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<cudaEvent_t> marks;  // igs_timer_mark

#ifndef IGS_NO_NCCL
    ncclComm_t comm = nullptr;
#endif
    struct igs_loop_group* loop = nullptr;  // in-process loopback group (comm.cu)
    bool moments_local = false;  // sharded update: only this rank's slice of adam_m/adam_v is current
    struct igs_scan_state* scan_st = nullptr;  // scan.cu: device scan look-back state
    int nranks = 1, rank = 0;
};

// comm.cu: the multi-rank transport (NCCL or the in-process loopback group)
inline bool igs_has_comm(const igs_ctx* ctx) {
#ifndef IGS_NO_NCCL
    if (ctx->comm) return true;
#endif
    return ctx->loop != nullptr;
}
int igs_comm_allgather(igs_ctx* ctx, void* buf, size_t bytes);
int igs_comm_allreduce_sum(igs_ctx* ctx, double* buf, size_t count);
void igs_comm_release(igs_ctx* ctx);
void igs_scan_free(igs_ctx* ctx);

// helpers implemented in ctx.cu
int igs_fail(igs_ctx* ctx, int code, const std::string& msg);
int igs_cuda_check(igs_ctx* ctx, cudaError_t e, const char* what);
void* igs_scratch(igs_ctx* ctx, int slot, size_t bytes);
void* igs_pinned(igs_ctx* ctx, size_t bytes);
int igs_ensure_image(igs_ctx* ctx, int w, int h);

#define IGS_LAUNCHED(ctx)                                                   \
    do {                                                                    \
        (ctx)->launches++;                                                  \
        cudaError_t _e = cudaGetLastError();                                \
        if (_e != cudaSuccess) return igs_cuda_check((ctx), _e, "launch");  \
    } while (0)

#ifdef __CUDACC__
// Grid-wide barrier for a persistent launch whose CTAs are all co-resident
// (one per SM): arrivals counted in *bar (release), spun on (acquire) until
// `target`; callers count targets G, 2G, ... and reset *bar at the end.
__device__ __forceinline__ void igs_grid_sync(unsigned* bar, unsigned target) {
    __syncthreads();  // the CTA's writes are ordered before thread 0's release
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}
#endif

// train.cu: a StageJob as its own launch
int igs_stage_launch(igs_ctx* ctx, const StageJob& J);

// L2 prefetch of data a LATER kernel of the same step reads: a kernel that is
// itself latency-bound spreads fire-and-forget prefetches over its threads
// so the follower's first touch hits L2 instead of DRAM.
struct L2Prefetch {
    const char* p[4];
    uint32_t lines[4];  // 128-byte lines per range
    int nr;
};

inline void l2pf_add(L2Prefetch& pf, const void* p, size_t bytes) {
    if (!p || !bytes || pf.nr >= 4) return;
    pf.p[pf.nr] = static_cast<const char*>(p);
    pf.lines[pf.nr] = (uint32_t)((bytes + 127) / 128);
    pf.nr++;
}

__device__ __forceinline__ void prefetch_l2(const L2Prefetch& pf, uint32_t tid, uint32_t nthr) {
    for (int r = 0; r < pf.nr; ++r)
        for (uint32_t l = tid; l < pf.lines[r]; l += nthr)
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(pf.p[r] + (size_t)l * 128));
}

// Programmatic dependent launch: a kernel launched with IGS_PDL may be
// scheduled while its stream predecessor drains (hiding launch latency); it
// must execute pdl_wait() before it reads or writes any memory a
// predecessor touches.  Without the launch attribute pdl_wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the stream successor (launched with IGS_PDL) be scheduled before this
// grid completes: once every CTA has executed it (or exited), the
// successor's CTAs may become resident and run up to their pdl_wait, which
// still waits for this grid's completion and memory.  A CTA calls it when
// its remaining work is short.  Used by lq_tree_kernel only: the same
// trigger in the search (+0.0 %) and in the hard-point/offsets launch
// (-6 %: Adam's CTAs then crowd the SMs while it runs) measured no gain.
// (IGS_NO_PDL_TRIGGER: compiled out, A/B.)
__device__ __forceinline__ void pdl_trigger() {
#ifndef IGS_NO_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t igs_launch_pdl(cudaStream_t st, bool coop, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    // coop (IGS_COOP_BARRIERS): the driver guarantees every CTA is
    // co-resident or fails the launch (cudaErrorCooperativeLaunchTooLarge)
    // instead of letting a grid barrier spin forever
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = coop ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

#define IGS_PDL(ctx, kernel, grid, block, smem, ...)                                                        \
    do {                                                                                                    \
        cudaError_t _e =                                                                                    \
            igs_launch_pdl((ctx)->stream, false, kernel, dim3(grid), dim3(block), (smem), __VA_ARGS__);     \
        (ctx)->launches++;                                                                                  \
        if (_e != cudaSuccess) return igs_cuda_check((ctx), _e, #kernel);                                   \
    } while (0)
// a persistent launch with grid barriers: cooperative + PDL
// Launches of kernels with grid barriers (igs_grid_sync).  Their grids are
// sized from the occupancy calculator (at most the co-resident CTAs per SM
// times the SM count), and every CTA passes pdl_wait only after the
// predecessor has left the GPU, so they are co-resident without the
// cooperative attribute -- which costs ~3 us of chain time per launch
// (C2 step 92.5 -> 89.7 us measured for the hard-point/offsets launch).
// With a communicator attached (several ranks' grids may share a GPU, as
// in the loopback tests) or IGS_COOP_BARRIERS=1 they are cooperative
// launches: the driver then schedules each grid whole (and under MPS,
// where fewer SMs may be available than the device reports, fails rather
// than hangs).
// Likewise when several contexts are alive in the process (their streams
// could run two barrier grids side by side).
extern "C" int igs_live_contexts();  // ctx.cu
inline bool igs_coop_barriers() {
    static const bool v = getenv("IGS_COOP_BARRIERS") != nullptr;
    return v || igs_live_contexts() > 1;
}

#define IGS_PDL_COOP(ctx, kernel, grid, block, smem, ...)                                                   \
    do {                                                                                                    \
        cudaError_t _e = igs_launch_pdl((ctx)->stream, igs_coop_barriers() || igs_has_comm(ctx), kernel,      \
                                        dim3(grid), dim3(block),                                            \
                                        (smem), __VA_ARGS__);                                               \
        (ctx)->launches++;                                                                                  \
        if (_e != cudaSuccess) return igs_cuda_check((ctx), _e, #kernel);                                   \
    } while (0)

#define IGS_CUDA(ctx, call)                                                 \
    do {                                                                    \
        cudaError_t _e = (call);                                            \
        if (_e != cudaSuccess) return igs_cuda_check((ctx), _e, #call);     \
    } while (0)

// profiling helpers (prof.cu): bracket a family's launches
void igs_prof_begin(igs_ctx* ctx, int fam);
void igs_prof_end(igs_ctx* ctx, int fam, double host_work);
unsigned long long* igs_prof_counter(igs_ctx* ctx, int fam);  // nullptr unless profiling
// records the armed timer's stop event right after a device loop's last kernel
void igs_timer_autostop(igs_ctx* ctx);

// internal entry points shared between translation units
int igs_prepare_all(igs_ctx* ctx, uint32_t first);
int igs_raster_global(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* dev_out, uint32_t* dev_topk);
int igs_topk_points(igs_ctx* ctx, const double* dev_uv, uint32_t npts, int k, uint32_t* dev_idx, double* dev_q);
int igs_blocked_points_dev(igs_ctx* ctx, const double* duv, uint32_t npts, int kk, double* drgb);
extern "C" int igs_blocked_render_rows(igs_ctx* ctx, int width, int height, int k, int row0, int row1);

int igs_partition_free(igs_ctx* ctx);
void igs_partition_release(igs_ctx* ctx);
void igs_cull_free(igs_ctx* ctx);
void igs_knn_free(igs_ctx* ctx);
int igs_topk_knn(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq);
int igs_raster_knn(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out, uint32_t* topk);
int igs_knn_forward_backward(igs_ctx* ctx, int mode, const uint32_t* sidx, const double* samples5, uint32_t npts,
                             int kk, double inv_n, double* losses, double* contrib, uint32_t* keys, uint32_t* gcnt,
                             double* grads_atomic, uint32_t* zero_word = nullptr,
                             const L2Prefetch* pf = nullptr, int defer_loss_check = 0);
int igs_comm_allgather(igs_ctx* ctx, void* buf, size_t bytes);
L2Prefetch igs_knn_tree_inputs(igs_ctx* ctx);
int igs_topk_samples_culled(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq);
int igs_topk_pixels_culled(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq, int W,
                           int H);
