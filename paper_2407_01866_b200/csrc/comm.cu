// comm.cu -- the multi-rank transport of the training exchange.
//
// Two transports carry the same two collectives (in-place all-gather of
// equal rank blocks; sum all-reduce of doubles):
//
//  * NCCL over NVLink / NVSwitch, one communicator per context (one process
//    or host thread per GPU, igs_comm_init).  NCCL is resolved with dlopen
//    at first use: the process may already hold a libnccl.so.2 (torch's
//    bundled one when torch.distributed is the plumbing), and linking the
//    system one at load time would shadow it.
//  * an in-process loopback group (igs_comm_init_loopback), for testing the
//    R-rank exchange where only one device exists: NCCL rejects two ranks on
//    one GPU.  The ranks' host threads meet at a barrier per collective; each
//    rank then enqueues, on its own stream and after the peer's "ready" event,
//    one cudaMemcpyAsync per peer rank block (device-to-device or peer), and
//    records "done"; a second barrier plus a wait on every peer's "done"
//    keeps a rank from overwriting its block before the peers have read it.
//    No kernel ever waits on another rank's kernel: the ordering is stream
//    events only.  The all-reduce adds the ranks' buffers in rank order, so
//    every rank computes the same bits.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "igs_internal.cuh"

#ifndef IGS_NO_NCCL
namespace {
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.allGather;
    return api;
}
}  // namespace
#endif

struct igs_loop_group {
    int nranks = 0;
    std::vector<igs_ctx*> ranks;
    std::vector<cudaEvent_t> ready, done;
    std::vector<char*> base;  // per rank: its buffer of the current collective
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0, members = 0;
    unsigned long long gen = 0;

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace {

__global__ void sum_ranks_kernel(const double* __restrict__ parts, int nranks, size_t count,
                                 double* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        double s = parts[i];
        for (int r = 1; r < nranks; ++r) s = __dadd_rn(s, parts[(size_t)r * count + i]);
        out[i] = s;
    }
}

// one loopback exchange: every rank publishes `mine`, then copies what it
// needs from the peers with `pull(peer, peer_base)`
template <class Pull>
int loop_exchange(igs_ctx* ctx, char* mine, Pull pull) {
    igs_loop_group* g = ctx->loop;
    const int me = ctx->rank;
    IGS_CUDA(ctx, cudaEventRecord(g->ready[me], ctx->stream));
    g->base[me] = mine;
    g->barrier();
    for (int p = 0; p < g->nranks; ++p) {
        if (p == me) continue;
        IGS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, g->ready[p], 0));
        int e;
        if ((e = pull(p, g->base[p]))) return e;
    }
    IGS_CUDA(ctx, cudaEventRecord(g->done[me], ctx->stream));
    g->barrier();
    for (int p = 0; p < g->nranks; ++p)
        if (p != me) IGS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, g->done[p], 0));
    return IGS_OK;
}

}  // namespace

// In-place all-gather: rank r's block is buf[r * bytes, (r + 1) * bytes).
int igs_comm_allgather(igs_ctx* ctx, void* buf, size_t bytes) {
    char* b = static_cast<char*>(buf);
    if (ctx->loop) {
        return loop_exchange(ctx, b, [&](int p, char* peer) -> int {
            IGS_CUDA(ctx, cudaMemcpyAsync(b + (size_t)p * bytes, peer + (size_t)p * bytes, bytes, cudaMemcpyDefault,
                                          ctx->stream));
            return IGS_OK;
        });
    }
#ifndef IGS_NO_NCCL
    if (!ctx->comm) return IGS_OK;
    if (nccl().allGather(b + (size_t)ctx->rank * bytes, b, bytes, ncclChar, ctx->comm, ctx->stream) != ncclSuccess)
        return igs_fail(ctx, IGS_E_CUDA, "ncclAllGather failed");
#endif
    return IGS_OK;
}

// In-place sum all-reduce of `count` doubles.
int igs_comm_allreduce_sum(igs_ctx* ctx, double* buf, size_t count) {
    if (ctx->loop) {
        const int R = ctx->nranks;
        double* parts = (double*)igs_scratch(ctx, 10, (size_t)R * count * sizeof(double));
        if (!parts) return igs_fail(ctx, IGS_E_CUDA, "out of device memory (all-reduce)");
        IGS_CUDA(ctx, cudaMemcpyAsync(parts + (size_t)ctx->rank * count, buf, count * sizeof(double),
                                      cudaMemcpyDeviceToDevice, ctx->stream));
        int e = loop_exchange(ctx, (char*)buf, [&](int p, char* peer) -> int {
            IGS_CUDA(ctx, cudaMemcpyAsync(parts + (size_t)p * count, peer, count * sizeof(double), cudaMemcpyDefault,
                                          ctx->stream));
            return IGS_OK;
        });
        if (e) return e;
        sum_ranks_kernel<<<(unsigned)std::min<size_t>(4 * ctx->sm_count, (count + 255) / 256), 256, 0, ctx->stream>>>(
            parts, R, count, buf);
        IGS_LAUNCHED(ctx);
        return IGS_OK;
    }
#ifndef IGS_NO_NCCL
    if (!ctx->comm) return IGS_OK;
    if (nccl().allReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream) != ncclSuccess)
        return igs_fail(ctx, IGS_E_CUDA, "ncclAllReduce failed");
#endif
    return IGS_OK;
}

void igs_comm_release(igs_ctx* ctx) {
#ifndef IGS_NO_NCCL
    if (ctx->comm) nccl().commDestroy(ctx->comm);
    ctx->comm = nullptr;
#endif
    if (igs_loop_group* g = ctx->loop) {
        ctx->loop = nullptr;
        bool last;
        {
            std::lock_guard<std::mutex> lk(g->mu);
            last = --g->members == 0;
        }
        if (last) {
            for (auto e : g->ready) cudaEventDestroy(e);
            for (auto e : g->done) cudaEventDestroy(e);
            delete g;
        }
    }
    ctx->nranks = 1;
    ctx->rank = 0;
}

extern "C" {

int igs_comm_unique_id(uint8_t id[128]) {
#ifndef IGS_NO_NCCL
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    if (!nccl().ok || nccl().getUniqueId(&u) != ncclSuccess) return IGS_E_CUDA;
    std::memcpy(id, &u, 128);
    return IGS_OK;
#else
    (void)id;
    return IGS_E_CUDA;
#endif
}

int igs_comm_init(igs_ctx* ctx, const uint8_t id[128], int nranks, int rank) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    cudaSetDevice(ctx->device);
    if (nranks < 1 || rank < 0 || rank >= nranks) return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "bad rank");
#ifndef IGS_NO_NCCL
    if (!nccl().ok) return igs_fail(ctx, IGS_E_CUDA, "libnccl.so.2 not found");
    igs_comm_release(ctx);
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (nccl().commInitRank(&ctx->comm, nranks, u, rank) != ncclSuccess)
        return igs_fail(ctx, IGS_E_CUDA, "ncclCommInitRank failed");
    ctx->nranks = nranks;
    ctx->rank = rank;
    return IGS_OK;
#else
    (void)id;
    return igs_fail(ctx, IGS_E_CUDA, "built without NCCL");
#endif
}

int igs_comm_init_loopback(igs_ctx** ctxs, int nranks) {
    if (!ctxs || nranks < 1) return IGS_E_INVALID_PARAMETER;
    for (int r = 0; r < nranks; ++r)
        if (!ctxs[r]) return IGS_E_INVALID_PARAMETER;
    auto* g = new igs_loop_group;
    g->nranks = nranks;
    g->members = nranks;
    g->ranks.assign(ctxs, ctxs + nranks);
    g->ready.assign(nranks, nullptr);
    g->done.assign(nranks, nullptr);
    g->base.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
        igs_ctx* c = ctxs[r];
        cudaSetDevice(c->device);
        igs_comm_release(c);
        if (cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess)
            return igs_fail(c, IGS_E_CUDA, "cudaEventCreate failed");
        c->loop = g;
        c->nranks = nranks;
        c->rank = r;
    }
    return IGS_OK;
}

int igs_comm_destroy(igs_ctx* ctx) {
    if (!ctx) return IGS_E_INVALID_PARAMETER;
    igs_comm_release(ctx);
    return IGS_OK;
}

}  // extern "C"
