// comm.cu -- NCCL plumbing for the row-partitioned multi-GPU path.
//
// Replaces the reference's in-process "device" set (distsim.hpp:77-146
// WorkerPool) and its counted reduce / broadcast (distsim.hpp:153-162
// tree_reduce, :248-252): one process per GPU, collectives over NVLink /
// NVSwitch.  NCCL is resolved with dlopen at first use (preferring the copy
// the host process -- e.g. PyTorch -- already loaded), so this library has
// no link-time dependency on a particular libnccl.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "lsqr.cuh"

namespace slq {

namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclReduce) reduce = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
        a.reduce = reinterpret_cast<decltype(a.reduce)>(dlsym(h, "ncclReduce"));
        a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
        a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.reduce && a.broadcast &&
               a.errorString;
    });
    if (!a.ok) fail(SLQ_NCCL, "NCCL library not available");
    return a;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(SLQ_NCCL, std::string(what) + ": " + api().errorString(r));
}

// Host collectives: stream sync, D2H into pinned staging, the caller's
// callback, H2D back (stream-ordered).
void host_collective(slq_ctx* ctx, double* buf, int64_t count, int (*fn)(void*, double*, int64_t)) {
    if (count > ctx->host_stage_n) {
        if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
        ctx->host_stage = nullptr;
        SLQ_CUDA_CHECK(cudaMallocHost(&ctx->host_stage, sizeof(double) * count));
        ctx->host_stage_n = count;
    }
    SLQ_CUDA_CHECK(cudaMemcpyAsync(ctx->host_stage, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (fn(ctx->host_comm.user, ctx->host_stage, count) != 0) fail(SLQ_NCCL, "host collective failed");
    SLQ_CUDA_CHECK(cudaMemcpyAsync(buf, ctx->host_stage, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    ctx->nccl_calls++;
}

}  // namespace

void comm_set_host(slq_ctx* ctx, const slq_host_comm& hc, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(SLQ_INVALID_DIMS, "set_host_comm: bad rank / size");
    if (!hc.allreduce_sum || !hc.reduce_sum_root || !hc.broadcast_root)
        fail(SLQ_INVALID_ARG, "set_host_comm: all three collectives are required");
    comm_destroy(ctx);
    ctx->host_comm = hc;
    ctx->rank = rank;
    ctx->nranks = nranks;
}

void comm_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(api().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, 128);
}

void comm_init(slq_ctx* ctx, const unsigned char id[128], int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(SLQ_INVALID_DIMS, "comm_init: bad rank / size");
    comm_destroy(ctx);
    ctx->rank = rank;
    ctx->nranks = nranks;
    // single rank: collectives are identities and are skipped, unless
    // SLQ_FORCE_NCCL asks for a real one-rank communicator (exercises the
    // NCCL path on one GPU)
    if (nranks == 1 && !slq_env_flag("SLQ_FORCE_NCCL")) return;
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    SLQ_CUDA_CHECK(cudaSetDevice(ctx->device));
    ncclComm_t c;
    nccl_check(api().commInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
    ctx->comm = c;
}

void comm_destroy(slq_ctx* ctx) {
    if (ctx->comm) api().commDestroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
    ctx->host_comm = slq_host_comm{};
    if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
    ctx->host_stage = nullptr;
    ctx->host_stage_n = 0;
}

// distsim.hpp:312-331 dist_rmatvec_and_norm's one reduction: sum of the
// per-rank {A^T u partial, ||u||^2 partial}, result on every rank.
void allreduce_sum(slq_ctx* ctx, double* buf, int64_t count) {
    if (ctx->host_comm.allreduce_sum) return host_collective(ctx, buf, count, ctx->host_comm.allreduce_sum);
    if (!ctx->comm) return;
    nccl_check(api().allReduce(buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum,
                               static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclAllReduce");
    ctx->nccl_calls++;
}

// distsim.hpp:383-396 dist_sketch_apply's reduction of d x n partials (to rank 0).
void reduce_sum_root(slq_ctx* ctx, double* buf, int64_t count) {
    if (ctx->host_comm.reduce_sum_root) return host_collective(ctx, buf, count, ctx->host_comm.reduce_sum_root);
    if (!ctx->comm) return;
    nccl_check(api().reduce(buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum, 0,
                            static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclReduce");
    ctx->nccl_calls++;
}

// The preconditioner hand-off (SPEC: worker 0 builds, everyone uses).
void broadcast_root(slq_ctx* ctx, double* buf, int64_t count) {
    if (ctx->host_comm.broadcast_root) return host_collective(ctx, buf, count, ctx->host_comm.broadcast_root);
    if (!ctx->comm) return;
    nccl_check(api().broadcast(buf, buf, static_cast<size_t>(count), ncclDouble, 0,
                               static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclBroadcast");
    ctx->nccl_calls++;
}

}  // namespace slq
