// comm.cpp — the collectives of the path: the in-place ncclAllGather of the
// grid's probe densities at each occupancy-grid update (every rank probes one
// equal block of cells; SURVEY §8e's all-reduce(max) of disjoint shards moves
// twice the bytes for the same result), ncclAllReduce(max) for callers combining
// overlapping probes, and ncclAllReduce(sum) of the voxel-field parameter
// gradients in data-parallel training (§8f rank 4).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the library loads
// (and the single-GPU path runs) on machines without NCCL. The all-reduce runs on
// the context's stream; probes are >= 0 (validated, occupancy_grid.cpp:128) so
// the f64 max equals the max of the u64 bit patterns and is exact.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "vm_internal.h"

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string load_error;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) {
            n.load_error = std::string("NCCL unavailable: ") + dlerror();
            return;
        }
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(n.h, "ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(n.h, "ncclAllGather"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
        if (!n.get_unique_id || !n.init_rank || !n.all_reduce || !n.all_gather || !n.destroy)
            n.load_error = "NCCL symbols missing";
    });
    return n;
}

int nccl_fail(ncclResult_t r, const char* where) {
    Nccl& n = nccl();
    return vmb::fail(VMB_RUNTIME, std::string("nccl error in ") + where + ": " +
                                      (n.error_string ? n.error_string(r) : "unknown"));
}

}  // namespace

extern "C" {

int vmb_comm_unique_id(void* out128) {
    Nccl& n = nccl();
    if (!n.load_error.empty()) return vmb::fail(VMB_NOT_SUPPORTED, n.load_error);
    ncclUniqueId id;
    ncclResult_t r = n.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
    return VMB_OK;
}

int vmb_comm_init(vmb_ctx* ctx, const void* id128, int nranks, int rank) {
    Nccl& n = nccl();
    if (!n.load_error.empty()) return vmb::fail(VMB_NOT_SUPPORTED, n.load_error);
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return vmb::fail(VMB_INVALID_ARGUMENT, "comm: rank out of range");
    cudaSetDevice(ctx->device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t comm;
    ncclResult_t r = n.init_rank(&comm, nranks, id, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    ctx->nccl_comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return VMB_OK;
}

int vmb_comm_destroy(vmb_ctx* ctx) {
    if (!ctx->nccl_comm) return VMB_OK;
    Nccl& n = nccl();
    cudaStreamSynchronize(ctx->stream);
    n.destroy(static_cast<ncclComm_t>(ctx->nccl_comm));
    ctx->nccl_comm = nullptr;
    ctx->nranks = 1;
    ctx->rank = 0;
    return VMB_OK;
}

int vmb_comm_allreduce_max_f64(vmb_ctx* ctx, double* buf, uint64_t count) {
    if (!ctx->nccl_comm) return VMB_OK;
    Nccl& n = nccl();
    // u64 bit patterns: order-identical to f64 for non-negative values, and max
    // over integers is exact (no NaN / signed-zero corner cases).
    ncclResult_t r = n.all_reduce(buf, buf, count, ncclUint64, ncclMax,
                                  static_cast<ncclComm_t>(ctx->nccl_comm), ctx->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    return VMB_OK;
}

int vmb_comm_allgather_f64(vmb_ctx* ctx, double* buf, uint64_t count_per_rank) {
    if (!ctx->nccl_comm) return VMB_OK;
    Nccl& n = nccl();
    // in place: rank k's block is buf[k * count, (k + 1) * count)
    ncclResult_t r = n.all_gather(buf + uint64_t(ctx->rank) * count_per_rank, buf, count_per_rank, ncclFloat64,
                                  static_cast<ncclComm_t>(ctx->nccl_comm), ctx->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    return VMB_OK;
}

int vmb_comm_allreduce_sum_f64(vmb_ctx* ctx, double* buf, uint64_t count) {
    if (!ctx->nccl_comm) return VMB_OK;
    Nccl& n = nccl();
    ncclResult_t r = n.all_reduce(buf, buf, count, ncclFloat64, ncclSum,
                                  static_cast<ncclComm_t>(ctx->nccl_comm), ctx->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    return VMB_OK;
}

}  // extern "C"
