// Multi-GPU plumbing: one process per GPU, A row-sharded, Q replicated.
//
// The only data-path exchange of the power loop is the fp64 sum of the
// per-shard n x l partials A_g^T (A_g Q) (and once of A_g^T Omega_g), plus an
// l x l sum of the finalize Gram B_g^T B_g. It runs as an in-place NCCL
// all-reduce on the context's stream (NVLink 5 / NVSwitch on a B200 node;
// NVLS in-switch reduction when NCCL selects it). NCCL is loaded with dlopen
// on first use so single-GPU processes never load it, and so this library
// shares whatever libnccl.so.2 the host process (e.g. torch) already mapped.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "engine.cuh"

namespace dsvd {
namespace {

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.lib) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(DSVD_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) fail(DSVD_NCCL, std::string("libnccl is missing ") + n);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.lib = h;
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(DSVD_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void comm_allreduce_sum(dsvd_ctx* ctx, double* buf, size_t count) {
    if (ctx->comm == nullptr || count == 0) return;
    nccl_check(nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum,
                                static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclAllReduce");
}

void comm_release(dsvd_ctx* ctx) {
    if (ctx->comm != nullptr) {
        nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
        ctx->comm = nullptr;
    }
    ctx->nranks = 1;
    ctx->rank = 0;
}

}  // namespace dsvd

extern "C" {

int dsvd_comm_unique_id(uint8_t out[128]) {
    try {
        ncclUniqueId id;
        dsvd::nccl_check(dsvd::nccl().GetUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(out, &id, 128);
        return DSVD_OK;
    } catch (const dsvd::Failure& e) {
        dsvd::set_error(e.what(), -1);
        return e.code;
    }
}

int dsvd_ctx_attach_comm(dsvd_ctx* ctx, int nranks, int rank, const uint8_t id[128]) {
    try {
        if (nranks < 1 || rank < 0 || rank >= nranks) dsvd::fail(DSVD_CONFIG, "bad rank / world size");
        DSVD_CUDA_CHECK(cudaSetDevice(ctx->device));
        dsvd::comm_release(ctx);
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        ncclComm_t comm;
        dsvd::nccl_check(dsvd::nccl().CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
        ctx->comm = comm;
        ctx->nranks = nranks;
        ctx->rank = rank;
        return DSVD_OK;
    } catch (const dsvd::Failure& e) {
        dsvd::set_error(e.what(), -1);
        return e.code;
    }
}

}  // extern "C"
