// Multi-GPU plumbing: one process per GPU, A row-sharded, Q replicated.
//
// The data-path exchanges of the power loop (reference exchange
// point solver.cpp:93-95, where the single-process reference simply holds the
// whole A^T (A Q)):
//   v1  an fp64 sum of the per-shard n x l partials A_g^T (A_g Q) — one
//       all-reduce per iteration — then the dense work redundantly per GPU;
//   v2  a reduce-scatter of the same partials (each rank gets an n/G-row slab
//       of the sum), an l x l all-reduce of the slab Grams, and an all-gather
//       of the rescaled slabs (same bytes on the wire, 1/G of the dense work).
// Plus the l x l sum of the finalize Gram B_g^T B_g.
//
// Two transports behind one interface:
//   NCCL      (production) on the context's stream — NVLink 5 / NVSwitch on a
//             B200 node, NVLS in-switch reduction when NCCL selects it. NCCL is
//             loaded with dlopen on first use, so single-GPU processes never load
//             it and this library shares whatever libnccl.so.2 the host process
//             (e.g. torch) already mapped. Asynchronous NCCL errors are polled
//             after every collective (ncclCommGetAsyncError) and raised as
//             DSVD_NCCL.
//   loopback  (testing) G contexts of ONE process on host threads, typically
//             on one GPU: each collective synchronises the rank's stream, meets
//             the other ranks at a host barrier, and sums their device buffers in
//             fixed rank order (so every rank holds bitwise the same result).
//             No kernel waits on another rank's kernel — the ranks only meet on
//             the host — so the sharded engine runs natively at G > 1 on a
//             single device (tests/test_gpu_sharded.py).
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "engine.cuh"

struct dsvd_loopback {
    int nranks = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool aborted = false;
    std::vector<const double*> posted;  // per-rank device pointer of the current collective
    std::vector<int> attached;
};

namespace dsvd {
namespace {

constexpr int kLoopbackTimeoutS = 600;

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
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
    api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
    api.Reduce = reinterpret_cast<decltype(api.Reduce)>(sym("ncclReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.lib = h;
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(DSVD_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// Asynchronous communicator errors (a peer died, a network/NVLink fault): NCCL
// reports them only through this query, so it is polled after every call.
void nccl_poll(dsvd_ctx* ctx, const char* what) {
    ncclResult_t async = ncclSuccess;
    nccl_check(nccl().CommGetAsyncError(static_cast<ncclComm_t>(ctx->comm), &async), "ncclCommGetAsyncError");
    if (async != ncclSuccess && async != ncclInProgress)
        fail(DSVD_NCCL, std::string(what) + ": asynchronous NCCL error: " + nccl().GetErrorString(async));
}

// ---- loopback transport ------------------------------------------------------

struct RankPtrs {
    const double* p[kMaxLoopbackRanks];
};

// out[i] = src[0][off + i] + src[1][off + i] + ... in rank order.
__global__ void rank_sum_kernel(RankPtrs src, int nranks, size_t off, double* __restrict__ out, size_t count) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double acc = src.p[0][off + i];
        for (int r = 1; r < nranks; ++r) acc += src.p[r][off + i];
        out[i] = acc;
    }
}

void lb_barrier(dsvd_loopback* g) {
    std::unique_lock<std::mutex> lock(g->mu);
    if (g->aborted) fail(DSVD_NCCL, "loopback group aborted by another rank");
    const uint64_t gen = g->generation;
    if (++g->arrived == g->nranks) {
        g->arrived = 0;
        ++g->generation;
        g->cv.notify_all();
        return;
    }
    if (!g->cv.wait_for(lock, std::chrono::seconds(kLoopbackTimeoutS),
                        [&] { return g->generation != gen || g->aborted; })) {
        g->aborted = true;
        g->cv.notify_all();
        fail(DSVD_NCCL, "loopback barrier timed out (a rank did not reach the collective)");
    }
    if (g->aborted) fail(DSVD_NCCL, "loopback group aborted by another rank");
}

// Post this rank's buffer, wait until every rank posted, return the pointers.
RankPtrs lb_post(dsvd_ctx* ctx, const double* mine, cudaStream_t stream = nullptr) {
    dsvd_loopback* g = ctx->loopback;
    DSVD_CUDA_CHECK(cudaStreamSynchronize(stream ? stream : ctx->stream));  // the partial is complete
    {
        std::lock_guard<std::mutex> lock(g->mu);
        g->posted[ctx->rank] = mine;
    }
    lb_barrier(g);
    RankPtrs r{};
    std::lock_guard<std::mutex> lock(g->mu);
    for (int i = 0; i < g->nranks; ++i) r.p[i] = g->posted[i];
    return r;
}

int sum_grid(size_t count) {
    const size_t b = (count + 255) / 256;
    return static_cast<int>(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}

void lb_allreduce(dsvd_ctx* ctx, double* buf, size_t count, cudaStream_t s) {
    const RankPtrs src = lb_post(ctx, buf, s);
    double* tmp = ctx->tbuf<double>("comm.lb.tmp", count);
    rank_sum_kernel<<<sum_grid(count), 256, 0, s>>>(src, ctx->nranks, 0, tmp, count);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cudaStreamSynchronize(s));
    lb_barrier(ctx->loopback);  // every rank has read every buffer
    DSVD_CUDA_CHECK(cudaMemcpyAsync(buf, tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(s));
}

void lb_reduce(dsvd_ctx* ctx, const double* send, double* recv, size_t count, int root, cudaStream_t s) {
    const RankPtrs src = lb_post(ctx, send, s);
    if (ctx->rank == root) {
        rank_sum_kernel<<<sum_grid(count), 256, 0, s>>>(src, ctx->nranks, 0, recv, count);
        DSVD_LAUNCH_CHECK();
        DSVD_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    lb_barrier(ctx->loopback);  // the root has read every send
}

void lb_reduce_scatter(dsvd_ctx* ctx, const double* send, double* recv, size_t recvcount) {
    const RankPtrs src = lb_post(ctx, send);
    rank_sum_kernel<<<sum_grid(recvcount), 256, 0, ctx->stream>>>(src, ctx->nranks, ctx->rank * recvcount, recv,
                                                                  recvcount);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    lb_barrier(ctx->loopback);  // nobody reads `send` any more
}

void lb_allgather(dsvd_ctx* ctx, const double* send, double* recv, size_t sendcount) {
    const RankPtrs src = lb_post(ctx, send);
    for (int r = 0; r < ctx->nranks; ++r) {
        double* dst = recv + r * sendcount;
        if (dst == src.p[r]) continue;  // in place (send is this rank's slot of recv)
        DSVD_CUDA_CHECK(cudaMemcpyAsync(dst, src.p[r], sizeof(double) * sendcount, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
    }
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    lb_barrier(ctx->loopback);
}

}  // namespace

void comm_allreduce_sum(dsvd_ctx* ctx, double* buf, size_t count, cudaStream_t stream) {
    if (ctx->comm_kind == COMM_NONE || count == 0) return;
    NvtxRange r("dsvd.allreduce");
    const cudaStream_t s = stream ? stream : ctx->stream;
    if (ctx->comm_kind == COMM_LOOPBACK) return lb_allreduce(ctx, buf, count, s);
    nccl_check(nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(ctx->comm), s),
               "ncclAllReduce");
    nccl_poll(ctx, "ncclAllReduce");
}

void comm_reduce_sum(dsvd_ctx* ctx, const double* send, double* recv, size_t count, int root, cudaStream_t stream) {
    const cudaStream_t s = stream ? stream : ctx->stream;
    if (ctx->comm_kind == COMM_NONE) {
        if (send != recv && count)
            DSVD_CUDA_CHECK(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (count == 0) return;
    NvtxRange r("dsvd.reduce");
    if (ctx->comm_kind == COMM_LOOPBACK) return lb_reduce(ctx, send, recv, count, root, s);
    nccl_check(nccl().Reduce(send, recv, count, ncclDouble, ncclSum, root, static_cast<ncclComm_t>(ctx->comm), s),
               "ncclReduce");
    nccl_poll(ctx, "ncclReduce");
}

void comm_reduce_scatter_sum(dsvd_ctx* ctx, const double* send, double* recv, size_t recvcount) {
    if (ctx->comm_kind == COMM_NONE) {
        if (send != recv)
            DSVD_CUDA_CHECK(cudaMemcpyAsync(recv, send, sizeof(double) * recvcount, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
        return;
    }
    NvtxRange r("dsvd.reduce_scatter");
    if (ctx->comm_kind == COMM_LOOPBACK) return lb_reduce_scatter(ctx, send, recv, recvcount);
    nccl_check(nccl().ReduceScatter(send, recv, recvcount, ncclDouble, ncclSum, static_cast<ncclComm_t>(ctx->comm),
                                    ctx->stream),
               "ncclReduceScatter");
    nccl_poll(ctx, "ncclReduceScatter");
}

void comm_allgather(dsvd_ctx* ctx, const double* send, double* recv, size_t sendcount) {
    if (ctx->comm_kind == COMM_NONE) {
        if (send != recv)
            DSVD_CUDA_CHECK(cudaMemcpyAsync(recv, send, sizeof(double) * sendcount, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
        return;
    }
    NvtxRange r("dsvd.allgather");
    if (ctx->comm_kind == COMM_LOOPBACK) return lb_allgather(ctx, send, recv, sendcount);
    nccl_check(nccl().AllGather(send, recv, sendcount, ncclDouble, static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclAllGather");
    nccl_poll(ctx, "ncclAllGather");
}

void comm_sum_slots(const double* slots, int nslots, size_t count, double* out, cudaStream_t stream) {
    RankPtrs src{};
    for (int g = 0; g < nslots; ++g) src.p[g] = slots + g * count;
    rank_sum_kernel<<<sum_grid(count), 256, 0, stream>>>(src, nslots, 0, out, count);
    DSVD_LAUNCH_CHECK();
}

void comm_barrier(dsvd_ctx* ctx, cudaStream_t stream) {
    if (ctx->comm_kind == COMM_NONE) return;
    const cudaStream_t s = stream ? stream : ctx->stream;
    NvtxRange r("dsvd.barrier");
    if (ctx->comm_kind == COMM_LOOPBACK) {
        DSVD_CUDA_CHECK(cudaStreamSynchronize(s));
        lb_barrier(ctx->loopback);
        return;
    }
    // a one-element all-reduce on the stream: no rank gets past it before every
    // rank's earlier work on its stream (incl. its peer stores) has completed
    double* d = ctx->tbuf<double>("comm.barrier", 1);
    nccl_check(nccl().AllReduce(d, d, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(ctx->comm), s),
               "ncclAllReduce (barrier)");
    nccl_poll(ctx, "barrier");
}

void comm_exchange_peers(dsvd_ctx* ctx, void* mine, std::vector<void*>& peers) {
    peers.assign(ctx->nranks, nullptr);
    peers[ctx->rank] = mine;
    if (ctx->comm_kind == COMM_NONE) return;
    if (ctx->comm_kind == COMM_LOOPBACK) {  // one process, one address space
        const RankPtrs src = lb_post(ctx, static_cast<const double*>(mine));
        for (int g = 0; g < ctx->nranks; ++g) peers[g] = const_cast<double*>(src.p[g]);
        lb_barrier(ctx->loopback);  // every rank has read the posted pointers
        return;
    }
    // NCCL: CUDA IPC handles of every rank's buffer, all-gathered, opened here
    cudaIpcMemHandle_t h;
    DSVD_CUDA_CHECK(cudaIpcGetMemHandle(&h, mine));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    char* d = ctx->tbuf<char>("comm.ipc", 64 * static_cast<size_t>(ctx->nranks + 1));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(d + 64 * ctx->nranks, &h, 64, cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(nccl().AllGather(d + 64 * ctx->nranks, d, 64, ncclChar, static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclAllGather (IPC handles)");
    std::vector<cudaIpcMemHandle_t> all(ctx->nranks);
    DSVD_CUDA_CHECK(cudaMemcpyAsync(all.data(), d, 64 * static_cast<size_t>(ctx->nranks), cudaMemcpyDeviceToHost,
                                    ctx->stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    nccl_poll(ctx, "IPC handle exchange");
    for (int g = 0; g < ctx->nranks; ++g) {
        if (g == ctx->rank) continue;
        DSVD_CUDA_CHECK(cudaIpcOpenMemHandle(&peers[g], all[g], cudaIpcMemLazyEnablePeerAccess));
    }
}

void comm_close_peers(dsvd_ctx* ctx, std::vector<void*>& peers) {
    if (ctx->comm_kind == COMM_NCCL)
        for (int g = 0; g < static_cast<int>(peers.size()); ++g)
            if (g != ctx->rank && peers[g] != nullptr) cudaIpcCloseMemHandle(peers[g]);
    peers.clear();
}

double comm_sum_host(dsvd_ctx* ctx, double v) {
    if (ctx->comm_kind == COMM_NONE) return v;
    double* d = ctx->tbuf<double>("comm.scalar", 1);
    DSVD_CUDA_CHECK(cudaMemcpyAsync(d, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    comm_allreduce_sum(ctx, d, 1);
    double out = 0.0;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&out, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (ctx->comm_kind == COMM_NCCL) nccl_poll(ctx, "scalar all-reduce");
    return out;
}

void comm_release(dsvd_ctx* ctx) {
    if (ctx->comm_kind == COMM_NCCL && ctx->comm != nullptr) nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    if (ctx->comm_kind == COMM_LOOPBACK && ctx->loopback != nullptr) {
        std::lock_guard<std::mutex> lock(ctx->loopback->mu);
        ctx->loopback->attached[ctx->rank] = 0;
    }
    ctx->comm = nullptr;
    ctx->loopback = nullptr;
    ctx->comm_kind = COMM_NONE;
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
        ctx->comm_kind = dsvd::COMM_NCCL;
        ctx->nranks = nranks;
        ctx->rank = rank;
        return DSVD_OK;
    } catch (const dsvd::Failure& e) {
        dsvd::set_error(e.what(), -1);
        return e.code;
    }
}

int dsvd_loopback_create(int nranks, dsvd_loopback** out) {
    try {
        if (nranks < 1 || nranks > dsvd::kMaxLoopbackRanks)
            dsvd::fail(DSVD_CONFIG, "loopback group: 1 <= nranks <= " + std::to_string(dsvd::kMaxLoopbackRanks));
        dsvd_loopback* g = new dsvd_loopback();
        g->nranks = nranks;
        g->posted.assign(nranks, nullptr);
        g->attached.assign(nranks, 0);
        *out = g;
        return DSVD_OK;
    } catch (const dsvd::Failure& e) {
        dsvd::set_error(e.what(), -1);
        return e.code;
    }
}

int dsvd_loopback_destroy(dsvd_loopback* g) {
    if (g == nullptr) return DSVD_OK;
    {
        std::lock_guard<std::mutex> lock(g->mu);
        for (int a : g->attached)
            if (a) {
                dsvd::set_error("loopback group still has attached contexts", -1);
                return DSVD_CONFIG;
            }
    }
    delete g;
    return DSVD_OK;
}

int dsvd_ctx_attach_loopback(dsvd_ctx* ctx, dsvd_loopback* g, int rank) {
    try {
        if (g == nullptr || rank < 0 || rank >= g->nranks) dsvd::fail(DSVD_CONFIG, "bad loopback rank");
        DSVD_CUDA_CHECK(cudaSetDevice(ctx->device));
        dsvd::comm_release(ctx);
        {
            std::lock_guard<std::mutex> lock(g->mu);
            if (g->attached[rank]) dsvd::fail(DSVD_CONFIG, "loopback rank already attached");
            g->attached[rank] = 1;
        }
        ctx->loopback = g;
        ctx->comm = g;
        ctx->comm_kind = dsvd::COMM_LOOPBACK;
        ctx->nranks = g->nranks;
        ctx->rank = rank;
        return DSVD_OK;
    } catch (const dsvd::Failure& e) {
        dsvd::set_error(e.what(), -1);
        return e.code;
    }
}

}  // extern "C"
