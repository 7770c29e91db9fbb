// Context / matrix-handle types shared by engine.cu and comm.cu.
#pragma once

#include <atomic>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "sparse.cuh"

struct dsvd_ctx;

namespace dsvd {

extern std::atomic<int64_t> g_launches;

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
};

enum KernelClass { K_SPMM1 = 0, K_SPMM2, K_GRAM, K_EIG, K_RESCALE, K_COMM, K_OTHER, K_NCLASS };

struct TimedSpan {
    int cls;
    cudaEvent_t a, b;
};

// Multi-GPU hooks (comm.cu). With one rank they are no-ops (reduce-scatter /
// all-gather then copy when send != recv).
enum CommKind { COMM_NONE = 0, COMM_NCCL = 1, COMM_LOOPBACK = 2 };
constexpr int kMaxLoopbackRanks = 8;
// (stream: the stream the collective is ordered on, nullptr = ctx->stream)
void comm_allreduce_sum(dsvd_ctx* ctx, double* buf, size_t count, cudaStream_t stream = nullptr);
// Peer buffers for the fused exchange (mgpu_overlap 2): every rank's `mine`
// (device memory from cudaMalloc, the same size on every rank) as addresses
// this rank can store to — the loopback group's own pointers, or CUDA IPC
// mappings exchanged over NCCL. peers[rank] == mine. comm_close_peers unmaps.
void comm_exchange_peers(dsvd_ctx* ctx, void* mine, std::vector<void*>& peers);
void comm_close_peers(dsvd_ctx* ctx, std::vector<void*>& peers);
// Every rank's work on `stream` so far is complete (and its stores visible)
// before any rank's later work on its stream.
void comm_barrier(dsvd_ctx* ctx, cudaStream_t stream = nullptr);
// out[i] = slots[i] + slots[count + i] + ... (nslots slots, in slot order: the
// loopback reduction's rank order)
void comm_sum_slots(const double* slots, int nslots, size_t count, double* out, cudaStream_t stream);
// recv (count, significant on rank `root` only) = the sum of every rank's send
void comm_reduce_sum(dsvd_ctx* ctx, const double* send, double* recv, size_t count, int root,
                     cudaStream_t stream = nullptr);
// recv (recvcount) = rows [rank * recvcount, (rank + 1) * recvcount) of the sum of every rank's send
void comm_reduce_scatter_sum(dsvd_ctx* ctx, const double* send, double* recv, size_t recvcount);
// recv (nranks * sendcount) = every rank's send in rank order (send may be this rank's slot of recv)
void comm_allgather(dsvd_ctx* ctx, const double* send, double* recv, size_t sendcount);
// sum of a host scalar over the ranks (synchronous)
double comm_sum_host(dsvd_ctx* ctx, double v);
void comm_release(dsvd_ctx* ctx);
// thread-local last-error state of the C ABI (engine.cu)
void set_error(const char* msg, long long index);

}  // namespace dsvd

struct dsvd_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool profiling = false;
    dsvd_stats stats{};
    std::map<std::string, dsvd::DevBuf> arena;
    std::vector<cudaEvent_t> event_pool;
    size_t event_next = 0;
    std::vector<dsvd::TimedSpan> spans;
    int spmm_variant = 0;
    // column-slab SpMM (sparse.cu spmm_slab_kernel): -1 auto by width, 0 off,
    // 32 / 64 columns per slab; spmm_slab_hint: L2 evict_first on streaming bytes
    // (1: every launch, 2: only the A X pass that writes a slab-major Y — the A^T
    // pass is faster without it on C4)
    int spmm_slab = -1;
    int spmm_slab_hint = 2;
    // column-slab kernel: hot X rows (as many as fit in spmm_hot_mb MB of slab
    // rows) gathered with L2 evict_last, the rest evict_first; 0 MB = off (default:
    // measured slower on C4 since the kernel's other changes)
    int64_t spmm_hot_mb = 0;
    int uniform_values = 1;  // detect all-equal values (DevCsr::uniform)
    int spmm_slab_depth = 2;  // gather depth / occupancy variant (sparse.cu launch_slab_u): 2 in flight, 32 warps
    // with the column-slab kernel, keep the gathered blocks slab-major (the
    // sketch and A Q written so, the pass-1 operand converted once per pass)
    int slab_layout = 1;
    int omega_slab_w = 0;  // layout of a pregenerated Omega
    int64_t hub_threshold = 4096;   // rows with >= this many nonzeros take the hub SpMM path
    // rows longer than split_chunk nonzeros are computed as chunk partials summed
    // in a fixed order (deterministic; 0 = whole chains, bit-exact vs reference)
    int64_t split_chunk = 512;
    int64_t split_chunk_t = 0;        // transpose (pass 2) chunk length; 0: split_chunk
    // transpose chunks are also cut / ordered by X-row panels of this many rows (0: off)
    int64_t split_panel_rows = 32768;
    int dense_method = 0;           // 0: FP64 tensor-core Gram / rescale (dmma.cu), 1: DFMA kernels
    int eig_method = 0;             // 0: tridiagonal + inverse iteration (Jacobi fallback), 1: Jacobi
    cudaStream_t side = nullptr;    // second stream: hub-row SpMM runs beside the bulk kernel
    // eigSVD stream (highest priority): with pipeline = 1 the Gram + l x l eig of
    // T_{j-1} run here beside the A T_{j-1} pass on `stream` (solve_tall)
    cudaStream_t eig = nullptr;
    cudaEvent_t ev_t = nullptr, ev_eig = nullptr;
    int gram_async = 0;
    // pipelined loop: A^T pass unshifted before the eig wait, shift as its own
    // kernel after it (1), or fused into the A^T pass after the wait (0)
    int shift_after = 0;  // pipelined loop: Gram on the eig stream too (beside the A T pass)
    int pipeline = -1;  // -1: auto (pipelined at or below an nnz bound), 0: serial, 1: pipelined
    // pipelined loop, where eigSVD(T_j) runs: 2 the tridiagonalisation (one long
    // single-CTA kernel) on the eig stream beside the A T pass, the rest of the chain on the
    // main stream after it; 1 the whole chain beside the A T pass; 0 all of it after the
    // pass; -1 (default) 2 above l = 160, else 1
    int eig_overlap = -1;
    int64_t pipeline_auto_nnz = 0;  // override of the auto rule's nnz bound (0: cost model)
    // Omega generated on `side` while the host CSR uploads (host-input solves):
    // the next solve_tall with the same (m, l, seed) waits on omega_ev instead
    // of generating it
    bool omega_pending = false;
    int64_t omega_m = 0, omega_l = 0;
    uint64_t omega_seed = 0;
    cudaEvent_t omega_ev = nullptr;
    cudaStream_t copy = nullptr;      // host->device copy of the CSR values (upload_pair)
    // staged copies to / from PAGEABLE host buffers (engine.cu copy_h2d / copy_d2h):
    // a ring of pinned slots, the device streaming one slot while host threads move
    // another (option host_staging = 0: plain cudaMemcpyAsync through the driver's
    // bounce buffer)
    static constexpr int kStageSlots = 4;
    char* stage = nullptr;  // kStageSlots x stage_chunk bytes, pinned
    size_t stage_alloc_chunk = 0;
    cudaEvent_t stage_ev[kStageSlots] = {};
    cudaEvent_t stage_ready = nullptr;  // a staged device->host source is complete
    int64_t stage_chunk = int64_t(32) << 20;
    int host_staging = 1;
    int host_copy_threads = 0;  // 0: min(16, host cores)
    // touches the pages of pageable host outputs while the solve runs (engine.cu prefault_outputs)
    std::unique_ptr<std::thread> prefault;
    int64_t coo_rows = -1, coo_cols = -1, coo_nnz = -1;  // last assembled CSR (dsvd_coo_fetch, _from_coo)
    cudaEvent_t copy_ev = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    int32_t* host_flags = nullptr;  // pinned ring for stop flags
    cudaEvent_t timer[2] = {nullptr, nullptr};
    // multi-GPU state (comm.cu): an NCCL communicator, or an in-process loopback
    // group (testing); comm != nullptr marks a row-sharded solve
    void* comm = nullptr;
    int comm_kind = dsvd::COMM_NONE;
    dsvd_loopback* loopback = nullptr;
    int nranks = 1, rank = 0;
    // sharded solves: 1 = v1 (all-reduce of the n x l partials, dense work
    // redundant), 2 = v2 (reduce-scatter, slab Gram + l x l all-reduce, slab
    // rescale, all-gather); SURVEY 8e
    int mgpu_mode = 2;
    // sharded solves: the A^T pass runs in G row panels (the v2 slabs) and each
    // panel's partial is reduced on comm_stream while the next panel computes (1,
    // default), or the whole pass first and then one collective (0)
    int mgpu_overlap = 1;
    // mgpu_overlap 2 (v2): the A^T pass stores each row panel straight into its
    // owner's landing buffer (G source slots of n_slab rows), the owner sums them
    double* landing = nullptr;
    size_t landing_bytes = 0;
    // single-GPU shifted-family solves on the non-empty columns only (engine.cu
    // build_compact): 1 (default) when >= 2% of the columns are empty, 0 off
    int compact_cols = 1;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t comm_ev = nullptr;
    int64_t shard_row_offset = 0, shard_global_rows = -1;  // for the CSR entry points

    void* buf(const std::string& name, size_t bytes) {
        auto& b = arena[name];
        if (b.bytes < bytes) {
            if (b.ptr) DSVD_CUDA_CHECK(cudaFree(b.ptr));
            b.ptr = nullptr;
            b.bytes = 0;
            DSVD_CUDA_CHECK(cudaMalloc(&b.ptr, bytes > 0 ? bytes : 1));
            b.bytes = bytes;
        }
        return b.ptr;
    }
    void release(const std::string& name) {
        auto it = arena.find(name);
        if (it == arena.end()) return;
        if (it->second.ptr) DSVD_CUDA_CHECK(cudaFree(it->second.ptr));
        arena.erase(it);
    }
    template <class T>
    T* tbuf(const std::string& name, size_t count) {
        return static_cast<T*>(buf(name, sizeof(T) * (count > 0 ? count : 1)));
    }
    cudaEvent_t event() {
        if (event_next == event_pool.size()) {
            cudaEvent_t e;
            DSVD_CUDA_CHECK(cudaEventCreate(&e));
            event_pool.push_back(e);
        }
        return event_pool[event_next++];
    }
    // Profiling spans: a CUDA-event pair around a group of launches.
    int span_begin(int cls) {
        if (!profiling) return -1;
        dsvd::TimedSpan s{cls, event(), event()};
        DSVD_CUDA_CHECK(cudaEventRecord(s.a, stream));
        spans.push_back(s);
        return static_cast<int>(spans.size()) - 1;
    }
    void span_end(int id) {
        if (id < 0) return;
        DSVD_CUDA_CHECK(cudaEventRecord(spans[id].b, stream));
    }
};

namespace dsvd {
// The spmm() variant bits of a launch at row stride ld: the context's explicit
// spmm_variant, plus the column-slab kernel where it pays.
// big_rows: the row count of the solve's larger n-row / m-row block (0: unknown).
inline int spmm_var(const dsvd_ctx* ctx, int64_t ld, int64_t big_rows = 0);
// Slab width of the slab-major X / Y blocks of a solve at row stride ld (0: all
// row-major): the column-slab kernel's width when it runs in split mode and
// the context allows the layout (option "slab_layout").
inline int slab_layout_width(const dsvd_ctx* ctx, int64_t ld, int64_t big_rows = 0) {
    if (!ctx->slab_layout || ctx->split_chunk <= 0) return 0;
    const int v = spmm_var(ctx, ld, big_rows);
    if ((v & (16 | 32)) != 0) return 0;
    return (v & 4096) ? 32 : (v & 8192) ? 64 : 0;
}
// Doubles of the Y / sketch buffer (m rows): row-major m x ld or slab-major.
inline int64_t block_doubles(int64_t rows, int64_t ld, int lw) {
    return lw > 0 ? std::max(rows * ld, ceil_div(ld, lw) * lw * rows) : rows * ld;
}
inline int spmm_var(const dsvd_ctx* ctx, int64_t ld, int64_t big_rows) {
    int v = ctx->spmm_variant;
    if ((v & (4096 | 8192)) != 0) return v;  // explicit choice
    int w = ctx->spmm_slab;
    // auto: 64-column slabs above 192 columns (C4, l = 300: both passes 10-15%
    // faster than the whole-row kernel, tools/ab_option.py); below,
    // 32-column slabs when the gathered blocks are far beyond the L2 (> 1 GB: C5
    // 2.96 -> 2.74 s, C3 -1.5%), the whole-row kernel otherwise (C2: X and Y of
    // 122 / 243 MB stay mostly L2-resident, slabs +20%)
    if (w < 0) w = ld > 192 ? 64 : (big_rows * ld * 8 > (int64_t(1) << 30) ? 32 : 0);
    if (w == 32) v |= 4096;
    else if (w == 64) v |= 8192;
    if (w > 0 && ctx->spmm_slab_hint) v |= 16384;
    if (w > 0 && ctx->spmm_slab_hint == 2) v |= 131072;
    if (w > 0 && ctx->spmm_slab_depth == 1) v |= 32768;
    if (w > 0 && ctx->spmm_slab_depth == 2) v |= 65536;
    return v;
}
}  // namespace dsvd

struct dsvd_matrix {
    dsvd_ctx* ctx = nullptr;
    int device = 0;  // destroy() must not touch ctx: it may already be gone
    dsvd::DevCsr a, at;
    std::vector<void*> owned;
    // row shard of a larger matrix (multi-GPU): global row offset and count
    int64_t row_offset = 0;
    int64_t global_rows = -1;
};

