// Engine + C ABI of the B200 dashSVD hot path.
//
// The solve mirrors run_shifted_iterations + finalize_row_basis
// (solver.cpp:76-116, :159-164) with every step on the device:
//
//   Omega (m x l, seeded)            gaussian_rowmajor
//   T = A^T Omega                    spmm (CSR of A^T)
//   Q = eigSVD(T).u                  gram -> jacobi -> finish -> rescale
//   loop j = 1..p (or until the PVE rule fires):
//     Y = A Q                        spmm pass 1
//     T = A^T Y - alpha Q            spmm pass 2, shift fused in the epilogue
//     (s, V) = eigSVD(T)             gram -> jacobi -> finish (+ trace, stop rule, shift)
//     Q = T V diag(1/s)              rescale
//   B = A Q; U, s, V' = eigSVD(B); V = Q V'[:, :k]
//
// Loop control never waits on the host in fixed-p mode; in accuracy-control
// mode the host reads a 4-byte stop flag with a lookahead of two iterations
// (iterations enqueued past the stop are skipped on the device through
// Control::stopped), so the GPU never idles on the check.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "engine.cuh"
#include "engine_internal.cuh"
#include "qr.cuh"

#include "eig.cuh"
#include "rng.cuh"
#include "sparse.cuh"

namespace dsvd {

std::atomic<int64_t> g_launches{0};

}  // namespace dsvd

namespace dsvd {
namespace {

thread_local std::string t_err;
thread_local long long t_err_index = -1;

constexpr int kMaxSweeps = 60;
constexpr int kLookahead = 2;

}  // namespace

void set_error(const char* msg, long long index) {
    t_err = msg;
    t_err_index = index;
}

void set_device(dsvd_ctx* ctx) { DSVD_CUDA_CHECK(cudaSetDevice(ctx->device)); }

void count_launch(int n) { g_launches += n; }

// ---- host <-> device copies that may touch pageable memory ----------------
// The reference-shaped API hands back std::vector / numpy factors, i.e.
// pageable memory, and its inputs usually live there too. A cudaMemcpyAsync
// to or from pageable memory runs through the driver's bounce buffer at a
// fraction of the PCIe rate (C4's 13.4 GB of U and V: ~2.9 s against ~0.25 s
// pinned). Pageable copies therefore go through a ring of pinned slots: the
// copy stream moves slot c over PCIe while host threads move slot c - 1 to or
// from the caller's buffer (host_parallel_memcpy, which also takes the
// buffer's first-touch page faults in parallel). Pinned, registered and
// device pointers keep the plain cudaMemcpyAsync.
void host_parallel_memcpy(void* dst, const void* src, size_t bytes, int threads);
void host_prefault(void* p, size_t bytes, int threads);

bool host_is_pageable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

namespace {

bool use_staging(dsvd_ctx* ctx, const void* host, size_t bytes) {
    return ctx->host_staging && bytes >= (size_t(1) << 20) && host_is_pageable(host);
}

int copy_threads(dsvd_ctx* ctx) {
    if (ctx->host_copy_threads > 0) return ctx->host_copy_threads;
    const int cores = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, std::min(16, cores));
}

// the staging ring, every slot idle (no copy in flight reads or writes it)
char* stage_ring(dsvd_ctx* ctx) {
    const size_t chunk = static_cast<size_t>(ctx->stage_chunk);
    for (cudaEvent_t& e : ctx->stage_ev) {
        if (!e) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventSynchronize(e));
    }
    if (ctx->stage && ctx->stage_alloc_chunk != chunk) {
        DSVD_CUDA_CHECK(cudaFreeHost(ctx->stage));
        ctx->stage = nullptr;
    }
    if (!ctx->stage) {
        DSVD_CUDA_CHECK(cudaHostAlloc(&ctx->stage, chunk * dsvd_ctx::kStageSlots, cudaHostAllocPortable));
        ctx->stage_alloc_chunk = chunk;
    }
    return ctx->stage;
}

}  // namespace

void prefault_join(dsvd_ctx* ctx) noexcept {
    if (ctx->prefault) {
        if (ctx->prefault->joinable()) ctx->prefault->join();
        ctx->prefault.reset();
    }
}

// A solve's pageable host outputs (u: rows x k, v: cols x k) are faulted in on
// a host thread while the device computes; the staged copies join it first.
void prefault_outputs(dsvd_ctx* ctx, const dsvd_outputs* out, int64_t rows, int64_t cols, int64_t k) {
    prefault_join(ctx);
    if (!ctx->host_staging || out->outputs_on_device) return;
    std::vector<std::pair<void*, size_t>> r;
    const size_t ub = sizeof(double) * rows * k, vb = sizeof(double) * cols * k;
    if (out->u && use_staging(ctx, out->u, ub)) r.emplace_back(out->u, ub);
    if (out->v && use_staging(ctx, out->v, vb)) r.emplace_back(out->v, vb);
    if (r.empty()) return;
    ctx->prefault = std::make_unique<std::thread>([r] {
        for (const auto& x : r) host_prefault(x.first, x.second, 4);
    });
}

// device -> host. The source is complete once `producer`'s work enqueued so
// far has run (or, when given, once `ready` has fired). Returns with the bytes in `dst` (host-blocking, like a
// cudaMemcpyAsync into pageable memory).
void copy_d2h(dsvd_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t producer,
              cudaEvent_t ready) {
    if (!use_staging(ctx, dst, bytes)) {
        if (ready) DSVD_CUDA_CHECK(cudaStreamWaitEvent(producer, ready, 0));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, producer));
        return;
    }
    prefault_join(ctx);  // the destination's pages are in
    char* ring = stage_ring(ctx);
    if (!ctx->copy) DSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    if (!ready) {
        if (!ctx->copy_ev) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->copy_ev, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->copy_ev, producer));
        ready = ctx->copy_ev;
    }
    DSVD_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy, ready, 0));
    const size_t chunk = static_cast<size_t>(ctx->stage_chunk);
    const size_t nch = (bytes + chunk - 1) / chunk;
    const int ns = dsvd_ctx::kStageSlots, threads = copy_threads(ctx);
    auto issue = [&](size_t c) {
        const size_t n = std::min(chunk, bytes - c * chunk);
        char* slot = ring + (c % ns) * chunk;
        DSVD_CUDA_CHECK(cudaMemcpyAsync(slot, static_cast<const char*>(src) + c * chunk, n,
                                        cudaMemcpyDeviceToHost, ctx->copy));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->stage_ev[c % ns], ctx->copy));
    };
    for (size_t c = 0; c < std::min<size_t>(ns, nch); ++c) issue(c);
    for (size_t c = 0; c < nch; ++c) {
        DSVD_CUDA_CHECK(cudaEventSynchronize(ctx->stage_ev[c % ns]));
        const size_t n = std::min(chunk, bytes - c * chunk);
        host_parallel_memcpy(static_cast<char*>(dst) + c * chunk, ring + (c % ns) * chunk, n, threads);
        if (c + ns < nch) issue(c + ns);
    }
}

// host -> device, ordered on `st` (later work on `st` sees the bytes). Returns
// once the source has been read (host-blocking for pageable sources).
void copy_h2d(dsvd_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!use_staging(ctx, src, bytes)) {
        DSVD_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    char* ring = stage_ring(ctx);
    const size_t chunk = static_cast<size_t>(ctx->stage_chunk);
    const size_t nch = (bytes + chunk - 1) / chunk;
    const int ns = dsvd_ctx::kStageSlots, threads = copy_threads(ctx);
    for (size_t c = 0; c < nch; ++c) {
        const size_t n = std::min(chunk, bytes - c * chunk);
        char* slot = ring + (c % ns) * chunk;
        DSVD_CUDA_CHECK(cudaEventSynchronize(ctx->stage_ev[c % ns]));  // the slot's last upload is done
        host_parallel_memcpy(slot, static_cast<const char*>(src) + c * chunk, n, threads);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + c * chunk, slot, n, cudaMemcpyHostToDevice, st));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->stage_ev[c % ns], st));
    }
}

namespace {

// ---- matrix construction --------------------------------------------------


// Chunk list of the rows longer than m.split_chunk (the prefix m.hub_rows of
// m.order), planned on the device (sparse.cu chunk_plan_*): each split row is
// cut into near-equal CSR ranges of at most split_chunk nonzeros. With
// npanel > 1 (rows with sorted indices only, i.e. the transpose) the ranges are
// also cut where the gathered X row index crosses a multiple of panel_rows,
// and the chunk list is ordered by panel: chunks that run together then gather
// from one panel_rows-row slice of X (~40 MB at ld 152, L2-resident) instead of
// all of it. Each row's chunks are still summed in CSR order (chunk_slot maps
// them to list positions).
struct ChunkPlan {
    int npanel = 1;
    int64_t panel_rows = 0;
    int32_t* row_nch = nullptr;
    int32_t* first = nullptr;
    int32_t* total_max = nullptr;  // device {total, max}
};

void plan_chunks_count(dsvd_ctx* ctx, CsrAlloc& al, DevCsr& m, const std::string& tag, int64_t panel_rows,
                       int32_t* total_max, ChunkPlan& cp) {
    cp.npanel = panel_rows > 0 ? static_cast<int>(std::max<int64_t>(1, ceil_div(m.cols, panel_rows))) : 1;
    cp.panel_rows = cp.npanel > 1 ? panel_rows : 0;
    cp.row_nch = ctx->tbuf<int32_t>("chunk.row_nch." + tag, m.rows);
    cp.first = static_cast<int32_t*>(al.get(tag + ".split_first", sizeof(int32_t) * (m.rows + 1)));
    cp.total_max = total_max;
    const size_t tb = chunk_plan_scratch_bytes(m.rows, 1);
    chunk_plan_count(m, cp.npanel, cp.panel_rows, cp.row_nch, cp.first, total_max, ctx->buf("chunk.temp", tb), tb,
                     ctx->stream);
    count_launch(3);
}

void plan_chunks_emit(dsvd_ctx* ctx, CsrAlloc& al, DevCsr& m, const std::string& tag, const ChunkPlan& cp,
                      int64_t nc, int64_t max_row) {
    const int64_t ns = m.hub_rows;
    m.nsplit = 0;
    m.nchunks = 0;
    m.hub_rows = 0;  // split mode does not use the hub kernels
    m.chunk_slot = nullptr;
    m.max_row_chunks = max_row;
    if (ns == 0 || nc == 0) return;
    m.chunk_p0 = static_cast<int64_t*>(al.get(tag + ".chunk_p0", sizeof(int64_t) * nc));
    m.chunk_p1 = static_cast<int64_t*>(al.get(tag + ".chunk_p1", sizeof(int64_t) * nc));
    m.split_first = cp.first;
    if (cp.npanel > 1) m.chunk_slot = static_cast<int32_t*>(al.get(tag + ".chunk_slot", sizeof(int32_t) * nc));
    const size_t tb = chunk_plan_scratch_bytes(m.rows, nc);
    chunk_plan_emit(m, ns, cp.npanel, cp.panel_rows, cp.first, nc, m.chunk_p0, m.chunk_p1, m.chunk_slot,
                    ctx->tbuf<int64_t>("chunk.tmp0", nc), ctx->tbuf<int64_t>("chunk.tmp1", nc),
                    ctx->tbuf<int32_t>("chunk.keys", nc), ctx->tbuf<int32_t>("chunk.keys_s", nc),
                    ctx->tbuf<int32_t>("chunk.ids", nc), ctx->tbuf<int32_t>("chunk.ids_s", nc),
                    ctx->buf("chunk.temp", tb), tb, ctx->stream);
    count_launch(cp.npanel > 1 ? 4 : 1);
    m.nsplit = ns;
    m.nchunks = nc;
}

// Partial-row workspace for the split chunks of `a` at width ld.
}  // namespace

// Device CSR (+ transpose + row orders) from int64 offsets / indices and
// values already on the device.
void build_pair(dsvd_ctx* ctx, CsrAlloc& al, int64_t rows, int64_t cols, int64_t nnz,
                const int64_t* d_off, const int64_t* d_idx64, const double* d_val, DevCsr& a,
                DevCsr& at, bool copy_inputs, cudaEvent_t values_ready) {
    NvtxRange nvtx("dsvd.csc_build");
    cudaStream_t st = ctx->stream;
    if (rows < 0 || cols < 0 || nnz < 0) fail(DSVD_SHAPE, "sparse matrix with negative dimension");
    if (rows > 0x7fffffffLL || cols > 0x7fffffffLL)
        fail(DSVD_UNSUPPORTED, "dimensions >= 2^31 are not supported on the device path");
    if (nnz > 0x7fffffffLL)  // int32 nonzero positions in the CSC build (row-shard larger matrices)
        fail(DSVD_UNSUPPORTED, "nnz >= 2^31 per device is not supported; shard the rows over GPUs");
    a.rows = rows;
    a.cols = cols;
    a.nnz = nnz;
    if (copy_inputs) {
        a.off = static_cast<int64_t*>(al.get("a.off", sizeof(int64_t) * (rows + 1)));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(a.off, d_off, sizeof(int64_t) * (rows + 1),
                                        cudaMemcpyDeviceToDevice, st));
        a.val = static_cast<double*>(al.get("a.val", sizeof(double) * nnz));
        if (nnz)
            DSVD_CUDA_CHECK(cudaMemcpyAsync(a.val, d_val, sizeof(double) * nnz,
                                            cudaMemcpyDeviceToDevice, st));
    } else {
        a.off = const_cast<int64_t*>(d_off);
        a.val = const_cast<double*>(d_val);
    }
    a.idx = static_cast<int32_t*>(al.get("a.idx", sizeof(int32_t) * nnz));
    a.order = static_cast<int32_t*>(al.get("a.order", sizeof(int32_t) * (rows > 0 ? rows : 1)));
    a.obeg = static_cast<int64_t*>(al.get("a.obeg", sizeof(int64_t) * (rows > 0 ? rows : 1)));
    a.olen = static_cast<int32_t*>(al.get("a.olen", sizeof(int32_t) * (rows > 0 ? rows : 1)));
    // device scalars read back by the host: {offsets bad, index bad} right away,
    // {hub rows of A, of A^T, chunk total / max of A, of A^T} in one read at the end
    // (+ [12] values not uniform, [14..15] the first value's bits)
    int32_t* sc = static_cast<int32_t*>(al.get("plan_scalars", sizeof(int32_t) * 18));
    DSVD_CUDA_CHECK(cudaMemsetAsync(sc, 0, sizeof(int32_t) * 18, st));
    check_offsets(a.off, rows, nnz, sc, st);
    count_launch();
    narrow_indices(d_idx64, a.idx, nnz, cols, sc + 1, st);
    count_launch(nnz > 0);
    {  // malformed offsets would send the transpose out of bounds: check before it runs
        int32_t hb[2];
        DSVD_CUDA_CHECK(cudaMemcpyAsync(hb, sc, sizeof(hb), cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
        if (hb[0]) fail(DSVD_SHAPE, "offsets must be non-decreasing and span [0, nnz]");
        if (hb[1]) fail(DSVD_SHAPE, "column index out of range");
    }

    at.rows = cols;
    at.cols = rows;
    at.nnz = nnz;
    at.off = static_cast<int64_t*>(al.get("at.off", sizeof(int64_t) * (cols + 1)));
    at.idx = static_cast<int32_t*>(al.get("at.idx", sizeof(int32_t) * nnz));
    at.val = static_cast<double*>(al.get("at.val", sizeof(double) * nnz));
    at.order = static_cast<int32_t*>(al.get("at.order", sizeof(int32_t) * (cols > 0 ? cols : 1)));
    at.obeg = static_cast<int64_t*>(al.get("at.obeg", sizeof(int64_t) * (cols > 0 ? cols : 1)));
    at.olen = static_cast<int32_t*>(al.get("at.olen", sizeof(int32_t) * (cols > 0 ? cols : 1)));
    const size_t scratch_bytes =
        std::max({csc_scratch_bytes(rows, cols, nnz), order_scratch_bytes(rows), order_scratch_bytes(cols)});
    void* scratch = ctx->buf("csc.scratch", scratch_bytes);
    build_transpose(a, at, scratch, scratch_bytes, st, values_ready);
    count_launch(nnz > 0 ? 8 : 1);  // 4 own kernels + CUB radix sort passes (estimate)
    // split mode: the "hub" prefix of the row order is the set of rows longer
    // than split_chunk, which are cut into chunks below
    if (ctx->uniform_values) {  // a.val is complete on st once the transpose has gathered it
        check_uniform_values(a.val, nnz, sc + 12, reinterpret_cast<double*>(sc + 14), st);
        count_launch(nnz > 0);
    }
    const int64_t C = ctx->split_chunk;
    // the transpose (pass 2) may split shorter rows than A (split_chunk_t)
    const int64_t Ct = C > 0 && ctx->split_chunk_t > 0 ? ctx->split_chunk_t : C;
    a.hub_threshold = C > 0 ? C + 1 : ctx->hub_threshold;
    at.hub_threshold = Ct > 0 ? Ct + 1 : ctx->hub_threshold;
    a.split_chunk = C;
    at.split_chunk = Ct;
    a.d_hub_rows = sc + 2;
    at.d_hub_rows = sc + 3;
    a.d_nonempty = sc + 8;
    at.d_nonempty = sc + 9;
    a.d_long = sc + 10;
    at.d_long = sc + 11;
    a.d_mid = sc + 16;
    at.d_mid = sc + 17;
    build_row_order(a, scratch, scratch_bytes, st);
    count_launch(rows > 0 ? 4 : 0);
    build_row_order(at, scratch, scratch_bytes, st);
    count_launch(cols > 0 ? 4 : 0);
    ChunkPlan cpa, cpt;
    if (C > 0) {
        // no panels for A: pass 1 gathers (Zipf columns) are L2-friendly already
        // and the caller's rows need not be sorted
        plan_chunks_count(ctx, al, a, "a", 0, sc + 4, cpa);
        plan_chunks_count(ctx, al, at, "at", ctx->split_panel_rows, sc + 6, cpt);
    }
    int32_t h[18];
    DSVD_CUDA_CHECK(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    a.uniform = at.uniform = ctx->uniform_values && nnz > 0 && h[12] == 0;
    std::memcpy(&a.uval, h + 14, sizeof(double));
    at.uval = a.uval;
    a.nonempty_rows = rows > 0 ? h[8] : 0;
    at.nonempty_rows = cols > 0 ? h[9] : 0;
    a.long_rows = rows > 0 ? h[10] : 0;
    at.long_rows = cols > 0 ? h[11] : 0;
    a.mid_rows = rows > 0 ? h[16] : 0;
    at.mid_rows = cols > 0 ? h[17] : 0;
    a.hub_rows = rows > 0 ? h[2] : 0;
    at.hub_rows = cols > 0 ? h[3] : 0;
    if (C > 0) {
        plan_chunks_emit(ctx, al, a, "a", cpa, h[4], h[5]);
        plan_chunks_emit(ctx, al, at, "at", cpt, h[6], h[7]);
    }
}

// Row panels [bounds[p], bounds[p+1]) of a device CSR as DevCsr views for the
// exchange overlap of row-sharded solves (solve_tall, mgpu_overlap): the
// views share the offsets / indices / values (a view's off points at its first
// row, positions stay absolute) and get their own length order, row ranges and
// split-row chunk plan. A split row is cut exactly as in the whole matrix
// (same split_chunk and X-row panels) and its chunks are combined in CSR order,
// so a panel's rows come out bitwise as in the whole-matrix pass.
std::vector<DevCsr> build_row_panels(dsvd_ctx* ctx, const DevCsr& m, const std::vector<int64_t>& bounds) {
    cudaStream_t st = ctx->stream;
    const int np = static_cast<int>(bounds.size()) - 1;
    std::vector<int64_t> hoff(bounds.size());
    for (size_t i = 0; i < bounds.size(); ++i)
        DSVD_CUDA_CHECK(cudaMemcpyAsync(&hoff[i], m.off + bounds[i], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    CsrAlloc al{ctx, "panel.", nullptr};
    int32_t* sc = static_cast<int32_t*>(al.get("scalars", sizeof(int32_t) * 8 * (np > 0 ? np : 1)));
    DSVD_CUDA_CHECK(cudaMemsetAsync(sc, 0, sizeof(int32_t) * 8 * (np > 0 ? np : 1), st));
    std::vector<DevCsr> v(np);
    std::vector<ChunkPlan> cp(np);
    int64_t maxrows = 1;
    for (int p = 0; p < np; ++p) maxrows = std::max(maxrows, bounds[p + 1] - bounds[p]);
    const size_t scratch_bytes = order_scratch_bytes(maxrows);
    void* scratch = ctx->buf("panel.scratch", scratch_bytes);
    for (int p = 0; p < np; ++p) {
        DevCsr& d = v[p];
        const std::string tag = "p" + std::to_string(p);
        d.rows = bounds[p + 1] - bounds[p];
        d.cols = m.cols;
        d.nnz = hoff[p + 1] - hoff[p];
        d.off = m.off + bounds[p];
        d.idx = m.idx;
        d.val = m.val;
        d.max_row_nnz = m.max_row_nnz;
        d.uniform = m.uniform;
        d.uval = m.uval;
        d.hub_threshold = m.hub_threshold;
        d.split_chunk = m.split_chunk;
        const int64_t r = d.rows > 0 ? d.rows : 1;
        d.order = static_cast<int32_t*>(al.get(tag + ".order", sizeof(int32_t) * r));
        d.obeg = static_cast<int64_t*>(al.get(tag + ".obeg", sizeof(int64_t) * r));
        d.olen = static_cast<int32_t*>(al.get(tag + ".olen", sizeof(int32_t) * r));
        d.d_hub_rows = sc + 8 * p;
        d.d_nonempty = sc + 8 * p + 1;
        d.d_long = sc + 8 * p + 2;
        d.d_mid = sc + 8 * p + 3;
        build_row_order(d, scratch, scratch_bytes, st);
        count_launch(d.rows > 0 ? 4 : 0);
        if (d.split_chunk > 0) plan_chunks_count(ctx, al, d, tag, ctx->split_panel_rows, sc + 8 * p + 4, cp[p]);
    }
    std::vector<int32_t> h(8 * (np > 0 ? np : 1));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(h.data(), sc, sizeof(int32_t) * h.size(), cudaMemcpyDeviceToHost, st));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int p = 0; p < np; ++p) {
        DevCsr& d = v[p];
        const int32_t* hp = h.data() + 8 * p;
        d.hub_rows = d.rows > 0 ? hp[0] : 0;
        d.nonempty_rows = d.rows > 0 ? hp[1] : 0;
        d.long_rows = d.rows > 0 ? hp[2] : 0;
        d.mid_rows = d.rows > 0 ? hp[3] : 0;
        if (d.split_chunk > 0) plan_chunks_emit(ctx, al, d, "p" + std::to_string(p), cp[p], hp[4], hp[5]);
    }
    return v;
}

void upload_pair(dsvd_ctx* ctx, CsrAlloc& al, int64_t rows, int64_t cols, int64_t nnz,
                 const int64_t* off, const int64_t* idx, const double* val, DevCsr& a, DevCsr& at,
                 const dsvd_config* omega_cfg) {
    cudaStream_t st = ctx->stream;
    int64_t* d_off = static_cast<int64_t*>(al.get("a.off", sizeof(int64_t) * (rows + 1)));
    int64_t* d_idx64 = ctx->tbuf<int64_t>("upload.idx64", nnz);
    double* d_val = static_cast<double*>(al.get("a.val", sizeof(double) * nnz));
    copy_h2d(ctx, d_off, off, sizeof(int64_t) * (rows + 1), st);
    // the sketch on the side stream once the offsets are there (its empty rows are not drawn)
    if (omega_cfg != nullptr) pregenerate_omega(ctx, rows, cols, *omega_cfg, d_off);
    cudaEvent_t vals = nullptr;
    if (nnz && (use_staging(ctx, idx, sizeof(int64_t) * nnz) || use_staging(ctx, val, sizeof(double) * nnz))) {
        // pageable CSR: both arrays through the staging ring, in order on st
        copy_h2d(ctx, d_idx64, idx, sizeof(int64_t) * nnz, st);
        copy_h2d(ctx, d_val, val, sizeof(double) * nnz, st);
    } else if (nnz) {
        DSVD_CUDA_CHECK(cudaMemcpyAsync(d_idx64, idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
        // the values travel on the copy stream while the structure is checked,
        // narrowed and sorted on the main stream (needed first by the CSC gather)
        if (!ctx->copy) DSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
        if (!ctx->copy_ev) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->copy_ev, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->copy_ev, st));  // d_val is free (earlier work on st)
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy, ctx->copy_ev, 0));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(d_val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->copy));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->copy_ev, ctx->copy));
        vals = ctx->copy_ev;
    }
    build_pair(ctx, al, rows, cols, nnz, d_off, d_idx64, d_val, a, at, false, vals);
}

namespace {

// ---- config validation (solver.cpp:15-32) ---------------------------------

int64_t effective_s(const dsvd_config& c) { return c.s >= 0 ? c.s : (c.k / 2 > 0 ? c.k / 2 : 1); }

void validate(const dsvd_config& cfg, int64_t rows, int64_t cols) {
    if (rows < 1 || cols < 1) fail(DSVD_SHAPE, "solver needs a non-empty matrix");
    if (cfg.k < 1) fail(DSVD_CONFIG, "k must be >= 1");
    const int64_t s = effective_s(cfg);
    if (cfg.k + s > std::min(rows, cols))
        fail(DSVD_CONFIG, "k + s = " + std::to_string(cfg.k + s) + " exceeds min(rows, cols) = " +
                              std::to_string(std::min(rows, cols)));
    if (cfg.alg == DSVD_ALG_DASH) {
        if (s < 1) fail(DSVD_CONFIG, "the accuracy-controlled mode needs oversampling s >= 1");
        if (!(cfg.tol > 0.0)) fail(DSVD_CONFIG, "tol must be positive");
        if (cfg.p_max < 1) fail(DSVD_CONFIG, "p_max must be >= 1");
    } else {
        if (cfg.p < 0) fail(DSVD_CONFIG, "fixed-power algorithms need p >= 0");
    }
    if (cfg.alg < DSVD_ALG_BASIC || cfg.alg > DSVD_ALG_DASH) fail(DSVD_CONFIG, "unknown algorithm");
    if ((cfg.flags & DSVD_FLAG_ORTH_QR) != 0 && cfg.alg != DSVD_ALG_BASIC)
        fail(DSVD_CONFIG, "the qr orthonormalizer applies to the basic algorithm only; shifted iterations need "
                          "the surrogate spectrum");
}

void raise_device_status(const Control& c) {
    if (c.status == DSVD_OK) return;
    if (c.status == DSVD_RANK_DEFICIENT && c.status_src == 1)
        fail(DSVD_RANK_DEFICIENT, "qr_orth: diagonal of R at or below the rank floor", c.status_index);
    if (c.status == DSVD_RANK_DEFICIENT)
        fail(DSVD_RANK_DEFICIENT, "eig_svd: singular value at or below the rank floor", c.status_index);
    if (c.status == DSVD_NUMERICAL)
        fail(DSVD_NUMERICAL, "eigensolver did not converge or produced non-finite values");
    fail(c.status, "device error");
}

// ---- eigSVD on a device block ----------------------------------------------

struct EigSvdOut {
    double* W;      // l x l row-major (V with the sign convention)
    double* s;      // l
    double* inv_s;  // l
};

// rescale() of the solve path: FP64 tensor cores when the shape allows
// (dmma.cu), else the DFMA kernel. Two launches either way on the DMMA path.
// With out2 != nullptr the DMMA path also writes a slab-major copy (width
// out2_w) of the row-major result and returns true; false: no copy was made.
bool solve_rescale(dsvd_ctx* ctx, const double* c, int64_t n, int64_t K, int64_t ldc, const double* w,
                   int64_t ldw, const double* scale, int64_t ncol, double* out, int64_t ld_out, int out_colmajor,
                   const int32_t* gate, double* out2 = nullptr, int out2_w = 0, const PeerOut* peers = nullptr) {
    if (ctx->dense_method == 0 && rescale_dmma_supported(K, ldc, ld_out, out_colmajor)) {
        const size_t ws = rescale_dmma_workspace_bytes(K, out_colmajor ? ncol : ld_out);
        rescale_dmma(c, n, K, ldc, w, ldw, scale, ncol, out, ld_out, out_colmajor, ctx->buf("rescale.ws", ws), gate,
                     ctx->stream, out2, out2_w, peers);
        count_launch(2);
        return out2 != nullptr;
    } else {
        if (peers != nullptr && peers->n > 0) fail(DSVD_OTHER, "rescale: peer outputs need the tensor-core rescale");
        rescale(c, n, K, ldc, w, ldw, scale, ncol, out, ld_out, out_colmajor, gate, ctx->stream);
        count_launch();
    }
    return false;
}

// (s, V) of the row-major block c (rows x l, stride ld); U is left to the caller.
void eig_svd_factors(dsvd_ctx* ctx, const double* c, int64_t rows, int64_t l, int64_t ld,
                     EigSvdOut& o, Control* ctrl, const LoopStep* loop, const int32_t* gate,
                     bool reduce_gram = false, int64_t floor_rows = -1, cudaStream_t eig_stream = nullptr,
                     int phase = 0) {
    // phase 0: all; 1: the Gram, then the tridiagonalisation on eig_stream;
    // 2: the rest of the eig and the assembly on the main stream (after phase 1)
    cudaStream_t st = ctx->stream;
    // the l x l eig and the factor assembly (latency-bound, a few SMs) may run
    // on eig_stream, after the Gram on ctx->stream (all SMs) — or, with
    // gram_async, the Gram too
    const cudaStream_t main_stream = ctx->stream;
    struct Restore {
        dsvd_ctx* c;
        cudaStream_t s;
        ~Restore() { c->stream = s; }
    } restore{ctx, main_stream};
    auto to_eig_stream = [&] {
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->ev_t, st));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(eig_stream, ctx->ev_t, 0));
        st = eig_stream;
        ctx->stream = eig_stream;  // spans; restored on return
    };
    if (eig_stream != nullptr && ctx->gram_async) to_eig_stream();
    double* G = ctx->tbuf<double>("eig.G", l * l);
    const bool tbi = ctx->eig_method == 0 && tbi_supported(static_cast<int>(l));
    if (phase == 2) {
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_eig, 0));
        EigWorkspace ew;
        void* em = ctx->buf("eig.ws", eig_workspace_bytes(static_cast<int>(l), kMaxSweeps));
        eig_workspace_bind(ew, static_cast<int>(l), kMaxSweeps, em);
        const int sp2 = ctx->span_begin(K_EIG);
        int32_t* flag = ctx->tbuf<int32_t>("tbi.flag", 1);
        tbi_eig(G, ew, ctx->buf("tbi.ws", tbi_workspace_bytes(static_cast<int>(l))), flag, gate, st, 2);
        count_launch(4);
        jacobi_eig(G, ew, ctrl, gate, st, flag);
        count_launch(1);
        eig_svd_finish(ew, floor_rows >= 0 ? floor_rows : rows, o.W, l, o.s, o.inv_s, ctrl, loop, gate, st);
        count_launch(1);
        ctx->span_end(sp2);
        return;
    }
    if (phase == 1 && (!tbi || eig_stream == nullptr)) fail(DSVD_OTHER, "eig phase 1 needs the tridiagonal path");
    int sp = ctx->span_begin(K_GRAM);
    if (ctx->dense_method == 0 && gram_dmma_supported(l, ld)) {
        const size_t gws = gram_dmma_workspace_bytes(rows, l);
        gram_dmma(c, rows, l, ld, G, ctx->buf("gram.dws." + std::to_string(rows), gws), gate, st);
    } else {
        const size_t gws = gram_workspace_bytes(rows, l);
        void* gw = ctx->buf("gram.ws." + std::to_string(rows), gws);
        gram(c, rows, l, ld, G, gw, gws, gate, st);
    }
    count_launch(2);
    ctx->span_end(sp);
    if (reduce_gram) {  // row-sharded B: G = sum_g B_g^T B_g
        sp = ctx->span_begin(K_COMM);
        comm_allreduce_sum(ctx, G, static_cast<size_t>(l * l));
        ctx->span_end(sp);
    }
    if (eig_stream != nullptr && !ctx->gram_async) to_eig_stream();
    EigWorkspace ew;
    void* em = ctx->buf("eig.ws", eig_workspace_bytes(static_cast<int>(l), kMaxSweeps));
    eig_workspace_bind(ew, static_cast<int>(l), kMaxSweeps, em);
    sp = ctx->span_begin(K_EIG);
    if (phase == 1) {
        int32_t* flag = ctx->tbuf<int32_t>("tbi.flag", 1);
        tbi_eig(G, ew, ctx->buf("tbi.ws", tbi_workspace_bytes(static_cast<int>(l))), flag, gate, st, 1);
        count_launch(2);
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->ev_eig, st));
        ctx->span_end(sp);
        return;
    }
    if (tbi) {
        // tridiagonal path; the Jacobi kernels run only if it flags a cluster
        int32_t* flag = ctx->tbuf<int32_t>("tbi.flag", 1);
        tbi_eig(G, ew, ctx->buf("tbi.ws", tbi_workspace_bytes(static_cast<int>(l))), flag, gate, st);
        count_launch(5);
        jacobi_eig(G, ew, ctrl, gate, st, flag);
        count_launch(1);
    } else {
        jacobi_eig(G, ew, ctrl, gate, st);
        count_launch(2);
    }
    eig_svd_finish(ew, floor_rows >= 0 ? floor_rows : rows, o.W, l, o.s, o.inv_s, ctrl, loop, gate, st);
    count_launch(1);
    ctx->span_end(sp);
}

Control read_control(dsvd_ctx* ctx, const Control* d) {
    Control h;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(Control), cudaMemcpyDeviceToHost, ctx->stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return h;
}

// Host copy of a row-major device block as column-major (rows x l).
std::vector<double> to_host_colmajor(dsvd_ctx* ctx, const double* d, int64_t rows, int64_t l,
                                     int64_t ld) {
    double* tmp = ctx->tbuf<double>("obs.cm", rows * l);
    rowmajor_to_colmajor(d, rows, l, ld, tmp, ctx->stream);
    count_launch();
    std::vector<double> h(static_cast<size_t>(rows * l));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(h.data(), tmp, sizeof(double) * rows * l, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return h;
}

// ---- the solve ---------------------------------------------------------------

struct SolveIO {
    // outputs (device or host per on_device); u is rows(A) x k, v is cols(A) x k
    double* u;
    double* s;
    double* v;
    bool on_device;
    double* alphas;
    double* s_hat;
    int64_t cap;
    int64_t iterations = 0;
    int stop_reason = 0;
    // column-compacted solve (build_compact): A's columns are the non-empty
    // columns v_rows[0 .. cols) of a v_full-column matrix; V is scattered back
    const int32_t* v_rows = nullptr;
    int64_t v_full = -1;
};

// Column compaction (option "compact_cols", default 1). A column of A without
// nonzeros (an empty row of A^T) leaves the matching rows of every n-row block
// exactly zero through the whole solve: T_0 = A^T Omega is 0 there, the shift
// keeps 0 at 0 (fma(-alpha, 0, 0) = +0), and the rescale maps a zero row to a
// zero row; the finalize's V = Q V' then has zero rows there too. The
// reference computes all of them (dense Gram and rescale over n rows). Here the
// solve runs on the non-empty columns only — A with its column indices
// renumbered, A^T with its empty rows dropped (same nonzero positions, row
// orders and chunk plans renumbered) — and V is scattered back with zero rows.
// Each SpMM chain and each rescaled row is computed exactly as before; the Gram
// sums the same non-zero rows over different row slabs (rounding-level
// differences, within the parity bars), and the eigSVD rank floor keeps the
// full row count. C4 (R-MAT, 46% empty columns): Gram and rescale over 2.27M
// instead of 4.19M rows, and no empty-row fill in the A^T pass.
struct Compact {
    DevCsr a, at;
    const int32_t* oldid = nullptr;
};

Compact build_compact(dsvd_ctx* ctx, const DevCsr& A, const DevCsr& AT) {
    cudaStream_t st = ctx->stream;
    const int64_t n = AT.rows, nne = AT.nonempty_rows;
    Compact c;
    c.a = A;
    c.at = AT;
    int32_t* newid = ctx->tbuf<int32_t>("cc.newid", n);
    int32_t* oldid = ctx->tbuf<int32_t>("cc.oldid", nne);
    int64_t* off_c = ctx->tbuf<int64_t>("cc.off", nne + 1);
    const size_t sb = compact_scratch_bytes(n);
    compact_rows_map(AT.off, n, newid, oldid, off_c, ctx->buf("cc.scratch", sb), sb, st);
    int32_t* idx_c = ctx->tbuf<int32_t>("cc.a.idx", A.nnz);
    remap_ids(A.idx, A.nnz, newid, idx_c, st);
    int32_t* order_c = ctx->tbuf<int32_t>("cc.at.order", nne);
    remap_ids(AT.order, nne, newid, order_c, st);  // the non-empty rows are the order's prefix
    count_launch(5);
    c.a.idx = idx_c;
    c.a.cols = nne;
    c.at.rows = nne;
    c.at.off = off_c;
    c.at.order = order_c;
    c.at.nonempty_rows = nne;
    if (c.at.long_rows > nne) c.at.long_rows = nne;
    if (c.at.mid_rows > nne) c.at.mid_rows = nne;
    c.oldid = oldid;
    return c;
}

// Shifted power iteration on the pair (A, AT) = (m x n, n x m) as given
// (solve_direct, solver.cpp:143-155): Q is a basis of A's row space.
// With a communicator attached, A is this rank's row shard (rows
// [row_offset, row_offset + m) of a global_m x n matrix): partial products are
// summed across ranks after each A^T pass and the finalize Gram; everything
// else runs redundantly on identical data, so every rank takes the same
// decisions without further exchange.
void solve_tall(dsvd_ctx* ctx, const DevCsr& A, const DevCsr& AT, const dsvd_config& cfg,
                SolveIO& io, dsvd_observer_fn observer, void* user, int64_t row_offset = 0,
                int64_t global_m = -1) {
    NvtxRange nvtx("dsvd.solve_tall");
    cudaStream_t st = ctx->stream;
    const int64_t m = A.rows, n = A.cols;
    const bool sharded = ctx->comm != nullptr;
    if (global_m < 0) global_m = m;
    const int64_t k = cfg.k;
    const int64_t l = k + effective_s(cfg);
    const int64_t ld = padded_ld(l);
    const bool dash = cfg.alg == DSVD_ALG_DASH;
    const int64_t max_iters = dash ? cfg.p_max : cfg.p;
    if (l > 512) fail(DSVD_UNSUPPORTED, "sketch width l > 512 is not supported");

    // Row-sharded v2: the n-row blocks carry n_full = G * n_slab rows
    // (zero padding rows at the end, so the reduce-scatter splits them evenly);
    // this rank owns rows [slab0, slab0 + n_slab) of every reduced sum.
    const bool v2 = sharded && ctx->mgpu_mode == 2;
    const int64_t n_slab = v2 ? ceil_div(n, ctx->nranks) : n;
    const int64_t n_full = v2 ? n_slab * ctx->nranks : n;
    const int64_t slab0 = v2 ? ctx->rank * n_slab : 0;
    // slab-major gathered blocks (column-slab kernel, lw-column slabs): the sketch
    // and Y = A Q are written slab-major; the pass-1 operand (Q or T, row-major
    // for the dense kernels) is copied into Xs before each A pass
    const int64_t big_rows = std::max(m, n);
    const int lw = slab_layout_width(ctx, ld, big_rows);
    double* Y = ctx->tbuf<double>("Y", block_doubles(m, ld, lw));  // Omega, then A Q, then B
    double* Xs = lw > 0 ? ctx->tbuf<double>("Xs", block_doubles(n, ld, lw)) : nullptr;
    double* T = ctx->tbuf<double>("T", n_full * ld);
    double* Qb[2] = {ctx->tbuf<double>("Q0", n_full * ld), ctx->tbuf<double>("Q1", n_full * ld)};
    double* S = v2 ? ctx->tbuf<double>("slab", n_slab * ld) : nullptr;
    if (n_full > n) {  // padding rows stay zero: SpMM writes rows [0, n) only
        for (double* b : {T, Qb[0], Qb[1]})
            DSVD_CUDA_CHECK(cudaMemsetAsync(b + n * ld, 0, sizeof(double) * (n_full - n) * ld, st));
    }
    double* W = ctx->tbuf<double>("W", l * l);
    double* sv = ctx->tbuf<double>("s", l);
    double* inv_s = ctx->tbuf<double>("inv_s", l);
    double* s_stored = ctx->tbuf<double>("s_stored", l);
    Control* ctrl = ctx->tbuf<Control>("ctrl", 1);
    const int64_t cap = max_iters > 0 ? max_iters : 1;
    double* d_alphas = ctx->tbuf<double>("trace.alphas", cap);
    double* d_shat = ctx->tbuf<double>("trace.s_hat", cap * l);
    EigSvdOut eo{W, sv, inv_s};
    const int32_t* gate = &ctrl->stopped;

    control_init(ctrl, s_stored, static_cast<int>(l), st);
    count_launch();

    // Omega = gaussian_matrix(m, l, seed) (solver.cpp:83), unless it was already
    // generated beside the host upload (pregenerate_omega)
    int sp = ctx->span_begin(K_OTHER);
    if (ctx->omega_pending && !sharded && ctx->omega_m == m && ctx->omega_l == l && ctx->omega_seed == cfg.seed &&
        ctx->omega_slab_w == lw) {
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->omega_ev, 0));
    } else {
        gaussian_rowmajor(Y, m, l, ld, cfg.seed, st, global_m, row_offset, lw, A.off);
        count_launch();
    }
    ctx->omega_pending = false;
    ctx->span_end(sp);

    LoopStep ls;
    ls.k = k;
    ls.tol = cfg.tol;
    ls.alg = cfg.alg;
    ls.alphas = d_alphas;
    ls.s_hat = d_shat;
    ls.cap = cap;
    ls.s_stored = s_stored;
    if (dash && ctx->host_flags == nullptr) {
        DSVD_CUDA_CHECK(cudaMallocHost(&ctx->host_flags, sizeof(int32_t) * (kLookahead + 1)));
    }
    std::vector<cudaEvent_t> flag_ev(kLookahead + 1, nullptr);
    Control hc;
    const double* Qf = nullptr;
    // auto: pipelined when the eig chain it hides is worth >= 5% of the two
    // SpMM passes it overlaps (gathers at ~20 TB/s; eig ~0.65 ms at l = 150,
    // quadratic in l; tools/ab_option.py pipeline on C2 / C3 / C4 in DESIGN 5)
    // (sharded: from the GLOBAL nnz, so every rank takes the same schedule — the
    // two schedules reduce different partials, A^T A T_{j-1} vs A^T A Q_{j-1})
    const double nnz_sched = (sharded && ctx->pipeline < 0) ? comm_sum_host(ctx, static_cast<double>(A.nnz))
                                                            : static_cast<double>(A.nnz);
    const double eig_s = 0.65e-3 * (static_cast<double>(l) / 150.0) * (static_cast<double>(l) / 150.0);
    // eig_s >= 0.05 spmm_s with spmm_s = 2 nnz ld 8 B / 20 TB/s, as an nnz bound
    const double nnz_auto = ctx->pipeline_auto_nnz > 0 ? static_cast<double>(ctx->pipeline_auto_nnz)
                                                       : eig_s / (0.05 * 2.0 * static_cast<double>(ld) * 8.0 / 20e12);
    const bool pipelined = ctx->pipeline == 1 || (ctx->pipeline < 0 && nnz_sched <= nnz_auto);
    ctx->stats.pipelined = pipelined ? 1 : 0;
    // Sharded exchange of an n x l partial P (the A^T pass of this rank's rows):
    // v1 all-reduces it in place and returns P (n rows); v2 reduce-scatters it
    // and returns this rank's n_slab-row slab of the sum.
    auto reduce_partial = [&](double* part) -> double* {
        const int s2 = ctx->span_begin(K_COMM);
        if (v2) comm_reduce_scatter_sum(ctx, part, S, static_cast<size_t>(n_slab * ld));
        else comm_allreduce_sum(ctx, part, static_cast<size_t>(n * ld));
        ctx->span_end(s2);
        return v2 ? S : part;
    };
    // rows of a reduced block handled by this rank, and their offset in a full block
    const int64_t red_rows = v2 ? n_slab : n;
    // eigSVD rank floor of the n-row blocks: the full row count (v2: the global n;
    // a column-compacted solve: the uncompacted n)
    const int64_t n_floor = io.v_full > 0 ? io.v_full : (v2 ? n : -1);
    // Exchange overlap (mgpu_overlap): the A^T pass in G row panels (the v2 slabs);
    // each panel's partial is reduced (v2: to its owner rank; v1: all-reduced) on
    // the communication stream while the next panel computes. Same values as the
    // whole-pass collective: bitwise in the loopback group's fixed rank order.
    const bool overlap = sharded && ctx->nranks > 1 && ctx->mgpu_overlap;
    // fused exchange (mgpu_overlap 2, v2): each panel's SpMM stores its rows
    // straight into the owner's landing buffer (slot `rank`), a barrier, then the
    // owner sums its G slots in rank order — no separate reduction collective
    const bool fused = overlap && v2 && ctx->mgpu_overlap == 2;
    std::vector<void*> peers;
    struct PeerGuard {
        dsvd_ctx* c;
        std::vector<void*>* p;
        ~PeerGuard() { comm_close_peers(c, *p); }
    } peer_guard{ctx, &peers};
    if (fused) {
        const size_t lb = sizeof(double) * static_cast<size_t>(ctx->nranks) * n_slab * ld;
        if (ctx->landing_bytes != lb) {
            if (ctx->landing) DSVD_CUDA_CHECK(cudaFree(ctx->landing));
            ctx->landing = nullptr;
            ctx->landing_bytes = 0;
            DSVD_CUDA_CHECK(cudaMalloc(&ctx->landing, lb));
            ctx->landing_bytes = lb;
            // padding rows of the last panel are never stored: they stay zero
            DSVD_CUDA_CHECK(cudaMemsetAsync(ctx->landing, 0, lb, st));
            DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
        }
        comm_exchange_peers(ctx, ctx->landing, peers);
    }
    // fused all-gather: the rescale stores each slab row into every rank's copy of
    // the destination block (the tensor-core rescale; peers of T, Q0 and Q1)
    const bool fused_ag = fused && ctx->dense_method == 0 && rescale_dmma_supported(l, ld, ld, 0) &&
                          ctx->nranks - 1 <= kMaxPeerOut;
    std::map<const double*, std::vector<void*>> blk_peers;
    struct BlkGuard {
        dsvd_ctx* c;
        std::map<const double*, std::vector<void*>>* m;
        ~BlkGuard() {
            for (auto& kv : *m) comm_close_peers(c, kv.second);
        }
    } blk_guard{ctx, &blk_peers};
    if (fused_ag)
        for (double* b : {T, Qb[0], Qb[1]}) comm_exchange_peers(ctx, b, blk_peers[b]);
    std::vector<DevCsr> panels;
    if (overlap) {
        const int64_t ps = ceil_div(n, ctx->nranks);
        std::vector<int64_t> bounds;
        for (int g = 0; g <= ctx->nranks; ++g) bounds.push_back(std::min(n, g * ps));
        panels = build_row_panels(ctx, AT, bounds);
        if (!ctx->comm_stream) DSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
        if (!ctx->comm_ev) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->comm_ev, cudaEventDisableTiming));
        int64_t maxc = 0;
        for (const DevCsr& pv : panels) maxc = std::max(maxc, pv.nchunks);
        if (maxc > 0) ctx->tbuf<double>("spmm.partial", maxc * ld);  // sized once, before the loop
    }
    // SpMM launches of the loop: pass 1 (A x -> Y) reads its row-major operand
    // through the slab-major copy Xs and writes Y slab-major when lw > 0; pass 2
    // (A^T Y [- alpha q] -> out, row-major) then gathers the slab-major Y
    // hot/cold tags for the slab kernel's L2 policies: the hot X rows of pass 1 are
    // the longest rows of A^T (most referenced columns of A), of pass 2 the
    // longest rows of A
    const int32_t* tag_a = nullptr;
    const int32_t* tag_at = nullptr;
    if (lw > 0 && ctx->spmm_hot_mb > 0 && A.nnz > 0) {
        const int64_t k_hot = ctx->spmm_hot_mb * (int64_t(1) << 20) / (8 * lw);
        uint8_t* hot = ctx->tbuf<uint8_t>("hot.flags", std::max(m, n));
        int32_t* ta = ctx->tbuf<int32_t>("tag.a", A.nnz);
        int32_t* tt = ctx->tbuf<int32_t>("tag.at", AT.nnz);
        tag_hot_indices(A, AT.order, k_hot, hot, ta, st);
        tag_hot_indices(AT, A.order, k_hot, hot, tt, st);
        count_launch(4);
        tag_a = ta;
        tag_at = tt;
    }
    // the block whose slab-major copy Xs currently holds (written by the
    // rescale that produced it, single-GPU solves), so pass 1 skips the copy
    const double* xs_holds = nullptr;
    auto pass1 = [&](const double* x, double* y_out, bool y_slab_major, const int32_t* g) {
        SpmmArgs sa{&A, x, y_out, ld, l, nullptr, nullptr, g};
        sa.idx_tag = tag_a;
        if (lw > 0) {
            if (xs_holds != x) {
                to_slab_major(x, n, ld, lw, Xs, st);
                count_launch();
                xs_holds = x;
            }
            sa.x = Xs;
            sa.slab = lw;
            sa.x_slab = true;
            sa.y_slab = y_slab_major;
            sa.skip_empty = y_slab_major;  // the loop's A Q: empty rows of A are never gathered by A^T
        }
        spmm(sa, st, spmm_var(ctx, ld, big_rows), ctx->side, ctx->fork, ctx->join, partial_for(ctx, A, ld));
        count_launch();
    };
    auto pass2 = [&](double* out, const double* q, const double* alpha, const int32_t* g) {
        SpmmArgs sa{&AT, Y, out, ld, l, q, alpha, g};
        sa.idx_tag = tag_at;
        if (lw > 0) {
            sa.slab = lw;
            sa.x_slab = true;
        }
        spmm(sa, st, spmm_var(ctx, ld, big_rows), ctx->side, ctx->fork, ctx->join, partial_for(ctx, AT, ld));
        count_launch();
    };
    // Sharded A^T pass + exchange: returns the reduced block (v1: part, v2: S)
    auto pass2_reduce = [&](double* part, const int32_t* g) -> double* {
        if (!overlap) {
            pass2(part, nullptr, nullptr, g);
            return reduce_partial(part);
        }
        const int64_t ps = ceil_div(n, ctx->nranks);
        if (fused) {
            for (int p = 0; p < ctx->nranks; ++p) {
                double* dst = static_cast<double*>(peers[p]) + ctx->rank * n_slab * ld;  // owner p, slot rank
                SpmmArgs sa{&panels[p], Y, dst, ld, l, nullptr, nullptr, g};
                sa.idx_tag = tag_at;
                if (lw > 0) {
                    sa.slab = lw;
                    sa.x_slab = true;
                }
                spmm(sa, st, spmm_var(ctx, ld, big_rows), ctx->side, ctx->fork, ctx->join,
                     partial_for(ctx, panels[p], ld));
                count_launch();
            }
            const int sp3 = ctx->span_begin(K_COMM);
            comm_barrier(ctx, st);  // every rank's stores into every landing buffer are done
            comm_sum_slots(ctx->landing, ctx->nranks, static_cast<size_t>(n_slab * ld), S, st);
            count_launch();
            ctx->span_end(sp3);
            return S;
        }
        for (int p = 0; p < ctx->nranks; ++p) {
            const int64_t r0 = std::min(n, p * ps);
            SpmmArgs sa{&panels[p], Y, part + r0 * ld, ld, l, nullptr, nullptr, g};
            sa.idx_tag = tag_at;
            if (lw > 0) {
                sa.slab = lw;
                sa.x_slab = true;
            }
            spmm(sa, st, spmm_var(ctx, ld, big_rows), ctx->side, ctx->fork, ctx->join,
                 partial_for(ctx, panels[p], ld));
            count_launch();
            DSVD_CUDA_CHECK(cudaEventRecord(ctx->comm_ev, st));
            DSVD_CUDA_CHECK(cudaStreamWaitEvent(ctx->comm_stream, ctx->comm_ev, 0));
            if (v2)  // rows [p n_slab, (p+1) n_slab) of the sum (zero padding rows included) to rank p
                comm_reduce_sum(ctx, part + p * n_slab * ld, S, static_cast<size_t>(n_slab * ld), p,
                                ctx->comm_stream);
            else
                comm_allreduce_sum(ctx, part + r0 * ld, static_cast<size_t>((std::min(n, r0 + ps) - r0) * ld),
                                   ctx->comm_stream);
        }
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->comm_ev, ctx->comm_stream));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->comm_ev, 0));
        return v2 ? S : part;
    };
    // eigSVD factors of a reduced block (v2: slab Gram + l x l all-reduce)
    auto factors = [&](const double* c, const LoopStep* lsp, const int32_t* g, cudaStream_t es) {
        eig_svd_factors(ctx, c, red_rows, l, ld, eo, ctrl, lsp, g, v2, n_floor, es);
    };
    // dst (full n-row block) = c W diag(1/s) for a reduced block c; v2 rescales
    // the slab into its rows of dst and all-gathers the other ranks' slabs
    auto rescale_into = [&](const double* c, double* dst, const int32_t* g) {
        int s2 = ctx->span_begin(K_RESCALE);
        const bool copy = lw > 0 && !sharded;  // the next A pass gathers dst: write its slab-major copy too
        auto bp = blk_peers.find(dst);
        if (fused_ag && bp != blk_peers.end()) {
            // this rank's slab rows, stored into every rank's dst; then a barrier for the all-gather
            PeerOut po{};
            for (int r = 0; r < ctx->nranks; ++r)
                if (r != ctx->rank) po.p[po.n++] = static_cast<double*>(bp->second[r]) + slab0 * ld;
            solve_rescale(ctx, c, red_rows, l, ld, W, l, inv_s, l, dst + slab0 * ld, ld, 0, g, nullptr, 0, &po);
            xs_holds = nullptr;
            ctx->span_end(s2);
            s2 = ctx->span_begin(K_COMM);
            comm_barrier(ctx, st);
            ctx->span_end(s2);
            return;
        }
        xs_holds = solve_rescale(ctx, c, red_rows, l, ld, W, l, inv_s, l, dst + slab0 * ld, ld, 0, g,
                                 copy ? Xs : nullptr, lw) ? dst : nullptr;
        ctx->span_end(s2);
        if (v2) {
            s2 = ctx->span_begin(K_COMM);
            comm_allgather(ctx, dst + slab0 * ld, dst, static_cast<size_t>(n_slab * ld));
            ctx->span_end(s2);
        }
    };
    if (pipelined) {
        // Deferred rescale. With Q_{j-1} = T_{j-1} W_{j-1} (W = V diag(1/s) of
        // eigSVD(T_{j-1}), sign convention folded in), the reference's
        //   T_j = A^T (A Q_{j-1}) - alpha Q_{j-1}            (solver.cpp:92-95)
        // equals (A^T (A T_{j-1}) - alpha T_{j-1}) W_{j-1}. Both SpMM passes run on
        // T_{j-1}, so once the Gram of T_{j-1} is formed (all SMs), its l x l eig
        // and the shift/stop update (a latency-bound chain on a few SMs) run on
        // the priority stream beside the A T_{j-1} pass instead of between the
        // passes; the A^T pass waits for them
        // (it needs the updated alpha), and one rescale forms T_j. The trace,
        // stop rule and alpha updates are the same device code on the same
        // values; Q_N = T_N W_N is formed once for the finalize.
        double* Tb[2] = {T, Qb[0]};
        double* P = Qb[1];
        // Gram on st (all SMs), then the eig chain on the priority stream
        // eig_overlap (DESIGN 5): 1 runs the whole eig chain on the priority stream
        // beside the A T pass; 2 (default) only the tridiagonalisation there and the
        // short multi-CTA kernels after the pass on the main stream (at high
        // priority their CTAs cost the gathering pass more than they take: C4
        // pass 1 20.1 -> 23.2 ms); 0 the whole chain after the pass
        // auto (-1): split above l = 160, where the tridiagonalisation is the long
        // L2-resident kernel (C4: 2.74 -> 2.68 s); whole chain beside the pass below
        // (C2: 73.6 vs 75.6 ms split); the split needs the tridiagonal eigensolver
        const bool tbi_ok = ctx->eig_method == 0 && tbi_supported(static_cast<int>(l));
        int eov = ctx->eig_overlap < 0 ? (l > 160 ? 2 : 1) : ctx->eig_overlap;
        if (observer || (eov == 2 && !tbi_ok)) eov = 1;
        const double* inl_t = nullptr;
        const LoopStep* inl_ls = nullptr;
        const int32_t* inl_g = nullptr;
        int64_t inl_j = -1;  // iteration whose stop flag the deferred part decides
        auto eig_async = [&](const double* tj, const LoopStep* lsp, const int32_t* g, int64_t jj) {
            if (eov == 1) {
                factors(tj + slab0 * ld, lsp, g, ctx->eig);  // v2: this rank's slab of T_j
                DSVD_CUDA_CHECK(cudaEventRecord(ctx->ev_eig, ctx->eig));
                return;
            }
            if (eov == 2)  // Gram on st, the tridiagonalisation on the eig stream
                eig_svd_factors(ctx, tj + slab0 * ld, red_rows, l, ld, eo, ctrl, lsp, g, v2, n_floor, ctx->eig,
                                1);
            inl_t = tj;
            inl_ls = lsp;
            inl_g = g;
            inl_j = jj;
        };
        // dash: the host's lookahead reads of stop_pending after eigSVD(T_jj)
        auto flag_copy = [&](int64_t jj, cudaStream_t fs) {
            if (!dash || jj < 1) return;
            const int slot = static_cast<int>(jj % (kLookahead + 1));
            if (flag_ev[slot] == nullptr) flag_ev[slot] = ctx->event();
            DSVD_CUDA_CHECK(cudaMemcpyAsync(&ctx->host_flags[slot], &ctrl->stop_pending, sizeof(int32_t),
                                            cudaMemcpyDeviceToHost, fs));
            DSVD_CUDA_CHECK(cudaEventRecord(flag_ev[slot], fs));
        };
        auto eig_deferred = [&] {  // the deferred part, on the main stream
            if (inl_t == nullptr) return;
            if (eov == 2)
                eig_svd_factors(ctx, inl_t + slab0 * ld, red_rows, l, ld, eo, ctrl, inl_ls, inl_g, v2, n_floor,
                                nullptr, 2);
            else
                factors(inl_t + slab0 * ld, inl_ls, inl_g, nullptr);
            DSVD_CUDA_CHECK(cudaEventRecord(ctx->ev_eig, st));
            flag_copy(inl_j, st);
            inl_t = nullptr;
        };
        double* Qobs[2] = {nullptr, nullptr};
        if (observer) {
            Qobs[0] = ctx->tbuf<double>("obs.q0", n * ld);
            Qobs[1] = ctx->tbuf<double>("obs.q1", n * ld);
        }
        // T_0 = A^T Omega; eigSVD(T_0) gives Q_0 = T_0 W_0 (solver.cpp:84)
        double* red0 = nullptr;
        sp = ctx->span_begin(K_SPMM2);
        if (sharded) red0 = pass2_reduce(Tb[0], nullptr);
        else pass2(Tb[0], nullptr, nullptr, nullptr);
        ctx->span_end(sp);
        if (sharded) {
            double* red = red0;
            if (v2) {  // T_0 = the gathered slabs of the sum
                DSVD_CUDA_CHECK(cudaMemcpyAsync(Tb[0] + slab0 * ld, red, sizeof(double) * n_slab * ld,
                                                cudaMemcpyDeviceToDevice, st));
                sp = ctx->span_begin(K_COMM);
                comm_allgather(ctx, Tb[0] + slab0 * ld, Tb[0], static_cast<size_t>(n_slab * ld));
                ctx->span_end(sp);
            }
        }
        eig_async(Tb[0], nullptr, nullptr, 0);
        if (observer) {
            DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_eig, 0));
            solve_rescale(ctx, Tb[0], n, l, ld, W, l, inv_s, l, Qobs[0], ld, 0, nullptr);
        }
        for (int64_t j = 1; j <= max_iters; ++j) {
            NvtxRange nvtx_it("dsvd.iteration");
            if (dash && !observer && j > kLookahead) {
                const int slot = static_cast<int>((j - kLookahead) % (kLookahead + 1));
                DSVD_CUDA_CHECK(cudaEventSynchronize(flag_ev[slot]));
                if (ctx->host_flags[slot]) break;
            }
            double* tprev = Tb[(j - 1) % 2];
            // Z = A T_{j-1}, beside eigSVD(T_{j-1}) (its output is only needed if
            // the loop continues, so a stop decided there just skips the rest)
            // (dash: gated on stop_pending, which eigSVD(T_{j-1}) may set while
            // this pass runs — blocks starting after a stop skip their rows)
            sp = ctx->span_begin(K_SPMM1);
            pass1(tprev, Y, true, dash ? &ctrl->stop_pending : gate);
            ctx->span_end(sp);
            eig_deferred();
            if (ctx->shift_after) {
                // P = A^T Z before the wait (both passes overlap the eig), then
                // P <- fma(-alpha, T_{j-1}, P): the same bits as the fused epilogue
                double* red = P;
                sp = ctx->span_begin(K_SPMM2);
                if (sharded) red = pass2_reduce(P, dash ? &ctrl->stop_pending : gate);
                else pass2(P, nullptr, nullptr, dash ? &ctrl->stop_pending : gate);
                ctx->span_end(sp);
                DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_eig, 0));
                loop_begin(ctrl, st);
                count_launch();
                shift_update(red, tprev + slab0 * ld, red_rows * ld, &ctrl->alpha, gate, st);
                count_launch();
                rescale_into(red, Tb[j % 2], gate);
            } else {
                DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_eig, 0));
                loop_begin(ctrl, st);
                count_launch();
                // P = A^T Z - alpha T_{j-1}  (the shift skipped when alpha == 0)
                double* red = P;
                sp = ctx->span_begin(K_SPMM2);
                if (sharded) red = pass2_reduce(P, gate);
                else pass2(P, tprev, &ctrl->alpha, gate);
                ctx->span_end(sp);
                if (sharded) {
                    shift_update(red, tprev + slab0 * ld, red_rows * ld, &ctrl->alpha, gate, st);
                    count_launch();
                }
                // T_j = P W_{j-1} diag(1/s_{j-1})  (= A^T A Q_{j-1} - alpha Q_{j-1})
                rescale_into(red, Tb[j % 2], gate);
            }
            eig_async(Tb[j % 2], &ls, gate, j);
            if (eov == 1) flag_copy(j, ctx->eig);
            if (observer) {
                DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_eig, 0));
                Control oc = read_control(ctx, ctrl);
                raise_device_status(oc);
                solve_rescale(ctx, Tb[j % 2], n, l, ld, W, l, inv_s, l, Qobs[j % 2], ld, 0, nullptr);
                std::vector<double> qb = to_host_colmajor(ctx, Qobs[(j - 1) % 2], n, l, ld);
                std::vector<double> qa = to_host_colmajor(ctx, Qobs[j % 2], n, l, ld);
                std::vector<double> sh(static_cast<size_t>(l));
                double alpha_used = 0.0;
                DSVD_CUDA_CHECK(cudaMemcpy(sh.data(), d_shat + (j - 1) * l, sizeof(double) * l,
                                           cudaMemcpyDeviceToHost));
                DSVD_CUDA_CHECK(cudaMemcpy(&alpha_used, d_alphas + (j - 1), sizeof(double),
                                           cudaMemcpyDeviceToHost));
                observer(j, alpha_used, sh.data(), l, qb.data(), qa.data(), n, user);
                if (oc.stop_pending) break;
            }
        }
        eig_deferred();
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->ev_eig, ctx->eig));  // incl. the last flag copy
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_eig, 0));
        hc = read_control(ctx, ctrl);
        raise_device_status(hc);
        io.iterations = hc.iteration;
        io.stop_reason = dash ? (hc.stop_pending ? DSVD_STOP_TOL_MET : DSVD_STOP_P_MAX_REACHED)
                              : DSVD_STOP_FIXED_P;
        ctx->stats.eig_sweeps = hc.total_sweeps;
        // Q_N = T_N W_N diag(1/s_N): the basis the finalize multiplies by A
        sp = ctx->span_begin(K_RESCALE);
        xs_holds = solve_rescale(ctx, Tb[hc.iteration % 2], n, l, ld, W, l, inv_s, l, P, ld, 0, nullptr,
                                 lw > 0 && !sharded ? Xs : nullptr, lw) ? P : nullptr;
        ctx->span_end(sp);
        Qf = P;
    } else {
        // Q = eigSVD(A^T Omega).u
        sp = ctx->span_begin(K_SPMM2);
        const double* red0 = T;
        if (sharded) red0 = pass2_reduce(T, nullptr);
        else pass2(T, nullptr, nullptr, nullptr);
        ctx->span_end(sp);
        factors(red0, nullptr, nullptr, nullptr);
        rescale_into(red0, Qb[0], nullptr);


        int cur = 0;
        for (int64_t j = 1; j <= max_iters; ++j) {
            NvtxRange nvtx_it("dsvd.iteration");
            if (dash && !observer && j > kLookahead) {
                const int slot = static_cast<int>((j - kLookahead) % (kLookahead + 1));
                DSVD_CUDA_CHECK(cudaEventSynchronize(flag_ev[slot]));
                if (ctx->host_flags[slot]) break;
            }
            loop_begin(ctrl, st);
            count_launch();
            // Y = A Q
            sp = ctx->span_begin(K_SPMM1);
            pass1(Qb[cur], Y, true, gate);
            ctx->span_end(sp);
            // T = A^T Y - alpha Q  (add_scaled skipped when alpha == 0)
            sp = ctx->span_begin(K_SPMM2);
            double* red = T;
            if (sharded) red = pass2_reduce(T, gate);
            else pass2(T, Qb[cur], &ctrl->alpha, gate);
            ctx->span_end(sp);
            if (sharded) {
                // sum the partials first, then apply the shift once (solver.cpp:94)
                shift_update(red, Qb[cur] + slab0 * ld, red_rows * ld, &ctrl->alpha, gate, st);
                count_launch();
            }
            factors(red, &ls, gate, nullptr);
            rescale_into(red, Qb[1 - cur], gate);
            if (dash) {
                const int slot = static_cast<int>(j % (kLookahead + 1));
                if (flag_ev[slot] == nullptr) flag_ev[slot] = ctx->event();
                DSVD_CUDA_CHECK(cudaMemcpyAsync(&ctx->host_flags[slot], &ctrl->stop_pending,
                                                sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                DSVD_CUDA_CHECK(cudaEventRecord(flag_ev[slot], st));
            }
            if (observer) {
                hc = read_control(ctx, ctrl);
                raise_device_status(hc);
                std::vector<double> qb = to_host_colmajor(ctx, Qb[cur], n, l, ld);
                std::vector<double> qa = to_host_colmajor(ctx, Qb[1 - cur], n, l, ld);
                std::vector<double> sh(static_cast<size_t>(l));
                double alpha_used = 0.0;
                DSVD_CUDA_CHECK(cudaMemcpy(sh.data(), d_shat + (j - 1) * l, sizeof(double) * l,
                                           cudaMemcpyDeviceToHost));
                DSVD_CUDA_CHECK(cudaMemcpy(&alpha_used, d_alphas + (j - 1), sizeof(double),
                                           cudaMemcpyDeviceToHost));
                observer(j, alpha_used, sh.data(), l, qb.data(), qa.data(), n, user);
                if (hc.stop_pending) {
                    cur = 1 - cur;
                    break;
                }
            }
            cur = 1 - cur;
        }
        hc = read_control(ctx, ctrl);
        raise_device_status(hc);
        io.iterations = hc.iteration;
        io.stop_reason = dash ? (hc.stop_pending ? DSVD_STOP_TOL_MET : DSVD_STOP_P_MAX_REACHED)
                              : DSVD_STOP_FIXED_P;
        ctx->stats.eig_sweeps = hc.total_sweeps;
        Qf = Qb[hc.iteration % 2];
    }

    // finalize_row_basis: B = A Q, eigSVD(B), U = B V' diag(1/s) [:, :k], V = Q V'[:, :k]
    NvtxRange nvtx_fin("dsvd.finalize");
    control_init(ctrl, s_stored, static_cast<int>(l), st);
    count_launch();
    // Row compaction of the finalize (single GPU, column-slab path): B's rows of
    // empty rows of A are exactly zero, so B is formed on the non-empty rows only
    // — a view of A whose length order is renumbered to compact row ids (the slab
    // kernels read each row's range from obeg / olen, not from the offsets) — and
    // the Gram and U = B V' diag(1/s) run on them; U is scattered back with zero
    // rows. The rank floor keeps the full row count.
    const int64_t m_ne = A.nonempty_rows;
    const bool compact_m = ctx->compact_cols && !sharded && lw > 0 && A.obeg != nullptr && m_ne >= l &&
                           m_ne < m && (m - m_ne) * 50 >= m;
    const int32_t* oldid_m = nullptr;
    const int64_t m_b = compact_m ? m_ne : m;
    sp = ctx->span_begin(K_SPMM1);
    if (compact_m) {
        int32_t* newid = ctx->tbuf<int32_t>("ccm.newid", m);
        int32_t* oldid = ctx->tbuf<int32_t>("ccm.oldid", m_ne);
        int64_t* off_c = ctx->tbuf<int64_t>("ccm.off", m_ne + 1);
        const size_t sb = compact_scratch_bytes(m);
        compact_rows_map(A.off, m, newid, oldid, off_c, ctx->buf("cc.scratch", sb), sb, st);
        int32_t* order_c = ctx->tbuf<int32_t>("ccm.order", m_ne);
        remap_ids(A.order, m_ne, newid, order_c, st);  // the non-empty rows are the order's prefix
        count_launch(4);
        DevCsr Av = A;
        Av.rows = m_ne;
        Av.off = off_c;
        Av.order = order_c;
        Av.nonempty_rows = m_ne;
        Av.long_rows = std::min(Av.long_rows, m_ne);
        Av.mid_rows = std::min(Av.mid_rows, m_ne);
        if (xs_holds != Qf) {
            to_slab_major(Qf, n, ld, lw, Xs, st);
            count_launch();
            xs_holds = Qf;
        }
        SpmmArgs sa{&Av, Xs, Y, ld, l, nullptr, nullptr, nullptr};
        sa.idx_tag = tag_a;
        sa.slab = lw;
        sa.x_slab = true;
        spmm(sa, st, spmm_var(ctx, ld, big_rows), ctx->side, ctx->fork, ctx->join, partial_for(ctx, Av, ld));
        count_launch();
        oldid_m = oldid;
    } else {
        pass1(Qf, Y, false, nullptr);  // B row-major: the Gram and the U product read it
    }
    ctx->span_end(sp);
    eig_svd_factors(ctx, Y, m_b, l, ld, eo, ctrl, nullptr, nullptr, sharded, global_m);
    hc = read_control(ctx, ctrl);
    raise_device_status(hc);
    ctx->stats.eig_sweeps += hc.total_sweeps;

    double* du = io.on_device && !compact_m ? io.u : ctx->tbuf<double>(compact_m ? "out.uc" : "out.u", m_b * k);
    const bool scatter_v = io.v_rows != nullptr;
    const int64_t n_out = scatter_v ? io.v_full : n;
    double* dv = io.on_device && !scatter_v ? io.v : ctx->tbuf<double>(scatter_v ? "out.vc" : "out.v", n * k);
    // V first: with host outputs its device->host copy (PCIe-bound, ~0.12 s at C4)
    // runs on the copy stream while U is formed
    sp = ctx->span_begin(K_RESCALE);
    solve_rescale(ctx, Qf, n, l, ld, W, l, nullptr, k, dv, 0, 1, nullptr);
    if (scatter_v) {  // V of the compacted columns -> the full column set (zero rows elsewhere)
        double* dvf = io.on_device ? io.v : ctx->tbuf<double>("out.v", n_out * k);
        scatter_rows_colmajor(dv, n, k, io.v_rows, dvf, n_out, st);
        count_launch();
        dv = dvf;
    }
    cudaStream_t vs = st;
    // pageable V: staged after U's rescale is enqueued (the staged copy blocks the host)
    const bool v_staged = !io.on_device && use_staging(ctx, io.v, sizeof(double) * n_out * k);
    if (v_staged) {
        if (!ctx->stage_ready) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->stage_ready, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->stage_ready, st));
    } else if (!io.on_device) {
        if (!ctx->copy) DSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
        if (!ctx->copy_ev) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->copy_ev, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->copy_ev, st));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy, ctx->copy_ev, 0));
        vs = ctx->copy;
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.v, dv, sizeof(double) * n_out * k, cudaMemcpyDeviceToHost, vs));
    }
    solve_rescale(ctx, Y, m_b, l, ld, W, l, inv_s, k, du, 0, 1, nullptr);
    if (compact_m) {  // U of the non-empty rows -> all rows (zero rows elsewhere)
        double* duf = io.on_device ? io.u : ctx->tbuf<double>("out.u", m * k);
        scatter_rows_colmajor(du, m_ne, k, oldid_m, duf, m, st);
        count_launch();
        du = duf;
    }
    ctx->span_end(sp);
    if (io.on_device) {
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.s, sv, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
    } else {
        sp = ctx->span_begin(K_OTHER);
        if (v_staged) copy_d2h(ctx, io.v, dv, sizeof(double) * n_out * k, st, ctx->stage_ready);
        copy_d2h(ctx, io.u, du, sizeof(double) * m * k, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.s, sv, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
        if (!v_staged) {
            DSVD_CUDA_CHECK(cudaEventRecord(ctx->copy_ev, vs));  // V's copy is part of the solve
            DSVD_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->copy_ev, 0));
        }
        ctx->span_end(sp);
    }
    const int64_t nrec = std::min(io.iterations, io.cap);
    if (nrec > 0 && io.alphas)
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.alphas, d_alphas, sizeof(double) * nrec,
                                        cudaMemcpyDeviceToHost, st));
    if (nrec > 0 && io.s_hat)
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.s_hat, d_shat, sizeof(double) * nrec * l,
                                        cudaMemcpyDeviceToHost, st));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
}

void begin_profile(dsvd_ctx* ctx) {
    ctx->stats = dsvd_stats{};
    ctx->spans.clear();
    ctx->event_next = 0;
}

void end_profile(dsvd_ctx* ctx, int64_t launches_before) {
    dsvd_stats& s = ctx->stats;
    s.kernel_launches = g_launches.load() - launches_before;
    if (!ctx->profiling) return;
    for (const auto& sp : ctx->spans) {
        float ms = 0.f;
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms, sp.a, sp.b));
        switch (sp.cls) {
            case K_SPMM1:
                s.spmm_pass_ms[0] += ms;
                s.spmm_pass_launches[0] += 1;
                s.spmm_ms += ms;
                s.spmm_launches += 1;
                break;
            case K_SPMM2:
                s.spmm_pass_ms[1] += ms;
                s.spmm_pass_launches[1] += 1;
                s.spmm_ms += ms;
                s.spmm_launches += 1;
                break;
            case K_GRAM: s.gram_ms += ms; break;
            case K_EIG: s.eig_ms += ms; break;
            case K_RESCALE: s.rescale_ms += ms; break;
            case K_COMM: s.allreduce_ms += ms; break;
            default: break;
        }
    }
}


// basic_core + finalize_col_basis (solver.cpp:118-141, :166-176) on the pair
// (A, AT) as given: Omega = gaussian_matrix(n, l, seed), q = orth(A Omega),
// then p times q = orth(A (A^T q)); orth = eigSVD(.).u (the default
// Orthonormalizer::eigsvd; its spectrum is the trace's s_hat, alphas are 0).
// Finalize: f = eigSVD(A^T q), U = q f.v[:, :k], V = f.u[:, :k], s = f.s[:k].
void solve_basic(dsvd_ctx* ctx, const DevCsr& A, const DevCsr& AT, const dsvd_config& cfg, SolveIO& io,
                 dsvd_observer_fn observer, void* user) {
    NvtxRange nvtx("dsvd.solve_basic");
    cudaStream_t st = ctx->stream;
    const int64_t m = A.rows, n = A.cols;
    const int64_t k = cfg.k;
    const int64_t l = k + effective_s(cfg);
    const int64_t ld = padded_ld(l);
    const int64_t p = cfg.p;
    if (l > 512) fail(DSVD_UNSUPPORTED, "sketch width l > 512 is not supported");
    const bool qr = (cfg.flags & DSVD_FLAG_ORTH_QR) != 0;
    if (qr && l > 160) fail(DSVD_UNSUPPORTED, "the device QR orthonormalizer supports l <= 160");

    double* Y = ctx->tbuf<double>("Y", m * ld);  // A Omega, A (A^T q)
    double* T = ctx->tbuf<double>("T", n * ld);  // Omega, A^T q
    double* Qb[2] = {ctx->tbuf<double>("QB0", m * ld), ctx->tbuf<double>("QB1", m * ld)};
    double* W = ctx->tbuf<double>("W", l * l);
    double* sv = ctx->tbuf<double>("s", l);
    double* inv_s = ctx->tbuf<double>("inv_s", l);
    double* s_stored = ctx->tbuf<double>("s_stored", l);
    Control* ctrl = ctx->tbuf<Control>("ctrl", 1);
    const int64_t cap = p > 0 ? p : 1;
    double* d_alphas = ctx->tbuf<double>("trace.alphas", cap);
    double* d_shat = ctx->tbuf<double>("trace.s_hat", cap * l);
    EigSvdOut eo{W, sv, inv_s};
    control_init(ctrl, s_stored, static_cast<int>(l), st);
    count_launch();
    if (qr) DSVD_CUDA_CHECK(cudaMemsetAsync(d_shat, 0, sizeof(double) * cap * l, st));  // no spectrum

    int sp = ctx->span_begin(K_OTHER);
    gaussian_rowmajor(T, n, l, ld, cfg.seed, st);  // gaussian_matrix(a.cols, l, seed)
    count_launch();
    ctx->span_end(sp);
    sp = ctx->span_begin(K_SPMM1);
    spmm(SpmmArgs{&A, T, Y, ld, l, nullptr, nullptr, nullptr}, st, spmm_var(ctx, ld), ctx->side, ctx->fork,
         ctx->join, partial_for(ctx, A, ld));
    count_launch();
    ctx->span_end(sp);
    // orth(y): eigSVD(y).u, or qr_orth(y) = CholeskyQR2 + Householder signs (qr.cu)
    auto orth = [&](const double* y, double* qout, const LoopStep* loop) {
        if (!qr) {
            eig_svd_factors(ctx, y, m, l, ld, eo, ctrl, loop, nullptr);
            const int s2 = ctx->span_begin(K_RESCALE);
            solve_rescale(ctx, y, m, l, ld, W, l, inv_s, l, qout, ld, 0, nullptr);
            ctx->span_end(s2);
            return;
        }
        double* G = ctx->tbuf<double>("qr.G", l * l);
        double* W1 = ctx->tbuf<double>("qr.W1", l * l);
        double* W2 = ctx->tbuf<double>("qr.W2", l * l);
        double* r1 = ctx->tbuf<double>("qr.r1", l);
        double* r2 = ctx->tbuf<double>("qr.r2", l);
        double* Q1 = ctx->tbuf<double>("qr.Q1", m * ld);
        double* Ptop = ctx->tbuf<double>("qr.Ptop", l * ld);
        auto gram_of = [&](const double* c) {
            const int s2 = ctx->span_begin(K_GRAM);
            if (gram_dmma_supported(l, ld)) {
                gram_dmma(c, m, l, ld, G, ctx->buf("gram.dws." + std::to_string(m), gram_dmma_workspace_bytes(m, l)),
                          nullptr, st);
            } else {
                const size_t gws = gram_workspace_bytes(m, l);
                gram(c, m, l, ld, G, ctx->buf("gram.ws." + std::to_string(m), gws), gws, nullptr, st);
            }
            count_launch(2);
            ctx->span_end(s2);
        };
        gram_of(y);
        chol_inv(G, static_cast<int>(l), W1, r1, ctrl, nullptr, st);
        count_launch();
        solve_rescale(ctx, y, m, l, ld, W1, l, nullptr, l, Q1, ld, 0, nullptr);  // Q1 = Y R1^{-1}
        gram_of(Q1);
        chol_inv(G, static_cast<int>(l), W2, r2, ctrl, nullptr, st);
        count_launch();
        solve_rescale(ctx, Q1, l, l, ld, W2, l, nullptr, l, Ptop, ld, 0, nullptr);  // top l rows of Q_pos
        qr_signs(Ptop, ld, static_cast<int>(l), W2, W1, r1, r2, m, ctrl, nullptr, st);  // W1 <- W2 diag(s)
        count_launch();
        solve_rescale(ctx, Q1, m, l, ld, W1, l, nullptr, l, qout, ld, 0, nullptr);  // Q = Q1 R2^{-1} diag(s)
        if (loop != nullptr) {  // the qr orthonormalizer has no spectrum: the trace records alpha = 0 only
            trace_basic_iteration(ctrl, loop->alphas, loop->cap, st);
            count_launch();
        }
    };
    orth(Y, Qb[0], nullptr);

    LoopStep ls;
    ls.k = k;
    ls.tol = cfg.tol;
    ls.alg = DSVD_ALG_BASIC;
    ls.alphas = d_alphas;
    ls.s_hat = d_shat;
    ls.cap = cap;
    ls.s_stored = s_stored;
    int cur = 0;
    for (int64_t j = 1; j <= p; ++j) {
        sp = ctx->span_begin(K_SPMM2);
        spmm(SpmmArgs{&AT, Qb[cur], T, ld, l, nullptr, nullptr, nullptr}, st, spmm_var(ctx, ld), ctx->side,
             ctx->fork, ctx->join, partial_for(ctx, AT, ld));
        count_launch();
        ctx->span_end(sp);
        sp = ctx->span_begin(K_SPMM1);
        spmm(SpmmArgs{&A, T, Y, ld, l, nullptr, nullptr, nullptr}, st, spmm_var(ctx, ld), ctx->side, ctx->fork,
             ctx->join, partial_for(ctx, A, ld));
        count_launch();
        ctx->span_end(sp);
        orth(Y, Qb[1 - cur], &ls);
        if (observer) {
            Control hc = read_control(ctx, ctrl);
            raise_device_status(hc);
            std::vector<double> qb = to_host_colmajor(ctx, Qb[cur], m, l, ld);
            std::vector<double> qa = to_host_colmajor(ctx, Qb[1 - cur], m, l, ld);
            std::vector<double> sh(static_cast<size_t>(l));
            DSVD_CUDA_CHECK(cudaMemcpy(sh.data(), d_shat + (j - 1) * l, sizeof(double) * l, cudaMemcpyDeviceToHost));
            observer(j, 0.0, sh.data(), l, qb.data(), qa.data(), m, user);
        }
        cur = 1 - cur;
    }
    Control hc = read_control(ctx, ctrl);
    raise_device_status(hc);
    io.iterations = p;
    io.stop_reason = DSVD_STOP_FIXED_P;
    ctx->stats.eig_sweeps = hc.total_sweeps;
    const double* Qf = Qb[cur];

    // finalize_col_basis: f = eigSVD(A^T q); U = q f.v[:, :k]; V = f.u[:, :k]
    control_init(ctrl, s_stored, static_cast<int>(l), st);
    count_launch();
    sp = ctx->span_begin(K_SPMM2);
    spmm(SpmmArgs{&AT, Qf, T, ld, l, nullptr, nullptr, nullptr}, st, spmm_var(ctx, ld), ctx->side, ctx->fork,
         ctx->join, partial_for(ctx, AT, ld));
    count_launch();
    ctx->span_end(sp);
    eig_svd_factors(ctx, T, n, l, ld, eo, ctrl, nullptr, nullptr);
    hc = read_control(ctx, ctrl);
    raise_device_status(hc);
    ctx->stats.eig_sweeps += hc.total_sweeps;
    double* du = io.on_device ? io.u : ctx->tbuf<double>("out.u", m * k);
    double* dv = io.on_device ? io.v : ctx->tbuf<double>("out.v", n * k);
    sp = ctx->span_begin(K_RESCALE);
    solve_rescale(ctx, Qf, m, l, ld, W, l, nullptr, k, du, 0, 1, nullptr);  // matmul(q, head_cols(f.v, k))
    solve_rescale(ctx, T, n, l, ld, W, l, inv_s, k, dv, 0, 1, nullptr);      // head_cols(f.u, k)
    ctx->span_end(sp);
    if (io.on_device) {
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.s, sv, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
    } else {
        copy_d2h(ctx, io.u, du, sizeof(double) * m * k, st);
        copy_d2h(ctx, io.v, dv, sizeof(double) * n * k, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.s, sv, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    }
    const int64_t nrec = std::min(io.iterations, io.cap);
    if (nrec > 0 && io.alphas)
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.alphas, d_alphas, sizeof(double) * nrec, cudaMemcpyDeviceToHost, st));
    if (nrec > 0 && io.s_hat)
        DSVD_CUDA_CHECK(cudaMemcpyAsync(io.s_hat, d_shat, sizeof(double) * nrec * l, cudaMemcpyDeviceToHost, st));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
}

}  // namespace

// Starts Omega for the solve of an m x n host matrix on the side stream, so it
// overlaps the CSR upload that follows on the main stream (single-GPU solves).
// d_off (optional): the device offsets of A's rows, ordered on ctx->stream; with the tall
// orientation the sketch rows of empty rows of A are then written as zeros, not drawn.
void pregenerate_omega(dsvd_ctx* ctx, int64_t rows, int64_t cols, const dsvd_config& cfg, const int64_t* d_off) {
    ctx->omega_pending = false;
    if (ctx->comm != nullptr || cfg.k < 1 || cfg.alg == DSVD_ALG_BASIC) return;
    const bool direct = (cfg.flags & DSVD_FLAG_DIRECT) != 0;
    const int64_t m = (rows < cols && !direct) ? cols : rows;  // the tall orientation (solve_pair)
    const int64_t l = cfg.k + effective_s(cfg);
    if (l > 512 || m < 1) return;
    const int64_t ld = padded_ld(l);
    const int lw = slab_layout_width(ctx, ld, std::max(rows, cols));  // as solve_tall
    double* Y = ctx->tbuf<double>("Y", block_doubles(m, ld, lw));
    if (!ctx->omega_ev) DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->omega_ev, cudaEventDisableTiming));
    DSVD_CUDA_CHECK(cudaEventRecord(ctx->fork, ctx->stream));  // earlier work on Y is done
    DSVD_CUDA_CHECK(cudaStreamWaitEvent(ctx->side, ctx->fork, 0));
    gaussian_rowmajor(Y, m, l, ld, cfg.seed, ctx->side, -1, 0, lw, m == rows ? d_off : nullptr);
    ctx->omega_slab_w = lw;
    count_launch();
    DSVD_CUDA_CHECK(cudaEventRecord(ctx->omega_ev, ctx->side));
    ctx->omega_pending = true;
    ctx->omega_m = m;
    ctx->omega_l = l;
    ctx->omega_seed = cfg.seed;
}

namespace {

void solve_pair(dsvd_ctx* ctx, const DevCsr& a, const DevCsr& at, const dsvd_config& cfg,
                dsvd_outputs* out, dsvd_observer_fn observer, void* user, int64_t row_offset = 0,
                int64_t global_rows = -1) {
    if (ctx->comm != nullptr) {
        // row-sharded solve: validate against the global shape
        const int64_t gm = global_rows >= 0 ? global_rows : a.rows;
        validate(cfg, gm, a.cols);
        if (cfg.alg == DSVD_ALG_BASIC)
            fail(DSVD_UNSUPPORTED, "the basic algorithm is not on the B200 path (shifted family only)");
        if (gm < a.cols) fail(DSVD_UNSUPPORTED, "row-sharded solves need rows >= cols");
        SolveIO io;
        io.on_device = out->outputs_on_device != 0;
        io.alphas = out->alphas;
        io.s_hat = out->s_hat;
        io.cap = out->trace_cap;
        io.u = out->u;
        io.v = out->v;
        io.s = out->s;
        solve_tall(ctx, a, at, cfg, io, observer, user, row_offset, gm);
        out->iterations = io.iterations;
        out->stop_reason = io.stop_reason;
        return;
    }
    validate(cfg, a.rows, a.cols);
    const int64_t l = cfg.k + effective_s(cfg);
    const bool direct = (cfg.flags & DSVD_FLAG_DIRECT) != 0;
    SolveIO io;
    io.on_device = out->outputs_on_device != 0;
    io.alphas = out->alphas;
    io.s_hat = out->s_hat;
    io.cap = out->trace_cap;
    // the shifted family on (X, XT): column-compacted when X has empty columns
    // (build_compact) — not with an observer (its Q snapshots are full n-row blocks)
    auto tall = [&](const DevCsr& X, const DevCsr& XT) {
        const int64_t nne = XT.nonempty_rows;
        if (ctx->compact_cols && observer == nullptr && nne >= l && nne < XT.rows &&
            (XT.rows - nne) * 50 >= XT.rows) {  // >= 2% of the columns empty
            const Compact c = build_compact(ctx, X, XT);
            io.v_rows = c.oldid;
            io.v_full = XT.rows;
            solve_tall(ctx, c.a, c.at, cfg, io, observer, user);
        } else {
            solve_tall(ctx, X, XT, cfg, io, observer, user);
        }
    };
    if (a.rows < a.cols && !direct) {
        // solve on the transpose and swap U/V (solver.cpp:217-220)
        io.u = out->v;
        io.v = out->u;
        io.s = out->s;
        if (cfg.alg == DSVD_ALG_BASIC) solve_basic(ctx, at, a, cfg, io, observer, user);
        else tall(at, a);
    } else {
        io.u = out->u;
        io.v = out->v;
        io.s = out->s;
        if (cfg.alg == DSVD_ALG_BASIC) solve_basic(ctx, a, at, cfg, io, observer, user);
        else tall(a, at);
    }
    out->iterations = io.iterations;
    out->stop_reason = io.stop_reason;
}

// Algorithmic SpMM bytes of one solve: per pass
// 12 nnz + 8 (rows+1) + 8 X + 8 Y (+ 8 Q for the shifted pass 2).
void account_spmm_bytes(dsvd_ctx* ctx, const DevCsr& a, const dsvd_config& cfg, int64_t iters) {
    const DevCsr* tall = &a;
    int64_t m = tall->rows, n = tall->cols;
    if (m < n) std::swap(m, n);
    const int64_t l = cfg.k + effective_s(cfg);
    const int64_t b1 = 12 * a.nnz + 8 * (m + 1) + 8 * n * l + 8 * m * l;
    const int64_t b2 = 12 * a.nnz + 8 * (n + 1) + 8 * m * l + 8 * n * l + 8 * n * l;
    const int64_t b2_first = 12 * a.nnz + 8 * (n + 1) + 8 * m * l + 8 * n * l;
    ctx->stats.spmm_pass_bytes[0] = b1 * (iters + 1);
    ctx->stats.spmm_pass_bytes[1] = b2 * iters + b2_first;
    ctx->stats.spmm_bytes = ctx->stats.spmm_pass_bytes[0] + ctx->stats.spmm_pass_bytes[1];
}

}  // namespace
}  // namespace dsvd

using namespace dsvd;

extern "C" {

const char* dsvd_last_error(void) { return t_err.c_str(); }
long long dsvd_last_error_index(void) { return t_err_index; }
const char* dsvd_version(void) { return "dashsvd-b200 0.1 (sm_100a)"; }

int dsvd_ctx_create(int device, dsvd_ctx** out) {
    return guarded([&] {
        int count = 0;
        DSVD_CUDA_CHECK(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(DSVD_CUDA, "no such CUDA device");
        std::unique_ptr<dsvd_ctx> c(new dsvd_ctx());
        c->device = device;
        DSVD_CUDA_CHECK(cudaSetDevice(device));
        DSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        DSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        int prio_lo = 0, prio_hi = 0;
        DSVD_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        DSVD_CUDA_CHECK(cudaStreamCreateWithPriority(&c->eig, cudaStreamNonBlocking, prio_hi));
        DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_t, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_eig, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        DSVD_CUDA_CHECK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        *out = c.release();
    });
}

int dsvd_ctx_destroy(dsvd_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->eig);
        for (auto& kv : ctx->arena)
            if (kv.second.ptr) cudaFree(kv.second.ptr);
        for (auto e : ctx->event_pool) cudaEventDestroy(e);
        if (ctx->timer[0]) {
            cudaEventDestroy(ctx->timer[0]);
            cudaEventDestroy(ctx->timer[1]);
        }
        if (ctx->host_flags) cudaFreeHost(ctx->host_flags);
        for (cudaEvent_t e : ctx->stage_ev)
            if (e) {
                cudaEventSynchronize(e);
                cudaEventDestroy(e);
            }
        if (ctx->stage) cudaFreeHost(ctx->stage);
        if (ctx->stage_ready) cudaEventDestroy(ctx->stage_ready);
        comm_release(ctx);
        cudaStreamDestroy(ctx->side);
        cudaStreamDestroy(ctx->eig);
        cudaEventDestroy(ctx->ev_t);
        cudaEventDestroy(ctx->ev_eig);
        cudaEventDestroy(ctx->fork);
        cudaEventDestroy(ctx->join);
        if (ctx->omega_ev) cudaEventDestroy(ctx->omega_ev);
        if (ctx->copy_ev) cudaEventDestroy(ctx->copy_ev);
        if (ctx->copy) cudaStreamDestroy(ctx->copy);
        if (ctx->comm_ev) cudaEventDestroy(ctx->comm_ev);
        if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
        if (ctx->landing) cudaFree(ctx->landing);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int dsvd_ctx_set_profiling(dsvd_ctx* ctx, int on) {
    return guarded([&] { ctx->profiling = on != 0; });
}

int dsvd_ctx_get_stats(const dsvd_ctx* ctx, dsvd_stats* out) {
    return guarded([&] { *out = ctx->stats; });
}

int dsvd_ctx_synchronize(dsvd_ctx* ctx) {
    return guarded([&] {
        set_device(ctx);
        DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int dsvd_ctx_trim(dsvd_ctx* ctx) {
    return guarded([&] {
        set_device(ctx);
        DSVD_CUDA_CHECK(cudaDeviceSynchronize());
        for (auto& kv : ctx->arena)
            if (kv.second.ptr) DSVD_CUDA_CHECK(cudaFree(kv.second.ptr));
        ctx->arena.clear();
        ctx->omega_pending = false;
        ctx->coo_rows = ctx->coo_cols = ctx->coo_nnz = -1;
    });
}

int dsvd_ctx_set_option(dsvd_ctx* ctx, const char* name, int64_t value) {
    return guarded([&] {
        const std::string n = name ? name : "";
        if (n == "spmm_variant") {
            ctx->spmm_variant = static_cast<int>(value);
        } else if (n == "spmm_slab") {
            if (value != -1 && value != 0 && value != 32 && value != 64)
                fail(DSVD_CONFIG, "spmm_slab: -1 (auto), 0 (whole rows), 32 or 64 columns");
            ctx->spmm_slab = static_cast<int>(value);
        } else if (n == "slab_layout") {
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "slab_layout must be 0 or 1");
            ctx->slab_layout = static_cast<int>(value);
        } else if (n == "gram_tiles") {
            if (value != 2 && value != 4) fail(DSVD_CONFIG, "gram_tiles must be 2 or 4");
            set_gram_wide_tiles(static_cast<int>(value));
        } else if (n == "spmm_short_rows") {
            if (value < 0 || value > 2) fail(DSVD_CONFIG, "spmm_short_rows: 0 off, 1 rows <= 8 nonzeros, 2 rows <= 32");
            set_spmm_short_rows(static_cast<int>(value));
        } else if (n == "gram_waves") {
            if (value < 1 || value > 64) fail(DSVD_CONFIG, "gram_waves must be in [1, 64]");
            set_gram_wide_waves(static_cast<int>(value));
        } else if (n == "rescale_row_ctas") {
            if (value < 1) fail(DSVD_CONFIG, "rescale_row_ctas must be >= 1");
            set_rescale_row_ctas(value);
        } else if (n == "uniform_values") {
            // 1: detect all-equal values at build time (the column-slab kernel then
            // skips the value stream), 0: always stream the values
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "uniform_values must be 0 or 1");
            ctx->uniform_values = static_cast<int>(value);
        } else if (n == "spmm_hot_mb") {
            if (value < 0) fail(DSVD_CONFIG, "spmm_hot_mb must be >= 0");
            ctx->spmm_hot_mb = value;
        } else if (n == "spmm_slab_depth") {
            if (value < 0 || value > 2) fail(DSVD_CONFIG, "spmm_slab_depth must be 0, 1 or 2");
            ctx->spmm_slab_depth = static_cast<int>(value);
        } else if (n == "spmm_slab_hint") {
            if (value < 0 || value > 2) fail(DSVD_CONFIG, "spmm_slab_hint: 0 off, 1 every launch, 2 A X pass only");
            ctx->spmm_slab_hint = static_cast<int>(value);
        } else if (n == "hub_threshold") {
            ctx->hub_threshold = value;
        } else if (n == "eig_method") {
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "eig_method: 0 = tridiagonal (auto), 1 = Jacobi");
            ctx->eig_method = static_cast<int>(value);
        } else if (n == "dense_method") {
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "dense_method: 0 = FP64 tensor cores, 1 = DFMA");
            ctx->dense_method = static_cast<int>(value);
        } else if (n == "pipeline") {
            if (value < -1 || value > 1)
                fail(DSVD_CONFIG, "pipeline: 1 = eig beside the A T pass, 0 = serial, -1 = auto");
            ctx->pipeline = static_cast<int>(value);
        } else if (n == "host_staging") {
            // 1 (default): pageable host buffers go through the pinned staging ring; 0: plain copies
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "host_staging must be 0 or 1");
            ctx->host_staging = static_cast<int>(value);
        } else if (n == "host_copy_threads") {
            if (value < 0 || value > 256) fail(DSVD_CONFIG, "host_copy_threads must be in [0, 256] (0: auto)");
            ctx->host_copy_threads = static_cast<int>(value);
        } else if (n == "host_stage_chunk") {
            // bytes per staging slot (4 slots)
            if (value < 4096 || value > (int64_t(1) << 30) || value % 4096)
                fail(DSVD_CONFIG, "host_stage_chunk must be a multiple of 4096 in [4 KB, 1 GB]");
            ctx->stage_chunk = value;
        } else if (n == "eig_priority") {
            // 1: the eig stream at the highest priority (default), 0: default priority
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "eig_priority must be 0 or 1");
            set_device(ctx);  // the new stream must belong to the context's device
            DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->eig));
            DSVD_CUDA_CHECK(cudaStreamDestroy(ctx->eig));
            int lo = 0, hi = 0;
            DSVD_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            DSVD_CUDA_CHECK(cudaStreamCreateWithPriority(&ctx->eig, cudaStreamNonBlocking, value ? hi : lo));
        } else if (n == "eig_overlap") {
            if (value < -1 || value > 2)
                fail(DSVD_CONFIG,
                     "eig_overlap: 2 = tridiagonalisation beside the A T pass, 1 = whole chain, 0 = none, -1 = auto");
            ctx->eig_overlap = static_cast<int>(value);
        } else if (n == "shift_after") {
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "shift_after must be 0 or 1");
            ctx->shift_after = static_cast<int>(value);
        } else if (n == "gram_async") {
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "gram_async: 1 = Gram on the eig stream too, 0 = main");
            ctx->gram_async = static_cast<int>(value);
        } else if (n == "split_chunk_t") {
            if (value < 0) fail(DSVD_CONFIG, "split_chunk_t must be >= 0");
            ctx->split_chunk_t = value;
        } else if (n == "split_panel_rows") {
            if (value < 0) fail(DSVD_CONFIG, "split_panel_rows must be >= 0");
            ctx->split_panel_rows = value;
        } else if (n == "pipeline_auto_nnz") {
            // the auto schedule's nnz bound (pipelined at or below it); 0 = the cost model
            if (value < 0) fail(DSVD_CONFIG, "pipeline_auto_nnz must be >= 0");
            ctx->pipeline_auto_nnz = value;
        } else if (n == "mgpu_mode") {
            if (value < 1 || value > 2) fail(DSVD_CONFIG, "mgpu_mode: 1 = all-reduce (v1), 2 = reduce-scatter (v2)");
            ctx->mgpu_mode = static_cast<int>(value);
        } else if (n == "compact_cols") {
            if (value < 0 || value > 1) fail(DSVD_CONFIG, "compact_cols must be 0 or 1");
            ctx->compact_cols = static_cast<int>(value);
        } else if (n == "mgpu_overlap") {
            if (value < 0 || value > 2)
                fail(DSVD_CONFIG, "mgpu_overlap: 0 whole-pass collective, 1 panelled reductions, 2 fused peer stores");
            ctx->mgpu_overlap = static_cast<int>(value);
        } else if (n == "split_chunk") {
            if (value < 0) fail(DSVD_CONFIG, "split_chunk must be >= 0");
            ctx->split_chunk = value;
        } else {
            fail(DSVD_CONFIG, "unknown option '" + n + "'");
        }
    });
}

int dsvd_host_register(void* ptr, size_t bytes) {
    return guarded([&] { DSVD_CUDA_CHECK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault)); });
}

int dsvd_host_unregister(void* ptr) {
    return guarded([&] { DSVD_CUDA_CHECK(cudaHostUnregister(ptr)); });
}

int dsvd_matrix_upload(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                       const int64_t* offsets, const int64_t* col_indices, const double* values,
                       dsvd_matrix** out) {
    return guarded([&] {
        set_device(ctx);
        std::unique_ptr<dsvd_matrix> m(new dsvd_matrix());
        m->ctx = ctx;
        m->device = ctx->device;
        CsrAlloc al{ctx, "", &m->owned};
        try {
            // upload_pair allocates a.off / a.val through `al` (owned)
            upload_pair(ctx, al, rows, cols, nnz, offsets, col_indices, values, m->a, m->at);
        } catch (...) {
            for (void* p : m->owned) cudaFree(p);
            throw;
        }
        *out = m.release();
    });
}

int dsvd_matrix_from_device(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                            const int64_t* d_offsets, const int64_t* d_col_indices,
                            const double* d_values, dsvd_matrix** out) {
    return guarded([&] {
        set_device(ctx);
        std::unique_ptr<dsvd_matrix> m(new dsvd_matrix());
        m->ctx = ctx;
        m->device = ctx->device;
        CsrAlloc al{ctx, "", &m->owned};
        try {
            build_pair(ctx, al, rows, cols, nnz, d_offsets, d_col_indices, d_values, m->a, m->at,
                       true);
        } catch (...) {
            for (void* p : m->owned) cudaFree(p);
            throw;
        }
        *out = m.release();
    });
}

int dsvd_matrix_destroy(dsvd_matrix* m) {
    return guarded([&] {
        if (!m) return;
        cudaSetDevice(m->device);
        cudaDeviceSynchronize();  // not the context's stream: the context may be destroyed already
        for (void* p : m->owned) cudaFree(p);
        delete m;
    });
}

int dsvd_matrix_set_shard(dsvd_matrix* m, int64_t row_offset, int64_t global_rows) {
    return guarded([&] {
        if (row_offset < 0 || global_rows < row_offset + m->a.rows)
            fail(DSVD_SHAPE, "shard rows exceed the global row count");
        m->row_offset = row_offset;
        m->global_rows = global_rows;
    });
}

int dsvd_matrix_shape(const dsvd_matrix* m, int64_t* rows, int64_t* cols, int64_t* nnz) {
    return guarded([&] {
        *rows = m->a.rows;
        *cols = m->a.cols;
        *nnz = m->a.nnz;
    });
}

int dsvd_matrix_bench_spmm(dsvd_matrix* m, int transpose, int64_t l, int variant, int iters,
                           double* ms_out) {
    return guarded([&] {
        dsvd_ctx* ctx = m->ctx;
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        const DevCsr& A = transpose ? m->at : m->a;
        const int64_t ld = padded_ld(l);
        double* X = ctx->tbuf<double>("bench.X", A.cols * ld);
        double* Y = ctx->tbuf<double>("bench.Y", A.rows * ld);
        gaussian_rowmajor(X, A.cols, l, ld, 1234, st);
        spmm(SpmmArgs{&A, X, Y, ld, l, nullptr, nullptr, nullptr}, st, variant, ctx->side, ctx->fork,
             ctx->join, partial_for(ctx, A, ld));
        cudaEvent_t e0 = ctx->event(), e1 = ctx->event();
        DSVD_CUDA_CHECK(cudaEventRecord(e0, st));
        for (int i = 0; i < iters; ++i)
            spmm(SpmmArgs{&A, X, Y, ld, l, nullptr, nullptr, nullptr}, st, variant, ctx->side,
                 ctx->fork, ctx->join, partial_for(ctx, A, ld));
        DSVD_CUDA_CHECK(cudaEventRecord(e1, st));
        DSVD_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.f;
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        *ms_out = ms / (iters > 0 ? iters : 1);
        ctx->event_next = 0;
    });
}

int dsvd_matrix_hub_rows(const dsvd_matrix* m, int64_t* hub_a, int64_t* hub_at) {
    return guarded([&] {
        *hub_a = m->a.hub_rows;
        *hub_at = m->at.hub_rows;
    });
}

namespace {
void download_csr(const dsvd_matrix* m, const DevCsr& c, int64_t* off, int64_t* idx, double* val) {
    dsvd_ctx* ctx = m->ctx;
    set_device(ctx);
    cudaStream_t st = ctx->stream;
    int64_t* w = ctx->tbuf<int64_t>("dl.idx64", c.nnz);
    widen_indices(c.idx, w, c.nnz, st);
    DSVD_CUDA_CHECK(cudaMemcpyAsync(off, c.off, sizeof(int64_t) * (c.rows + 1), cudaMemcpyDeviceToHost, st));
    if (c.nnz) {
        DSVD_CUDA_CHECK(cudaMemcpyAsync(idx, w, sizeof(int64_t) * c.nnz, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(val, c.val, sizeof(double) * c.nnz, cudaMemcpyDeviceToHost, st));
    }
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
}
}  // namespace

int dsvd_matrix_download_transpose(const dsvd_matrix* m, int64_t* t_off, int64_t* t_idx,
                                   double* t_val) {
    return guarded([&] { download_csr(m, m->at, t_off, t_idx, t_val); });
}

int dsvd_matrix_download(const dsvd_matrix* m, int64_t* off, int64_t* idx, double* val) {
    return guarded([&] { download_csr(m, m->a, off, idx, val); });
}

int dsvd_matrix_download_rows(const dsvd_matrix* m, int64_t r0, int64_t r1, int64_t* off, int64_t* idx,
                              double* val) {
    return guarded([&] {
        const DevCsr& c = m->a;
        if (r0 < 0 || r1 < r0 || r1 > c.rows) fail(DSVD_SHAPE, "download_rows: row range out of bounds");
        dsvd_ctx* ctx = m->ctx;
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        DSVD_CUDA_CHECK(cudaMemcpyAsync(off, c.off + r0, sizeof(int64_t) * (r1 - r0 + 1), cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
        const int64_t p0 = off[0], n = off[r1 - r0] - p0;
        for (int64_t i = 0; i <= r1 - r0; ++i) off[i] -= p0;
        if (n > 0) {
            int64_t* w = ctx->tbuf<int64_t>("dl.idx64", n);
            widen_indices(c.idx + p0, w, n, st);
            DSVD_CUDA_CHECK(cudaMemcpyAsync(idx, w, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
            DSVD_CUDA_CHECK(cudaMemcpyAsync(val, c.val + p0, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        }
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_matrix_row_offsets(const dsvd_matrix* m, int64_t* off) {
    return guarded([&] {
        set_device(m->ctx);
        DSVD_CUDA_CHECK(cudaMemcpy(off, m->a.off, sizeof(int64_t) * (m->a.rows + 1), cudaMemcpyDeviceToHost));
    });
}

int dsvd_solve(dsvd_ctx* ctx, const dsvd_matrix* a, const dsvd_config* cfg, dsvd_outputs* out,
               dsvd_observer_fn observer, void* user) {
    return guarded([&] {
        set_device(ctx);
        ctx->omega_pending = false;
        const int64_t l0 = g_launches.load();
        begin_profile(ctx);
        cudaEvent_t e0 = ctx->event(), e1 = ctx->event();
        DSVD_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        PrefaultScope pf{ctx};
        prefault_outputs(ctx, out, a->a.rows, a->a.cols, cfg->k);
        solve_pair(ctx, a->a, a->at, *cfg, out, observer, user, a->row_offset, a->global_rows);
        DSVD_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        DSVD_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.f;
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        end_profile(ctx, l0);
        ctx->stats.total_ms = ms;
        account_spmm_bytes(ctx, a->a, *cfg, out->iterations);
    });
}

int dsvd_solve_csr(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                   const int64_t* col_indices, const double* values, const dsvd_config* cfg,
                   dsvd_outputs* out) {
    return guarded([&] {
        set_device(ctx);
        if (ctx->comm == nullptr) validate(*cfg, rows, cols);
        const int64_t l0 = g_launches.load();
        begin_profile(ctx);
        cudaEvent_t e0 = ctx->event(), e1 = ctx->event(), e2 = ctx->event();
        DSVD_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        PrefaultScope pf{ctx};
        prefault_outputs(ctx, out, rows, cols, cfg->k);
        DevCsr a, at;
        CsrAlloc al{ctx, "csr.", nullptr};
        upload_pair(ctx, al, rows, cols, nnz, offsets, col_indices, values, a, at, cfg);
        DSVD_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        solve_pair(ctx, a, at, *cfg, out, nullptr, nullptr, ctx->shard_row_offset,
                   ctx->shard_global_rows);
        DSVD_CUDA_CHECK(cudaEventRecord(e2, ctx->stream));
        DSVD_CUDA_CHECK(cudaEventSynchronize(e2));
        float ms = 0.f, ms_up = 0.f;
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e2));
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms_up, e0, e1));
        end_profile(ctx, l0);
        ctx->stats.total_ms = ms;
        ctx->stats.csc_ms = ms_up;
        account_spmm_bytes(ctx, a, *cfg, out->iterations);
    });
}

int dsvd_solve_csr_device(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                          const int64_t* d_off, const int64_t* d_idx, const double* d_val,
                          const dsvd_config* cfg, dsvd_outputs* out) {
    return guarded([&] {
        set_device(ctx);
        ctx->omega_pending = false;
        if (ctx->comm == nullptr) validate(*cfg, rows, cols);
        const int64_t l0 = g_launches.load();
        begin_profile(ctx);
        cudaEvent_t e0 = ctx->event(), e1 = ctx->event(), e2 = ctx->event();
        DSVD_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
        DevCsr a, at;
        CsrAlloc al{ctx, "csr.", nullptr};
        pregenerate_omega(ctx, rows, cols, *cfg, d_off);  // Omega on the side stream beside the CSC build
        build_pair(ctx, al, rows, cols, nnz, d_off, d_idx, d_val, a, at, false);
        DSVD_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
        solve_pair(ctx, a, at, *cfg, out, nullptr, nullptr, ctx->shard_row_offset,
                   ctx->shard_global_rows);
        DSVD_CUDA_CHECK(cudaEventRecord(e2, ctx->stream));
        DSVD_CUDA_CHECK(cudaEventSynchronize(e2));
        float ms = 0.f, ms_up = 0.f;
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e2));
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms_up, e0, e1));
        end_profile(ctx, l0);
        ctx->stats.total_ms = ms;
        ctx->stats.csc_ms = ms_up;
        account_spmm_bytes(ctx, a, *cfg, out->iterations);
    });
}

int dsvd_ctx_set_shard(dsvd_ctx* ctx, int64_t row_offset, int64_t global_rows) {
    return guarded([&] {
        if (row_offset < 0) fail(DSVD_SHAPE, "negative shard offset");
        ctx->shard_row_offset = row_offset;
        ctx->shard_global_rows = global_rows;
    });
}

int dsvd_ctx_timer_start(dsvd_ctx* ctx) {
    return guarded([&] {
        set_device(ctx);
        if (!ctx->timer[0]) {
            DSVD_CUDA_CHECK(cudaEventCreate(&ctx->timer[0]));
            DSVD_CUDA_CHECK(cudaEventCreate(&ctx->timer[1]));
        }
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->timer[0], ctx->stream));
    });
}

int dsvd_ctx_timer_stop(dsvd_ctx* ctx, double* elapsed_ms) {
    return guarded([&] {
        set_device(ctx);
        if (!ctx->timer[0]) fail(DSVD_CONFIG, "timer not started");
        DSVD_CUDA_CHECK(cudaEventRecord(ctx->timer[1], ctx->stream));
        DSVD_CUDA_CHECK(cudaEventSynchronize(ctx->timer[1]));
        float ms = 0.f;
        DSVD_CUDA_CHECK(cudaEventElapsedTime(&ms, ctx->timer[0], ctx->timer[1]));
        *elapsed_ms = ms;
    });
}

int dsvd_finalize_row_basis(dsvd_ctx* ctx, const dsvd_matrix* a, const double* q, int64_t l,
                            int64_t k, double* u, double* s, double* v) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        const DevCsr& A = a->a;
        const int64_t m = A.rows, n = A.cols;
        if (k < 1 || k > l) fail(DSVD_SHAPE, "finalize_row_basis: k out of range");
        if (l > m) fail(DSVD_SHAPE, "eig_svd: needs rows >= cols (factor the transpose instead)");
        const int64_t ld = padded_ld(l);
        double* qh = ctx->tbuf<double>("fin.qcm", n * l);
        double* Q = ctx->tbuf<double>("fin.Q", n * ld);
        double* B = ctx->tbuf<double>("fin.B", m * ld);
        double* W = ctx->tbuf<double>("W", l * l);
        double* sv = ctx->tbuf<double>("s", l);
        double* inv_s = ctx->tbuf<double>("inv_s", l);
        double* s_stored = ctx->tbuf<double>("s_stored", l);
        Control* ctrl = ctx->tbuf<Control>("ctrl", 1);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(qh, q, sizeof(double) * n * l, cudaMemcpyHostToDevice, st));
        colmajor_to_rowmajor(qh, n, l, Q, ld, st);
        control_init(ctrl, s_stored, static_cast<int>(l), st);
        spmm(SpmmArgs{&A, Q, B, ld, l, nullptr, nullptr, nullptr}, st, spmm_var(ctx, ld), ctx->side,
             ctx->fork, ctx->join, partial_for(ctx, A, ld));
        EigSvdOut eo{W, sv, inv_s};
        eig_svd_factors(ctx, B, m, l, ld, eo, ctrl, nullptr, nullptr);
        raise_device_status(read_control(ctx, ctrl));
        double* du = ctx->tbuf<double>("out.u", m * k);
        double* dv = ctx->tbuf<double>("out.v", n * k);
        solve_rescale(ctx, B, m, l, ld, W, l, inv_s, k, du, 0, 1, nullptr);
        solve_rescale(ctx, Q, n, l, ld, W, l, nullptr, k, dv, 0, 1, nullptr);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(u, du, sizeof(double) * m * k, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(v, dv, sizeof(double) * n * k, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(s, sv, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_validate_config(const dsvd_config* cfg, int64_t rows, int64_t cols) {
    return guarded([&] { validate(*cfg, rows, cols); });
}

double dsvd_update_shift(double alpha, double s_ll) {
    return s_ll > alpha ? (s_ll + alpha) / 2.0 : alpha;
}

int dsvd_pve_stop_check(const double* prev, int64_t n_prev, double alpha_prev, const double* cur,
                        int64_t n, double alpha, int64_t k, double tol, int* stop) {
    return guarded([&] {
        if (k < 1) fail(DSVD_SHAPE, "pve_stop_check: k must be >= 1");
        if (n_prev < k + 1 || n < k + 1)
            fail(DSVD_SHAPE, "pve_stop_check: surrogate arrays must hold at least k+1 values");
        const double denom = cur[k] + alpha;
        *stop = 1;
        for (int64_t i = 0; i < k; ++i) {
            const double change = std::fabs(prev[i] + alpha_prev - cur[i] - alpha);
            if (!(change / denom <= tol)) {
                *stop = 0;
                return;
            }
        }
    });
}

uint64_t dsvd_splitmix64_at(uint64_t seed, uint64_t i) { return splitmix64_at(seed, i); }

// ---- kernel-level entry points ------------------------------------------------

int dsvd_spmm(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
              const int64_t* col_indices, const double* values, const double* x, int64_t l,
              double* y) {
    return dsvd_spmm_shift(ctx, rows, cols, nnz, offsets, col_indices, values, x, l, 0.0, nullptr, y);
}

int dsvd_spmm_shift(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                    const int64_t* col_indices, const double* values, const double* x, int64_t l,
                    double alpha, const double* q, double* y) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        if (l < 0) fail(DSVD_SHAPE, "spmm: negative width");
        DevCsr a, at;
        CsrAlloc al{ctx, "k.", nullptr};
        upload_pair(ctx, al, rows, cols, nnz, offsets, col_indices, values, a, at);
        if (l == 0 || rows == 0) return;
        const int64_t ld = padded_ld(l);
        double* xc = ctx->tbuf<double>("k.xcm", std::max(cols * l, rows * l));
        double* X = ctx->tbuf<double>("k.X", cols * ld);
        double* Yd = ctx->tbuf<double>("k.Y", rows * ld);
        double* Qd = nullptr;
        double* d_alpha = ctx->tbuf<double>("k.alpha", 1);
        if (cols > 0) {
            DSVD_CUDA_CHECK(cudaMemcpyAsync(xc, x, sizeof(double) * cols * l, cudaMemcpyHostToDevice, st));
            colmajor_to_rowmajor(xc, cols, l, X, ld, st);
        }
        if (q != nullptr) {
            Qd = ctx->tbuf<double>("k.Q", rows * ld);
            double* qc = ctx->tbuf<double>("k.qcm", rows * l);
            DSVD_CUDA_CHECK(cudaMemcpyAsync(qc, q, sizeof(double) * rows * l, cudaMemcpyHostToDevice, st));
            colmajor_to_rowmajor(qc, rows, l, Qd, ld, st);
            DSVD_CUDA_CHECK(cudaMemcpyAsync(d_alpha, &alpha, sizeof(double), cudaMemcpyHostToDevice, st));
        }
        spmm(SpmmArgs{&a, X, Yd, ld, l, Qd, Qd ? d_alpha : nullptr, nullptr}, st, spmm_var(ctx, ld), ctx->side, ctx->fork, ctx->join,
             partial_for(ctx, a, ld));
        rowmajor_to_colmajor(Yd, rows, l, ld, xc, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(y, xc, sizeof(double) * rows * l, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_transpose(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                   const int64_t* col_indices, const double* values, int64_t* t_off,
                   int64_t* t_idx, double* t_val) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        DevCsr a, at;
        CsrAlloc al{ctx, "k.", nullptr};
        upload_pair(ctx, al, rows, cols, nnz, offsets, col_indices, values, a, at);
        int64_t* w = ctx->tbuf<int64_t>("dl.idx64", nnz);
        widen_indices(at.idx, w, nnz, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(t_off, at.off, sizeof(int64_t) * (cols + 1), cudaMemcpyDeviceToHost, st));
        if (nnz) {
            DSVD_CUDA_CHECK(cudaMemcpyAsync(t_idx, w, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, st));
            DSVD_CUDA_CHECK(cudaMemcpyAsync(t_val, at.val, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st));
        }
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_gram(dsvd_ctx* ctx, int64_t rows, int64_t cols, const double* c, double* g) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        if (cols == 0) return;
        const int64_t ld = padded_ld(cols);
        double* cc = ctx->tbuf<double>("k.ccm", rows * cols);
        double* C = ctx->tbuf<double>("k.C", rows * ld);
        double* G = ctx->tbuf<double>("k.G", cols * cols);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(cc, c, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, st));
        colmajor_to_rowmajor(cc, rows, cols, C, ld, st);
        if (ctx->dense_method == 0 && gram_dmma_supported(cols, ld)) {
            gram_dmma(C, rows, cols, ld, G, ctx->buf("k.gdws", gram_dmma_workspace_bytes(rows, cols)), nullptr, st);
        } else {
            const size_t gws = gram_workspace_bytes(rows, cols);
            gram(C, rows, cols, ld, G, ctx->buf("k.gws", gws), gws, nullptr, st);
        }
        DSVD_CUDA_CHECK(cudaMemcpyAsync(g, G, sizeof(double) * cols * cols, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_sym_eig(dsvd_ctx* ctx, int64_t n, const double* g, double* values, double* vectors) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        if (n == 0) return;
        if (n > 512) fail(DSVD_UNSUPPORTED, "sym_eig: n > 512 is not supported");
        // symmetry check exactly as sym_eig.cpp:139-146
        double scale = 0.0, asym = 0.0;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                scale = std::max(scale, std::fabs(g[j * n + i]));
                asym = std::max(asym, std::fabs(g[j * n + i] - g[i * n + j]));
            }
        if (asym > 1e-10 * std::max(scale, 1e-300)) fail(DSVD_SHAPE, "sym_eig: matrix is not symmetric");
        double* G = ctx->tbuf<double>("k.G", n * n);
        // row-major copy of a column-major matrix: transpose on the host side of the copy
        std::vector<double> rm(static_cast<size_t>(n * n));
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) rm[i * n + j] = g[j * n + i];
        DSVD_CUDA_CHECK(cudaMemcpyAsync(G, rm.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, st));
        Control* ctrl = ctx->tbuf<Control>("ctrl", 1);
        double* s_stored = ctx->tbuf<double>("s_stored", n);
        control_init(ctrl, s_stored, static_cast<int>(n), st);
        EigWorkspace ew;
        eig_workspace_bind(ew, static_cast<int>(n), kMaxSweeps,
                           ctx->buf("eig.ws", eig_workspace_bytes(static_cast<int>(n), kMaxSweeps)));
        jacobi_eig(G, ew, ctrl, nullptr, st);
        double* dv = ctx->tbuf<double>("k.vals", n);
        double* dV = ctx->tbuf<double>("k.vecs", n * n);
        sym_eig_finish(ew, dv, dV, st);
        Control hc = read_control(ctx, ctrl);
        if (hc.status == DSVD_NUMERICAL) fail(DSVD_NUMERICAL, "symmetric Jacobi iteration did not converge");
        DSVD_CUDA_CHECK(cudaMemcpyAsync(values, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(vectors, dV, sizeof(double) * n * n, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_eig_svd(dsvd_ctx* ctx, int64_t rows, int64_t cols, const double* c, double* u, double* s,
                 double* v) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        if (rows < cols) fail(DSVD_SHAPE, "eig_svd: needs rows >= cols (factor the transpose instead)");
        if (cols == 0) return;
        if (cols > 512) fail(DSVD_UNSUPPORTED, "eig_svd: cols > 512 is not supported");
        const int64_t l = cols, ld = padded_ld(cols);
        double* cc = ctx->tbuf<double>("k.ccm", rows * l);
        double* C = ctx->tbuf<double>("k.C", rows * ld);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(cc, c, sizeof(double) * rows * l, cudaMemcpyHostToDevice, st));
        colmajor_to_rowmajor(cc, rows, l, C, ld, st);
        double* W = ctx->tbuf<double>("W", l * l);
        double* sv = ctx->tbuf<double>("s", l);
        double* inv_s = ctx->tbuf<double>("inv_s", l);
        double* s_stored = ctx->tbuf<double>("s_stored", l);
        Control* ctrl = ctx->tbuf<Control>("ctrl", 1);
        control_init(ctrl, s_stored, static_cast<int>(l), st);
        EigSvdOut eo{W, sv, inv_s};
        eig_svd_factors(ctx, C, rows, l, ld, eo, ctrl, nullptr, nullptr);
        raise_device_status(read_control(ctx, ctrl));
        rescale(C, rows, l, ld, W, l, inv_s, l, cc, 0, 1, nullptr, st);
        double* vcm = ctx->tbuf<double>("k.vcm", l * l);
        rowmajor_to_colmajor(W, l, l, l, vcm, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(u, cc, sizeof(double) * rows * l, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(s, sv, sizeof(double) * l, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(v, vcm, sizeof(double) * l * l, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_matmul(dsvd_ctx* ctx, int64_t m, int64_t kk, int64_t n, const double* a, const double* b,
                double* c) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        if (m == 0 || n == 0) return;
        const int64_t lda = padded_ld(kk), ldb = padded_ld(n);
        double* ac = ctx->tbuf<double>("k.acm", std::max(m * kk, m * n));
        double* A = ctx->tbuf<double>("k.A", m * lda);
        double* bc = ctx->tbuf<double>("k.bcm", kk * n);
        double* B = ctx->tbuf<double>("k.B", kk * ldb);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(ac, a, sizeof(double) * m * kk, cudaMemcpyHostToDevice, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(bc, b, sizeof(double) * kk * n, cudaMemcpyHostToDevice, st));
        colmajor_to_rowmajor(ac, m, kk, A, lda, st);
        colmajor_to_rowmajor(bc, kk, n, B, ldb, st);
        rescale(A, m, kk, lda, B, ldb, nullptr, n, ac, 0, 1, nullptr, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(c, ac, sizeof(double) * m * n, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int dsvd_gaussian_matrix(dsvd_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return dsvd_gaussian_rows(ctx, rows, cols, seed, rows, 0, out);
}

int dsvd_gaussian_rows(dsvd_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, int64_t global_rows,
                       int64_t row_offset, double* out) {
    return guarded([&] {
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        if (rows < 0 || cols < 0 || row_offset < 0 || global_rows < row_offset + rows)
            fail(DSVD_SHAPE, "gaussian rows exceed the global row count");
        if (rows * cols == 0) return;
        const int64_t ld = padded_ld(cols);
        double* R = ctx->tbuf<double>("k.omega", rows * ld);
        double* Cm = ctx->tbuf<double>("k.omegacm", rows * cols);
        gaussian_rowmajor(R, rows, cols, ld, seed, st, global_rows, row_offset);
        rowmajor_to_colmajor(R, rows, cols, ld, Cm, st);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(out, Cm, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
