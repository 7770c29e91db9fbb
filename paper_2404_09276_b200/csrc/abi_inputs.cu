// C ABI of the input side: device CSR validation, the DSH1
// cache, COO / Matrix Market assembly, dense-array and spectrum files, the
// R-MAT generator (see include/dashsvd_b200.h for the reference mapping).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "engine_internal.cuh"
#include "ingest.cuh"
#include "mtx.hpp"
#include "rng.cuh"

using namespace dsvd;

extern "C" {

// ---- inputs: validation, DSH1 cache, COO assembly ------------------------------------

namespace {
// Device validation of a CSR already in HBM, raising the reference's error.
void validate_device_csr(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_off,
                         const int64_t* d_idx, const double* d_val) {
    if (rows < 0 || cols < 0) fail(DSVD_SHAPE, "sparse matrix with negative dimension");
    int64_t fb[2] = {0, 0};
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&fb[0], d_off, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&fb[1], d_off + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    unsigned long long* first = ctx->tbuf<unsigned long long>("val.first", 1);
    csr_validate(d_off, d_idx, d_val, rows, cols, nnz, first, ctx->stream);
    unsigned long long hf = ~0ull;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&hf, first, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (fb[0] != 0 || fb[1] != nnz) fail(DSVD_SHAPE, "offsets must span [0, nnz]");
    if (hf == ~0ull) return;
    const int64_t row = static_cast<int64_t>(hf >> 3);
    const std::string r = std::to_string(row);
    switch (static_cast<int>(hf & 7)) {
        case 0: fail(DSVD_SHAPE, "offsets must be non-decreasing");
        case 1: fail(DSVD_SHAPE, "column index out of range in row " + r);
        case 2: fail(DSVD_SHAPE, "column indices not strictly increasing in row " + r);
        case 3: fail(DSVD_NUMERICAL, "non-finite value in row " + r);
        default: fail(DSVD_NUMERICAL, "explicit zero stored in row " + r);
    }
}
}  // namespace

int dsvd_csr_validate(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                      const int64_t* col_indices, const double* values) {
    return guarded([&] {
        set_device(ctx);
        if (rows < 0 || cols < 0 || nnz < 0) fail(DSVD_SHAPE, "sparse matrix with negative dimension");
        int64_t* off = ctx->tbuf<int64_t>("val.off", rows + 1);
        int64_t* idx = ctx->tbuf<int64_t>("val.idx", nnz);
        double* val = ctx->tbuf<double>("val.val", nnz);
        cudaStream_t st = ctx->stream;
        DSVD_CUDA_CHECK(cudaMemcpyAsync(off, offsets, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice, st));
        if (nnz) {
            DSVD_CUDA_CHECK(cudaMemcpyAsync(idx, col_indices, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
            DSVD_CUDA_CHECK(cudaMemcpyAsync(val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
        }
        validate_device_csr(ctx, rows, cols, nnz, off, idx, val);
    });
}

namespace {
constexpr char kDsh1[4] = {'D', 'S', 'H', '1'};
}

int dsvd_save_cache(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                    const int64_t* col_indices, const double* values) {
    return guarded([&] {
        std::FILE* f = std::fopen(path, "wb");
        if (!f) fail(DSVD_OTHER, std::string("cannot open ") + path + " for writing");
        const uint64_t dims[3] = {static_cast<uint64_t>(rows), static_cast<uint64_t>(cols),
                                  static_cast<uint64_t>(nnz)};
        bool ok = std::fwrite(kDsh1, 1, 4, f) == 4 && std::fwrite(dims, 8, 3, f) == 3 &&
                  std::fwrite(offsets, 8, static_cast<size_t>(rows + 1), f) == static_cast<size_t>(rows + 1) &&
                  std::fwrite(col_indices, 8, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz) &&
                  std::fwrite(values, 8, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz);
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) fail(DSVD_OTHER, std::string("failed writing ") + path);
    });
}

int dsvd_matrix_load_cache(dsvd_ctx* ctx, const char* path, int validate, dsvd_matrix** out, int64_t* dims_out) {
    return guarded([&] {
        set_device(ctx);
        std::FILE* f = std::fopen(path, "rb");
        if (!f) fail(DSVD_OTHER, std::string("cannot open ") + path);
        struct Closer {
            std::FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{f};
        char magic[4];
        uint64_t dims[3];
        if (std::fread(magic, 1, 4, f) != 4) fail(DSVD_FORMAT, "truncated cache file");
        if (std::memcmp(magic, kDsh1, 4) != 0) fail(DSVD_FORMAT, "not a DSH1 cache file");
        if (std::fread(dims, 8, 3, f) != 3) fail(DSVD_FORMAT, "truncated cache file");
        const int64_t rows = static_cast<int64_t>(dims[0]), cols = static_cast<int64_t>(dims[1]),
                      nnz = static_cast<int64_t>(dims[2]);
        // one pinned staging buffer: offsets | indices | values, read then uploaded;
        // a header promising more than the file holds is a truncated file
        const long here = std::ftell(f);
        std::fseek(f, 0, SEEK_END);
        const uint64_t avail = static_cast<uint64_t>(std::ftell(f) - here);
        std::fseek(f, here, SEEK_SET);
        if (dims[0] >= avail / 8 || dims[2] > avail / 16 || 8 * (dims[0] + 1 + 2 * dims[2]) > avail)
            fail(DSVD_FORMAT, "truncated cache file");
        const size_t bytes = sizeof(int64_t) * (static_cast<size_t>(rows) + 1 + 2 * static_cast<size_t>(nnz));
        void* host = nullptr;
        DSVD_CUDA_CHECK(cudaHostAlloc(&host, bytes, cudaHostAllocDefault));
        struct Freer {
            void* p;
            ~Freer() { cudaFreeHost(p); }
        } freer{host};
        if (std::fread(host, 1, bytes, f) != bytes) fail(DSVD_FORMAT, "truncated cache file");
        const int64_t* off = static_cast<const int64_t*>(host);
        const int64_t* idx = off + rows + 1;
        const double* val = reinterpret_cast<const double*>(idx + nnz);
        std::unique_ptr<dsvd_matrix> m(new dsvd_matrix());
        m->ctx = ctx;
        m->device = ctx->device;
        CsrAlloc al{ctx, "", &m->owned};
        try {
            if (validate) {
                // a.validate() (matrix_market.cpp:274) on the device, before the pair is built
                int64_t* d_off = ctx->tbuf<int64_t>("val.off", rows + 1);
                int64_t* d_idx = ctx->tbuf<int64_t>("val.idx", nnz);
                double* d_val = ctx->tbuf<double>("val.val", nnz);
                cudaStream_t st = ctx->stream;
                DSVD_CUDA_CHECK(cudaMemcpyAsync(d_off, off, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice, st));
                if (nnz) {
                    DSVD_CUDA_CHECK(cudaMemcpyAsync(d_idx, idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
                    DSVD_CUDA_CHECK(cudaMemcpyAsync(d_val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
                }
                validate_device_csr(ctx, rows, cols, nnz, d_off, d_idx, d_val);
                build_pair(ctx, al, rows, cols, nnz, d_off, d_idx, d_val, m->a, m->at, true);
            } else {
                upload_pair(ctx, al, rows, cols, nnz, off, idx, val, m->a, m->at);
                DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // the staging buffer dies here
            }
        } catch (...) {
            for (void* p : m->owned) cudaFree(p);
            throw;
        }
        if (dims_out) {
            dims_out[0] = rows;
            dims_out[1] = cols;
            dims_out[2] = nnz;
        }
        *out = m.release();
    });
}

namespace {
// assemble() (matrix_market.cpp:90-115) of host triplets into the context's
// COO result buffers (dsvd_coo_fetch / dsvd_matrix_from_coo read them).
int64_t assemble_host_triplets(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* r,
                               const int64_t* c, const double* v) {
    if (rows < 0 || cols < 0 || n < 0) fail(DSVD_SHAPE, "sparse matrix with negative dimension");
    if (n > 0x7fffffffLL) fail(DSVD_UNSUPPORTED, "more than 2^31 - 1 triplets per assembly");
    cudaStream_t st = ctx->stream;
    int64_t* dr = ctx->tbuf<int64_t>("coo.r", n);
    int64_t* dc = ctx->tbuf<int64_t>("coo.c", n);
    double* dv = ctx->tbuf<double>("coo.v", n);
    if (n) {
        DSVD_CUDA_CHECK(cudaMemcpyAsync(dr, r, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(dc, c, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(dv, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    }
    int64_t* off = ctx->tbuf<int64_t>("coo.off", rows + 1);
    int64_t* idx = ctx->tbuf<int64_t>("coo.idx", n);
    double* val = ctx->tbuf<double>("coo.val", n);
    int32_t* bad = ctx->tbuf<int32_t>("coo.bad", 1);
    ctx->coo_rows = ctx->coo_cols = ctx->coo_nnz = -1;
    const int64_t nnz =
        coo_assemble(dr, dc, dv, n, rows, cols, ctx->buf("coo.scratch", coo_scratch_bytes(n)), off, idx, val, bad, st);
    int32_t hb = 0;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&hb, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    if (hb) fail(DSVD_SHAPE, "coordinate out of range");
    ctx->coo_rows = rows;
    ctx->coo_cols = cols;
    ctx->coo_nnz = nnz;
    return nnz;
}

void require_coo(dsvd_ctx* ctx) {
    if (ctx->coo_rows < 0) fail(DSVD_CONFIG, "no assembled matrix in this context");
}
}  // namespace

int dsvd_coo_assemble(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* r, const int64_t* c,
                      const double* v, int64_t* nnz_out) {
    return guarded([&] {
        set_device(ctx);
        *nnz_out = assemble_host_triplets(ctx, rows, cols, n, r, c, v);
    });
}

int dsvd_mtx_assemble(dsvd_ctx* ctx, const char* path, int64_t* dims) {
    return guarded([&] {
        set_device(ctx);
        MtxTriplets t;
        const MtxStatus stt = mtx_read(path, t);
        if (stt.code != DSVD_OK) fail(stt.code, stt.what, stt.code == DSVD_PARSE ? stt.line : -1);
        const int64_t nnz = assemble_host_triplets(ctx, t.rows, t.cols, static_cast<int64_t>(t.v.size()), t.r.data(),
                                                   t.c.data(), t.v.data());
        dims[0] = t.rows;
        dims[1] = t.cols;
        dims[2] = nnz;
    });
}

namespace {
thread_local MtxTriplets t_mtx;  // dsvd_mtx_read -> dsvd_mtx_fetch
}

int dsvd_mtx_read(const char* path, int64_t* dims) {
    return guarded([&] {
        t_mtx = MtxTriplets{};
        const MtxStatus stt = mtx_read(path, t_mtx);
        if (stt.code != DSVD_OK) fail(stt.code, stt.what, stt.code == DSVD_PARSE ? stt.line : -1);
        dims[0] = t_mtx.rows;
        dims[1] = t_mtx.cols;
        dims[2] = static_cast<int64_t>(t_mtx.v.size());
    });
}

int dsvd_mtx_fetch(int64_t* r, int64_t* c, double* v) {
    return guarded([&] {
        std::copy(t_mtx.r.begin(), t_mtx.r.end(), r);
        std::copy(t_mtx.c.begin(), t_mtx.c.end(), c);
        std::copy(t_mtx.v.begin(), t_mtx.v.end(), v);
        t_mtx = MtxTriplets{};
    });
}

namespace {
thread_local DenseArray t_dense;          // dsvd_dense_read -> dsvd_dense_fetch
thread_local std::vector<double> t_spec;  // dsvd_spectrum_read -> dsvd_spectrum_fetch
void raise_mtx(const MtxStatus& stt) {
    if (stt.code != DSVD_OK) fail(stt.code, stt.what, stt.code == DSVD_PARSE ? stt.line : -1);
}
}  // namespace

int dsvd_dense_read(const char* path, int64_t* dims) {
    return guarded([&] {
        t_dense = DenseArray{};
        raise_mtx(dense_read(path, t_dense));
        dims[0] = t_dense.rows;
        dims[1] = t_dense.cols;
    });
}

int dsvd_dense_fetch(double* colmajor) {
    return guarded([&] {
        std::copy(t_dense.data.begin(), t_dense.data.end(), colmajor);
        t_dense = DenseArray{};
    });
}

int dsvd_dense_write(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
    return guarded([&] { raise_mtx(dense_write(path, rows, cols, colmajor)); });
}

int dsvd_spectrum_read(const char* path, int64_t* n) {
    return guarded([&] {
        t_spec.clear();
        raise_mtx(spectrum_read(path, t_spec));
        *n = static_cast<int64_t>(t_spec.size());
    });
}

int dsvd_spectrum_fetch(double* sigmas) {
    return guarded([&] {
        std::copy(t_spec.begin(), t_spec.end(), sigmas);
        t_spec.clear();
    });
}

int dsvd_spectrum_write(const char* path, const double* sigmas, int64_t n) {
    return guarded([&] { raise_mtx(spectrum_write(path, sigmas, n)); });
}

int dsvd_matrix_from_coo(dsvd_ctx* ctx, dsvd_matrix** out) {
    return guarded([&] {
        set_device(ctx);
        require_coo(ctx);
        std::unique_ptr<dsvd_matrix> m(new dsvd_matrix());
        m->ctx = ctx;
        m->device = ctx->device;
        CsrAlloc al{ctx, "", &m->owned};
        try {
            build_pair(ctx, al, ctx->coo_rows, ctx->coo_cols, ctx->coo_nnz, ctx->tbuf<int64_t>("coo.off", 1),
                       ctx->tbuf<int64_t>("coo.idx", 1), ctx->tbuf<double>("coo.val", 1), m->a, m->at, true);
            DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            for (void* p : m->owned) cudaFree(p);
            throw;
        }
        *out = m.release();
    });
}

int dsvd_synth_rmat(dsvd_ctx* ctx, int scale, int64_t draws, double a, double b, double c, int value_mode,
                    uint64_t seed, dsvd_matrix** out, int64_t* nnz_out) {
    return guarded([&] {
        set_device(ctx);
        if (scale < 1 || scale > 30) fail(DSVD_SHAPE, "rmat: scale must be in [1, 30]");
        if (draws < 0 || draws > 0x7fffffffLL) fail(DSVD_SHAPE, "rmat: draws must be in [0, 2^31)");
        if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) fail(DSVD_CONFIG, "rmat: need a, b, c >= 0, a+b+c <= 1");
        if (value_mode != 0 && value_mode != 1) fail(DSVD_CONFIG, "rmat: value_mode 0 (ones) or 1 (uniform (0,1])");
        RmatParams P;
        P.scale = scale;
        P.draws = draws;
        P.t_a = static_cast<uint32_t>(std::llround(a * 65536.0));
        P.t_ab = static_cast<uint32_t>(std::llround((a + b) * 65536.0));
        P.t_abc = static_cast<uint32_t>(std::llround((a + b + c) * 65536.0));
        P.value_mode = value_mode;
        P.edge_seed = splitmix64_at(seed, 0);
        P.val_seed = splitmix64_at(seed, 1);
        const int64_t n = int64_t(1) << scale;
        int64_t* off = ctx->tbuf<int64_t>("rmat.off", n + 1);
        int64_t* idx = ctx->tbuf<int64_t>("upload.idx64", draws);
        double* val = ctx->tbuf<double>("rmat.val", draws);
        const int64_t nnz = rmat_generate(P, ctx->buf("rmat.scratch", rmat_scratch_bytes(draws)), off, idx, val,
                                          ctx->stream);
        ctx->release("rmat.scratch");
        std::unique_ptr<dsvd_matrix> m(new dsvd_matrix());
        m->ctx = ctx;
        m->device = ctx->device;
        CsrAlloc al{ctx, "", &m->owned};
        try {
            build_pair(ctx, al, n, n, nnz, off, idx, val, m->a, m->at, true);
            DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            for (void* p : m->owned) cudaFree(p);
            throw;
        }
        ctx->release("rmat.off");
        ctx->release("rmat.val");
        *nnz_out = nnz;
        *out = m.release();
    });
}

int dsvd_write_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* offsets,
                             const int64_t* col_indices, const double* values) {
    return guarded([&] {
        const MtxStatus stt = mtx_write(path, rows, cols, offsets, col_indices, values);
        if (stt.code != DSVD_OK) fail(stt.code, stt.what);
    });
}

int dsvd_coo_fetch(dsvd_ctx* ctx, int64_t* offsets, int64_t* col_indices, double* values) {
    return guarded([&] {
        set_device(ctx);
        require_coo(ctx);
        const int64_t rows = ctx->coo_rows, nnz = ctx->coo_nnz;
        cudaStream_t st = ctx->stream;
        DSVD_CUDA_CHECK(cudaMemcpyAsync(offsets, ctx->tbuf<int64_t>("coo.off", rows + 1), sizeof(int64_t) * (rows + 1),
                                        cudaMemcpyDeviceToHost, st));
        if (nnz) {
            DSVD_CUDA_CHECK(cudaMemcpyAsync(col_indices, ctx->tbuf<int64_t>("coo.idx", 1), sizeof(int64_t) * nnz,
                                            cudaMemcpyDeviceToHost, st));
            DSVD_CUDA_CHECK(cudaMemcpyAsync(values, ctx->tbuf<double>("coo.val", 1), sizeof(double) * nnz,
                                            cudaMemcpyDeviceToHost, st));
        }
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
