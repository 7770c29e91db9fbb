// C ABI of the validation metrics (metrics.cpp:99-206) on the device matrix.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "dense.cuh"
#include "engine_internal.cuh"

namespace dsvd {  // metrics.cu
void col_norms(dsvd_ctx* ctx, const double* x, int64_t ldx, const double* z, int64_t ldz, const double* s,
               int64_t rows, int k, double* out);
void lowrank_coef(dsvd_ctx* ctx, const double* w, int64_t ldw, const double* s, const double* v, int64_t ldv,
                  int64_t rows, int k, double* coef);
void lowrank_sub(dsvd_ctx* ctx, const double* u, int64_t ldu, const double* coef, int k, double* y, int64_t ldy,
                 int64_t rows);
void scale_vec(dsvd_ctx* ctx, const double* z, int64_t ldz, const double* nrm, double* v, int64_t ldv,
               int64_t rows, int32_t* zero);
}  // namespace dsvd

using namespace dsvd;

extern "C" {

// ---- validation metrics (metrics.cpp:99-206) ----------------------------------------

namespace {
// Host column-major (rows x k) -> device row-major, stride ld.
double* upload_block(dsvd_ctx* ctx, const std::string& tag, const double* h, int64_t rows, int64_t k,
                     int64_t ld) {
    double* cm = ctx->tbuf<double>(tag + ".cm", rows * k);
    double* rm = ctx->tbuf<double>(tag, rows * ld);
    DSVD_CUDA_CHECK(cudaMemcpyAsync(cm, h, sizeof(double) * rows * k, cudaMemcpyHostToDevice, ctx->stream));
    colmajor_to_rowmajor(cm, rows, k, rm, ld, ctx->stream);
    return rm;
}
void mspmm(dsvd_ctx* ctx, const DevCsr& A, const double* x, double* y, int64_t ld, int64_t l) {
    spmm(SpmmArgs{&A, x, y, ld, l, nullptr, nullptr, nullptr}, ctx->stream, spmm_var(ctx, ld), ctx->side,
         ctx->fork, ctx->join, partial_for(ctx, A, ld));
}
std::vector<double> col_norms_host(dsvd_ctx* ctx, const double* x, int64_t ldx, const double* z, int64_t ldz,
                                   const double* s_dev, int64_t rows, int64_t k) {
    double* d = ctx->tbuf<double>("met.norms", k);
    col_norms(ctx, x, ldx, z, ldz, s_dev, rows, static_cast<int>(k), d);
    std::vector<double> h(static_cast<size_t>(k));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(h.data(), d, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return h;
}
void require_sigmas(int64_t n_ref, int64_t count) {
    if (n_ref < count)
        fail(DSVD_DEGENERATE, "reference provides " + std::to_string(n_ref) + " singular values, need " +
                                  std::to_string(count));
}
}  // namespace

int dsvd_eps_pve(dsvd_ctx* ctx, const dsvd_matrix* m, const double* u, int64_t k, const double* sigmas,
                 int64_t n_ref, double* out) {
    return guarded([&] {
        set_device(ctx);
        if (k < 1) fail(DSVD_SHAPE, "eps_pve: U has no columns");
        require_sigmas(n_ref, k + 1);
        const double denom = sigmas[k] * sigmas[k];
        if (denom == 0.0) fail(DSVD_DEGENERATE, "sigma_{k+1} is zero");
        const DevCsr& A = m->a;
        const int64_t ld = padded_ld(k);
        double* U = upload_block(ctx, "met.U", u, A.rows, k, ld);
        double* W = ctx->tbuf<double>("met.W", A.cols * ld);
        mspmm(ctx, m->at, U, W, ld, k);  // A^T u_i
        const std::vector<double> q = col_norms_host(ctx, W, ld, nullptr, 0, nullptr, A.cols, k);
        double worst = 0.0;
        for (int64_t i = 0; i < k; ++i) worst = std::max(worst, std::abs(sigmas[i] * sigmas[i] - q[i] * q[i]) / denom);
        *out = worst;
    });
}

int dsvd_eps_res(dsvd_ctx* ctx, const dsvd_matrix* m, const double* u, const double* s, const double* v, int64_t k,
                 const double* sigmas, int64_t n_ref, double* out) {
    return guarded([&] {
        set_device(ctx);
        if (k < 1) fail(DSVD_SHAPE, "eps_res: no triplets");
        require_sigmas(n_ref, k);
        const DevCsr& A = m->a;
        const int64_t ld = padded_ld(k);
        double* U = upload_block(ctx, "met.U", u, A.rows, k, ld);
        double* V = upload_block(ctx, "met.V", v, A.cols, k, ld);
        double* sd = ctx->tbuf<double>("met.s", k);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(sd, s, sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
        double* W = ctx->tbuf<double>("met.W", A.cols * ld);
        mspmm(ctx, m->at, U, W, ld, k);
        const std::vector<double> r = col_norms_host(ctx, W, ld, V, ld, sd, A.cols, k);  // ||A^T u_i - s_i v_i||
        double worst = 0.0;
        for (int64_t i = 0; i < k; ++i) {
            if (sigmas[i] == 0.0) fail(DSVD_DEGENERATE, "sigma_i is zero");
            worst = std::max(worst, r[i] / sigmas[i]);
        }
        *out = worst;
    });
}

int dsvd_max_triplet_residual(dsvd_ctx* ctx, const dsvd_matrix* m, const double* u, const double* s, const double* v,
                              int64_t k, double* out) {
    return guarded([&] {
        set_device(ctx);
        const DevCsr& A = m->a;
        if (k < 1) {
            *out = 0.0;
            return;
        }
        const int64_t ld = padded_ld(k);
        double* U = upload_block(ctx, "met.U", u, A.rows, k, ld);
        double* V = upload_block(ctx, "met.V", v, A.cols, k, ld);
        double* sd = ctx->tbuf<double>("met.s", k);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(sd, s, sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
        double* AV = ctx->tbuf<double>("met.AV", A.rows * ld);
        mspmm(ctx, A, V, AV, ld, k);
        const std::vector<double> r = col_norms_host(ctx, AV, ld, U, ld, sd, A.rows, k);  // ||A v_i - s_i u_i||
        double worst = 0.0;
        for (int64_t i = 0; i < k; ++i) worst = std::max(worst, r[i]);
        *out = worst;
    });
}

int dsvd_eps_spec(dsvd_ctx* ctx, const dsvd_matrix* m, const double* u, const double* s, const double* v, int64_t k,
                  const double* sigmas, int64_t n_ref, int64_t power_iters, uint64_t seed, double* out) {
    return guarded([&] {
        set_device(ctx);
        if (k < 1) fail(DSVD_SHAPE, "eps_spec: no triplets");
        require_sigmas(n_ref, k + 1);
        const double sk1 = sigmas[k];
        if (sk1 == 0.0) fail(DSVD_DEGENERATE, "sigma_{k+1} is zero");
        cudaStream_t st = ctx->stream;
        const DevCsr& A = m->a;
        const int64_t rows = A.rows, cols = A.cols;
        const int64_t ld = padded_ld(k), lv = padded_ld(1);  // vectors as rows x 4 blocks (column 0)
        double* U = upload_block(ctx, "met.U", u, rows, k, ld);
        double* V = upload_block(ctx, "met.V", v, cols, k, ld);
        double* sd = ctx->tbuf<double>("met.s", k);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(sd, s, sizeof(double) * k, cudaMemcpyHostToDevice, st));
        double* vv = ctx->tbuf<double>("met.v", cols * lv);
        double* zz = ctx->tbuf<double>("met.z", cols * lv);
        double* ww = ctx->tbuf<double>("met.w", rows * lv);
        double* coef = ctx->tbuf<double>("met.coef", k);
        double* nrm = ctx->tbuf<double>("met.nrm", 1);
        int32_t* zero = ctx->tbuf<int32_t>("met.zero", 1);
        DSVD_CUDA_CHECK(cudaMemsetAsync(zero, 0, sizeof(int32_t), st));
        DSVD_CUDA_CHECK(cudaMemsetAsync(zz, 0, sizeof(double) * cols * lv, st));
        gaussian_rowmajor(zz, cols, 1, lv, seed, st);  // gaussian_matrix(op.cols, 1, seed)
        col_norms(ctx, zz, lv, nullptr, 0, nullptr, cols, 1, nrm);
        DSVD_CUDA_CHECK(cudaMemsetAsync(vv, 0, sizeof(double) * cols * lv, st));
        scale_vec(ctx, zz, lv, nrm, vv, lv, cols, zero);
        // op(x) = A x - U diag(s) V^T x ; op^T(y) = A^T y - V diag(s) U^T y (metrics.cpp:146-153)
        auto apply = [&]() {
            mspmm(ctx, A, vv, ww, lv, 1);
            lowrank_coef(ctx, V, ld, sd, vv, lv, cols, static_cast<int>(k), coef);
            lowrank_sub(ctx, U, ld, coef, static_cast<int>(k), ww, lv, rows);
        };
        for (int64_t it = 0; it < power_iters; ++it) {
            apply();
            mspmm(ctx, m->at, ww, zz, lv, 1);
            lowrank_coef(ctx, U, ld, sd, ww, lv, rows, static_cast<int>(k), coef);
            lowrank_sub(ctx, V, ld, coef, static_cast<int>(k), zz, lv, cols);
            col_norms(ctx, zz, lv, nullptr, 0, nullptr, cols, 1, nrm);
            scale_vec(ctx, zz, lv, nrm, vv, lv, cols, zero);  // v = z / ||z|| (0 -> estimate 0)
        }
        apply();
        double hn = 0.0;
        int32_t hz = 0;
        col_norms(ctx, ww, lv, nullptr, 0, nullptr, rows, 1, nrm);
        DSVD_CUDA_CHECK(cudaMemcpyAsync(&hn, nrm, sizeof(double), cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaMemcpyAsync(&hz, zero, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        DSVD_CUDA_CHECK(cudaStreamSynchronize(st));
        const double norm = hz ? 0.0 : hn;
        *out = (norm - sk1) / sk1;
    });
}

}  // extern "C"
