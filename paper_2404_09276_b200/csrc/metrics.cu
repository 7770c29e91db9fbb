// Validation metrics at scale (metrics.cpp:99-206) on the
// device: eps_pve, eps_res, eps_spec and max_triplet_residual from the
// SpMM kernels of the solve plus deterministic column reductions (per-block
// partial sums added in block order). The reference's sums are sequential;
// these are fixed trees, so values agree to rounding, not bitwise.
#include <cmath>
#include <vector>

#include "dense.cuh"
#include "engine.cuh"
#include "sparse.cuh"

namespace dsvd {

namespace {

constexpr int kRedBlocks = 296;  // partial-sum blocks (2 per SM)

// partial[b][j] = sum over the block's rows of (x(r, j) - s_j z(r, j))^2  (z may be null)
//   or, with wv != null, sum of x(r, j) * wv(r) (a transposed GEMV)
__global__ void __launch_bounds__(256)
col_partial_kernel(const double* __restrict__ x, int64_t ldx, const double* __restrict__ z, int64_t ldz,
                   const double* __restrict__ s, const double* __restrict__ wv, int64_t ldw, int64_t rows, int k,
                   double* __restrict__ partial) {
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const double sj = (z != nullptr) ? s[j] : 0.0;
        double acc = 0.0;
        for (int64_t r = r0; r < r1; ++r) {
            if (wv != nullptr) {
                acc = fma(x[r * ldx + j], wv[r * ldw], acc);
            } else {
                const double d = z != nullptr ? fma(-sj, z[r * ldz + j], x[r * ldx + j]) : x[r * ldx + j];
                acc = fma(d, d, acc);
            }
        }
        partial[static_cast<int64_t>(blockIdx.x) * k + j] = acc;
    }
}

// out[j] = sum_b partial[b][j] (block order); mode 1: sqrt; mode 2: times s[j]
__global__ void col_reduce_kernel(const double* __restrict__ partial, int nb, int k, const double* __restrict__ s,
                                  int mode, double* __restrict__ out) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int b = 0; b < nb; ++b) acc += partial[static_cast<int64_t>(b) * k + j];
        out[j] = mode == 1 ? sqrt(acc) : (mode == 2 ? acc * s[j] : acc);
    }
}

// y(r) -= sum_j u(r, j) coef[j]   (vectors stored with stride ldy)
__global__ void lowrank_sub_kernel(const double* __restrict__ u, int64_t ldu, const double* __restrict__ coef,
                                   int k, double* __restrict__ y, int64_t ldy, int64_t rows) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < k; ++j) acc = fma(u[r * ldu + j], coef[j], acc);
        y[r * ldy] -= acc;
    }
}

// v = z / *nrm unless *nrm == 0 (then *zero = 1: the estimate is 0)
__global__ void scale_vec_kernel(const double* __restrict__ z, int64_t ldz, const double* __restrict__ nrm,
                                 double* __restrict__ v, int64_t ldv, int64_t rows, int32_t* __restrict__ zero) {
    const double n = *nrm;
    if (n == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *zero = 1;
        return;
    }
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[r * ldv] = z[r * ldz] / n;
}

int grid_rows(int64_t rows) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 256), 4 * kNumSMs))); }

}  // namespace

// Column norms ||x(:, j) - s_j z(:, j)|| (z may be null) of a row-major block.
void col_norms(dsvd_ctx* ctx, const double* x, int64_t ldx, const double* z, int64_t ldz, const double* s,
               int64_t rows, int k, double* out) {
    cudaStream_t st = ctx->stream;
    double* partial = ctx->tbuf<double>("met.partial", static_cast<size_t>(kRedBlocks) * k);
    col_partial_kernel<<<kRedBlocks, 256, 0, st>>>(x, ldx, z, ldz, s, nullptr, 0, rows, k, partial);
    DSVD_LAUNCH_CHECK();
    col_reduce_kernel<<<static_cast<unsigned>(ceil_div(k, 256)), 256, 0, st>>>(partial, kRedBlocks, k, nullptr, 1,
                                                                              out);
    DSVD_LAUNCH_CHECK();
}

// coef[j] = s_j * sum_r w(r, j) v(r)   (v with stride ldv)
void lowrank_coef(dsvd_ctx* ctx, const double* w, int64_t ldw, const double* s, const double* v, int64_t ldv,
                  int64_t rows, int k, double* coef) {
    cudaStream_t st = ctx->stream;
    double* partial = ctx->tbuf<double>("met.partial2", static_cast<size_t>(kRedBlocks) * k);
    col_partial_kernel<<<kRedBlocks, 256, 0, st>>>(w, ldw, nullptr, 0, nullptr, v, ldv, rows, k, partial);
    DSVD_LAUNCH_CHECK();
    col_reduce_kernel<<<static_cast<unsigned>(ceil_div(k, 256)), 256, 0, st>>>(partial, kRedBlocks, k, s, 2, coef);
    DSVD_LAUNCH_CHECK();
}

void lowrank_sub(dsvd_ctx* ctx, const double* u, int64_t ldu, const double* coef, int k, double* y, int64_t ldy,
                 int64_t rows) {
    lowrank_sub_kernel<<<grid_rows(rows), 256, 0, ctx->stream>>>(u, ldu, coef, k, y, ldy, rows);
    DSVD_LAUNCH_CHECK();
}

void scale_vec(dsvd_ctx* ctx, const double* z, int64_t ldz, const double* nrm, double* v, int64_t ldv,
               int64_t rows, int32_t* zero) {
    scale_vec_kernel<<<grid_rows(rows), 256, 0, ctx->stream>>>(z, ldz, nrm, v, ldv, rows, zero);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
