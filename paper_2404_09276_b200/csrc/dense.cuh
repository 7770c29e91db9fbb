// Dense tall-skinny kernels: Gaussian sketch, Gram reduction, rescale GEMM,
// layout conversions.
#pragma once

#include "common.cuh"

namespace dsvd {

// Omega(i, j) = normal_at(seed, j*rows + i) (random.cpp:29-36), written
// row-major with stride ld; columns [l, ld) are zero.
// For a row shard, rows [row_offset, row_offset + rows) of the global
// global_rows x l sketch are generated (global_rows < 0 means rows).
// slab_w > 0: written slab-major instead (sparse.cuh slab_index, width slab_w).
// row_off (optional, device CSR offsets of the matrix these rows belong to):
// rows without nonzeros are written as 0.0 instead of drawn (never gathered).
void gaussian_rowmajor(double* out, int64_t rows, int64_t l, int64_t ld, uint64_t seed,
                       cudaStream_t stream, int64_t global_rows = -1, int64_t row_offset = 0, int slab_w = 0,
                       const int64_t* row_off = nullptr);

// t = fma(-alpha, q, t) elementwise unless *alpha == 0 (add_scaled,
// dense_kernels.cpp:128-136, as applied at solver.cpp:94). Used after the
// multi-GPU partial sum, where the shift cannot ride the SpMM epilogue.
void shift_update(double* t, const double* q, int64_t count, const double* alpha,
                  const int32_t* gate, cudaStream_t stream);

// G = C^T C for row-major C (n x l, stride ld): split-K partial 64x64 tiles
// over the upper triangle, then a fixed-order reduction across row chunks and
// an exact mirror (dense_kernels.cpp:91-108 makes G exactly symmetric too).
// G is l x l (row-major == column-major, it is symmetric).
size_t gram_workspace_bytes(int64_t n, int64_t l);
void gram(const double* c, int64_t n, int64_t l, int64_t ld, double* g, void* ws,
          size_t ws_bytes, const int32_t* gate, cudaStream_t stream);

// out(r, j) = (sum_t c(r, t) * w(t, j)) * scale[j] for j < ncol, the sum one
// FMA chain over t ascending from 0.0 (the matmul order of
// dense_kernels.cpp:34-53, scale as scale_columns :118-126).
//   c: row-major n x K (stride ldc); w: row-major K x ldw; scale may be null.
//   out_colmajor == 0: row-major with stride ld_out, columns [ncol, ld_out) zeroed.
//   out_colmajor != 0: column-major n x ncol.
void rescale(const double* c, int64_t n, int64_t K, int64_t ldc, const double* w, int64_t ldw,
             const double* scale, int64_t ncol, double* out, int64_t ld_out, int out_colmajor,
             const int32_t* gate, cudaStream_t stream);

// FP64 tensor-core versions used inside the solve (dmma.cu): same contracts as
// gram / rescale (rescale's scale folded into W), summation order not the
// reference's FMA chain. Workspace from the *_workspace_bytes functions.
bool gram_dmma_supported(int64_t l, int64_t ld);
// tile shape of the wide (l > 160) DMMA Gram: 2 (2x2 blocks of 8x8, default) or 4
// (4x4); process-wide, for A/B runs (option "gram_tiles")
void set_gram_wide_tiles(int t);
void set_gram_wide_waves(int w);
void set_rescale_row_ctas(int64_t c);  // grid.y cap of the DMMA rescale (option "rescale_row_ctas")  // CTAs per SM of the wide Gram grid (option "gram_waves")
size_t gram_dmma_workspace_bytes(int64_t n, int64_t l);
void gram_dmma(const double* c, int64_t n, int64_t l, int64_t ld, double* g, void* ws, const int32_t* gate,
               cudaStream_t stream);
bool rescale_dmma_supported(int64_t K, int64_t ldc, int64_t ld_out, int out_colmajor);
size_t rescale_dmma_workspace_bytes(int64_t K, int64_t width);
// Extra row-major destinations of the rescale (the fused all-gather of a
// row-sharded solve: the same rows stored into the other ranks' blocks over
// peer memory); n == 0: none.
constexpr int kMaxPeerOut = 8;
struct PeerOut {
    double* p[kMaxPeerOut];
    int n;
};
void rescale_dmma(const double* c, int64_t n, int64_t K, int64_t ldc, const double* w, int64_t ldw,
                  const double* scale, int64_t ncol, double* out, int64_t ld_out, int out_colmajor, void* ws,
                  const int32_t* gate, cudaStream_t stream, double* out2 = nullptr, int out2_w = 0,
                  const PeerOut* peers = nullptr);

// Column-major (rows x cols) <-> row-major (stride ld, pad columns zeroed).
void colmajor_to_rowmajor(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ld,
                          cudaStream_t stream);
void rowmajor_to_colmajor(const double* src, int64_t rows, int64_t cols, int64_t ld, double* dst,
                          cudaStream_t stream);

}  // namespace dsvd
