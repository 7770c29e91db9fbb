// Small l x l kernels of the device QR orthonormalizer (qr.cu).
#pragma once

#include "common.cuh"

namespace dsvd {

// smem bytes of the one-CTA l x l kernels below (l <= 160)
size_t qr_small_smem_bytes(int l);

// G = R^T R (upper R); w = R^{-1} (row-major, upper), rdiag = diag(R). A
// non-positive pivot k raises RankDeficient(k) in ctrl.
void chol_inv(const double* g, int l, double* w, double* rdiag, Control* ctrl, const int32_t* gate,
              cudaStream_t stream);

// Householder reconstruction signs of the top l x l block `a` (stride lda) of
// the positive-diagonal Q; w2s = w2 diag(s); rank floor on r1 .* r2 with
// max(rows, l) * eps.
void qr_signs(const double* a, int64_t lda, int l, const double* w2, double* w2s, const double* r1,
              const double* r2, int64_t rows, Control* ctrl, const int32_t* gate, cudaStream_t stream);

}  // namespace dsvd
