// The QR orthonormalizer of the basic algorithm (qr_orth,
// decompositions.cpp:77-126) on sm_100a: CholeskyQR2 (two rounds of Gram ->
// Cholesky -> triangular inverse -> GEMM, the tensor-core Gram and rescale of
// dmma.cu), then the column signs of the Householder factorization recovered
// by Householder reconstruction (a sign-choosing LU of the top l x l block of
// Q, Ballard et al.): Q = Q_pos diag(s), s_k = sign(R_hh(k, k)), so Q matches
// the reference's Householder Q (beta = -sign(alpha) ||x||) column for column.
// The rank check is the reference's: |R(k, k)| <= max(m, n) eps max |R(j, j)|
// raises RankDeficient(k); a Cholesky breakdown at pivot k (numerically
// dependent column) raises it too.
#include "qr.cuh"

namespace dsvd {

namespace {

constexpr int kQrThreads = 512;

__device__ __forceinline__ void raise_rank(Control* ctrl, int k) {
    if (ctrl->status == DSVD_OK) {
        ctrl->status = DSVD_RANK_DEFICIENT;
        ctrl->status_index = k;
        ctrl->status_src = 1;
    }
}

// G (l x l, symmetric) = R^T R (R upper, positive diagonal); W = R^{-1} (upper,
// row-major l x l), rdiag = diag(R). One CTA. Shared layout M (l x (l+1)):
// upper triangle R, strictly lower triangle W^T.
__global__ void __launch_bounds__(kQrThreads, 1)
chol_inv_kernel(const double* __restrict__ g, int l, double* __restrict__ w, double* __restrict__ rdiag,
                Control* ctrl, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ double qsm[];
    const int ldm = l + 1;
    double* M = qsm;
    double* wdiag = M + l * ldm;
    __shared__ int s_fail;
    const int tid = threadIdx.x;
    for (int x = tid; x < l * l; x += blockDim.x) M[(x / l) * ldm + x % l] = g[x];
    if (tid == 0) s_fail = -1;
    __syncthreads();
    // right-looking Cholesky on the upper triangle
    for (int k = 0; k < l; ++k) {
        const double piv = M[k * ldm + k];
        if (!(piv > 0.0)) {  // numerically dependent column k
            if (tid == 0) s_fail = k;
            break;  // uniform: every thread read the same pivot
        }
        const double r = sqrt(piv), ir = 1.0 / r;
        __syncthreads();
        if (tid == 0) M[k * ldm + k] = r;
        for (int j = k + 1 + tid; j < l; j += blockDim.x) M[k * ldm + j] *= ir;
        __syncthreads();
        const int rem = l - k - 1;  // trailing upper triangle, row-major pairs (i <= j)
        for (int x = tid; x < rem * rem; x += blockDim.x) {
            const int i = k + 1 + x / rem, j = k + 1 + x % rem;
            if (j >= i) M[i * ldm + j] -= M[k * ldm + i] * M[k * ldm + j];
        }
        __syncthreads();
    }
    __syncthreads();
    if (s_fail >= 0) {
        if (tid == 0) raise_rank(ctrl, s_fail);
        for (int x = tid; x < l * l; x += blockDim.x) w[x] = 0.0;
        for (int i = tid; i < l; i += blockDim.x) rdiag[i] = 0.0;
        return;
    }
    // W = R^{-1}, rows bottom-up: W(i, j) = -(sum_{t=i+1..j} R(i, t) W(t, j)) / R(i, i)
    for (int i = tid; i < l; i += blockDim.x) wdiag[i] = 1.0 / M[i * ldm + i];
    __syncthreads();
    for (int i = l - 2; i >= 0; --i) {
        for (int j = i + 1 + tid; j < l; j += blockDim.x) {
            double acc = M[i * ldm + j] * wdiag[j];
            for (int t = i + 1; t < j; ++t) acc = fma(M[i * ldm + t], M[j * ldm + t], acc);
            M[j * ldm + i] = -acc * wdiag[i];  // W(i, j), stored transposed
        }
        __syncthreads();
    }
    for (int x = tid; x < l * l; x += blockDim.x) {
        const int i = x / l, j = x % l;
        w[x] = i == j ? wdiag[i] : (j > i ? M[j * ldm + i] : 0.0);
    }
    for (int i = tid; i < l; i += blockDim.x) rdiag[i] = M[i * ldm + i];
}

// a = the top l x l block of Q_pos (row-major, stride lda). Householder
// reconstruction: s_k = -sign(a_kk) (a_kk >= 0 -> -1, the reference's beta rule),
// a_kk -= s_k, then an unpivoted LU step. Writes w2s = w2 diag(s) and applies
// the rank floor to |R(k, k)| = r1_k r2_k.
__global__ void __launch_bounds__(kQrThreads, 1)
qr_signs_kernel(const double* __restrict__ a, int64_t lda, int l, const double* __restrict__ w2,
                double* __restrict__ w2s, const double* __restrict__ r1, const double* __restrict__ r2,
                int64_t rows, Control* ctrl, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ double qsm[];
    const int ldm = l + 1;
    double* A = qsm;
    double* sg = A + l * ldm;
    const int tid = threadIdx.x;
    for (int x = tid; x < l * l; x += blockDim.x) A[(x / l) * ldm + x % l] = a[(x / l) * lda + x % l];
    __syncthreads();
    for (int k = 0; k < l; ++k) {
        const double akk = A[k * ldm + k];
        const double s = akk >= 0.0 ? -1.0 : 1.0;
        const double piv = akk - s;
        __syncthreads();
        if (tid == 0) {
            sg[k] = s;
            A[k * ldm + k] = piv;
        }
        const double ip = 1.0 / piv;
        for (int i = k + 1 + tid; i < l; i += blockDim.x) A[i * ldm + k] *= ip;
        __syncthreads();
        const int rem = l - k - 1;
        for (int x = tid; x < rem * rem; x += blockDim.x) {
            const int i = k + 1 + x / rem, j = k + 1 + x % rem;
            A[i * ldm + j] -= A[i * ldm + k] * A[k * ldm + j];
        }
        __syncthreads();
    }
    for (int x = tid; x < l * l; x += blockDim.x) w2s[x] = w2[x] * sg[x % l];
    if (tid == 0) {
        double mx = 0.0;
        for (int k = 0; k < l; ++k) mx = fmax(mx, fabs(r1[k] * r2[k]));
        const double floor_ = static_cast<double>(rows > l ? rows : l) * 2.220446049250313e-16 * mx;
        for (int k = 0; k < l; ++k)
            if (fabs(r1[k] * r2[k]) <= floor_) {
                raise_rank(ctrl, k);
                break;
            }
    }
}

}  // namespace

size_t qr_small_smem_bytes(int l) { return sizeof(double) * (static_cast<size_t>(l) * (l + 1) + l); }

void chol_inv(const double* g, int l, double* w, double* rdiag, Control* ctrl, const int32_t* gate,
              cudaStream_t stream) {
    const size_t smem = qr_small_smem_bytes(l);
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    chol_inv_kernel<<<1, kQrThreads, smem, stream>>>(g, l, w, rdiag, ctrl, gate);
    DSVD_LAUNCH_CHECK();
}

void qr_signs(const double* a, int64_t lda, int l, const double* w2, double* w2s, const double* r1,
              const double* r2, int64_t rows, Control* ctrl, const int32_t* gate, cudaStream_t stream) {
    const size_t smem = qr_small_smem_bytes(l);
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(qr_signs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    qr_signs_kernel<<<1, kQrThreads, smem, stream>>>(a, lda, l, w2, w2s, r1, r2, rows, ctrl, gate);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
