// Tridiagonal eigensolver path for eigSVD's l x l Gram matrix on sm_100a:
//
//   1. tbi_tridiag_kernel  — Householder reduction A = Q T Q^T on one SM (the
//      reference's first stage, sym_eig.cpp:19-74, parallelised per step:
//      warp reductions for the norm, warp-per-row for p = tau A v, a
//      symmetric rank-2 update of the lower triangle in shared memory).
//   2. tbi_eig_kernel      — one warp per eigenvalue: 33-way multisection on
//      Sturm counts (each lane evaluates one point) to full precision, then
//      inverse iteration with a partially pivoted tridiagonal LU (lane 0).
//   3. tbi_orth_kernel     — two Newton-Schulz polar steps Z <- Z (3I - Z^T Z)/2
//      make the eigenvectors orthonormal to working precision.
//   4. tbi_backtransform_kernel — V = H_0 ... H_{n-3} Z, one warp per column, on
//      all SMs.
//
// The reference's implicit QL (sym_eig.cpp:78-130) is a serial bulge chase;
// bisection + inverse iteration exposes one independent task per eigenvalue
// instead. Inverse iteration needs separated eigenvalues, so tbi_eig_kernel
// raises a flag when two eigenvalues are closer than kTbiGap (relative to
// ||T||); the caller then runs the Jacobi solver instead (its kernels are
// launched gated on that flag), so clustered or repeated spectra keep full
// accuracy. Accuracy class on separated spectra: absolute eigenvalue error
// ~ n eps ||A||, the same as the reference's QL.
#include <cfloat>

#include "eig.cuh"

namespace dsvd {

namespace {

constexpr int kTbiThreads = 1024;
constexpr double kTbiGap = 1e-9;  // minimum relative eigenvalue gap for inverse iteration

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


// Copy a row-major n x n matrix from global (stride ldg) into shared memory
// (stride lds), 8 independent loads in flight per thread.
__device__ __forceinline__ void load_square(double* __restrict__ dst, int lds, const double* __restrict__ src,
                                            int ldg, int n) {
    const int total = n * n;
    for (int base = threadIdx.x; base < total; base += 8 * blockDim.x) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int x = base + u * blockDim.x;
            v[u] = x < total ? src[static_cast<int64_t>(x / n) * ldg + x % n] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int x = base + u * blockDim.x;
            if (x < total) dst[(x / n) * lds + x % n] = v[u];
        }
    }
}

// ---- 1. Householder tridiagonalisation ---------------------------------------
// A (n x n, symmetric) in shared memory, lower triangle authoritative, stride
// lda = n | 1. Outputs d (n), e (n-1), reflectors hv[k*n + i] (i > k) and tau[k].
__global__ void __launch_bounds__(kTbiThreads, 1)
tbi_tridiag_kernel(const double* __restrict__ g, int n, double* __restrict__ d, double* __restrict__ e,
                   double* __restrict__ hv, double* __restrict__ tau_out, const int32_t* __restrict__ gate,
                   const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double tsm[];
    const int lda = n | 1;
    double* A = tsm;                 // n x lda
    double* v = A + n * lda;         // n
    double* w = v + n;               // n
    __shared__ double s_tau, s_K;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    load_square(A, lda, g, n, n);
    __syncthreads();
    auto L = [&](int i, int j) -> double& { return i >= j ? A[i * lda + j] : A[j * lda + i]; };
    // four threads per row for the O(m^2) parts: row = tid / 4, quarter q = tid % 4
    const int rq = tid & 3, rgrp = tid >> 2, ngrp = blockDim.x >> 2;
    for (int k = 0; k + 2 < n; ++k) {
        const int k1 = k + 1, m = n - k1;
        if (warp == 0) {
            double sig = 0.0;
            for (int i = k1 + lane; i < n; i += 32) {
                const double x = L(i, k);
                sig = fma(x, x, sig);
            }
            sig = warp_sum(sig);
            const double x0 = L(k1, k);
            double alpha = 0.0, tau = 0.0, v0 = x0;
            const double tail = sig - x0 * x0;  // sum of squares below the first entry
            if (tail > 0.0) {
                alpha = -copysign(sqrt(sig), x0);
                v0 = x0 - alpha;
                tau = 2.0 / (tail + v0 * v0);
            } else {
                alpha = x0;  // already tridiagonal in this column
            }
            for (int i = k1 + lane; i < n; i += 32) {
                const double vi = (i == k1) ? v0 : L(i, k);
                v[i] = vi;
                hv[static_cast<int64_t>(k) * n + i] = vi;
            }
            if (lane == 0) {
                s_tau = tau;
                tau_out[k] = tau;
                e[k] = alpha;
                d[k] = L(k, k);
            }
        }
        __syncthreads();
        const double tau = s_tau;
        if (tau != 0.0) {
            // p = tau * A22 v: four threads per row (n <= 160 < 256 groups), each a
            // quarter of the columns; every lane reaches the shuffles
            {
                const int i = k1 + rgrp;
                double acc = 0.0;
                if (i < n) {
                    const double* row = A + i * lda;
                    for (int j = k1 + rq; j <= i; j += 4) acc = fma(row[j], v[j], acc);
                    for (int j = i + 1 + ((rq - (i + 1 - k1)) & 3); j < n; j += 4)
                        acc = fma(A[j * lda + i], v[j], acc);
                }
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                if (i < n && rq == 0) w[i] = tau * acc;
            }
            __syncthreads();
            if (warp == 0) {
                double acc = 0.0;
                for (int i = k1 + lane; i < n; i += 32) acc = fma(w[i], v[i], acc);
                acc = warp_sum(acc);
                if (lane == 0) s_K = 0.5 * tau * acc;
            }
            __syncthreads();
            const double K = s_K;
            for (int i = k1 + tid; i < n; i += blockDim.x) w[i] = fma(-K, v[i], w[i]);
            __syncthreads();
            // A22 -= v w^T + w v^T on the lower triangle, four threads per row
            for (int i = k1 + rgrp; i < n; i += ngrp) {
                const double vi = v[i], wi = w[i];
                double* row = A + i * lda;
                for (int j = k1 + rq; j <= i; j += 4) row[j] = row[j] - vi * w[j] - wi * v[j];
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = L(n - 2, n - 2);
            e[n - 2] = L(n - 1, n - 2);
        }
        d[n - 1] = L(n - 1, n - 1);
    }
}

// ---- 2. eigenvalues (multisection) and eigenvectors (inverse iteration) ----------------
__device__ __forceinline__ double rcp_fast(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    return r * fma(-q, r, 2.0);  // one Newton step: ~2^-56; counts only need signs
}

__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - x) - e2[i - 1] * rcp_fast(q);
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

constexpr int kTbiWarps = 8;

__global__ void __launch_bounds__(32 * kTbiWarps)
tbi_eig_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
               double* __restrict__ lam, double* __restrict__ z, int ldz, int32_t* __restrict__ clustered,
               const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double esm[];
    double* d = esm;                       // n
    double* e = d + n;                     // n
    double* e2 = e + n;                    // n
    double* work = e2 + n;                 // kTbiWarps x 6n (per-warp LU + iterate)
    __shared__ double s_gl, s_gu, s_pivmin, s_tnorm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += blockDim.x) {
        d[i] = dg[i];
        const double ei = i + 1 < n ? eg[i] : 0.0;
        e[i] = ei;
        e2[i] = ei * ei;
    }
    __syncthreads();
    if (warp == 0) {
        double gl = DBL_MAX, gu = -DBL_MAX, emax = 0.0, tn = 0.0;
        for (int i = lane; i < n; i += 32) {
            const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
            gl = fmin(gl, d[i] - r);
            gu = fmax(gu, d[i] + r);
            emax = fmax(emax, e2[i]);
            tn = fmax(tn, fabs(d[i]) + r);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
            gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
            emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
            tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
        }
        if (lane == 0) {
            const double pad = 2.0 * DBL_EPSILON * fmax(fabs(gl), fabs(gu)) + 1e-300;
            s_gl = gl - pad;
            s_gu = gu + pad;
            s_pivmin = DBL_MIN * fmax(1.0, emax);
            s_tnorm = tn;
        }
    }
    __syncthreads();
    const int j = blockIdx.x * kTbiWarps + warp;
    if (j >= n) return;
    const double pivmin = s_pivmin, tnorm = s_tnorm;
    // j-th smallest eigenvalue: count(lo) <= j < count(hi)
    double lo = s_gl, hi = s_gu;
    for (int it = 0; it < 40; ++it) {
        const double width = hi - lo;
        if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin) break;
        const double x = lo + width * (lane + 1) / 33.0;
        const int c = sturm_count(d, e2, n, x, pivmin);
        const unsigned above = __ballot_sync(0xffffffffu, c > j);
        const int first = above ? __ffs(above) - 1 : 32;
        const double xf = __shfl_sync(0xffffffffu, x, first < 32 ? first : 31);
        const double xp = __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0);
        if (first < 32) hi = xf;
        if (first > 0) lo = xp;
        if (first == 32) lo = xf;  // all points below: root in (x_31, hi]
    }
    const double lmb = 0.5 * (lo + hi);
    if (lane == 0) lam[j] = lmb;
    // neighbours closer than kTbiGap ||T|| -> inverse iteration is not reliable
    if (lane == 0 && j + 1 < n) {
        const int c = sturm_count(d, e2, n, lmb + kTbiGap * tnorm, pivmin);
        if (c > j + 1) atomicExch(clustered, 1);
    }
    // inverse iteration on (T - lmb I): LU with partial pivoting (the dgttrf /
    // dgttrs recurrences), three solves from a fixed non-degenerate start (lane 0)
    if (lane == 0) {
        double* dd = work + warp * 6 * n;  // diagonal of U
        double* du = dd + n;               // first superdiagonal of U
        double* du2 = du + n;              // second superdiagonal (fill-in)
        double* dl = du2 + n;              // multipliers
        double* sw = dl + n;               // 1.0 where rows i, i+1 were interchanged
        for (int i = 0; i < n; ++i) {
            dd[i] = d[i] - lmb;
            du[i] = i + 1 < n ? e[i] : 0.0;
            dl[i] = i + 1 < n ? e[i] : 0.0;
            du2[i] = 0.0;
            sw[i] = 0.0;
        }
        const double tiny = DBL_EPSILON * fmax(tnorm, DBL_MIN);
        for (int i = 0; i + 1 < n; ++i) {
            if (fabs(dd[i]) >= fabs(dl[i])) {
                const double fact = dd[i] != 0.0 ? dl[i] / dd[i] : 0.0;
                dl[i] = fact;
                dd[i + 1] -= fact * du[i];
            } else {
                const double fact = dd[i] / dl[i];
                dd[i] = dl[i];
                dl[i] = fact;
                const double t = du[i];
                du[i] = dd[i + 1];
                dd[i + 1] = t - fact * dd[i + 1];
                if (i + 2 < n) {
                    du2[i] = du[i + 1];
                    du[i + 1] = -fact * du[i + 1];
                }
                sw[i] = 1.0;
            }
            if (fabs(dd[i]) < tiny) dd[i] = copysign(tiny, dd[i]);
        }
        if (fabs(dd[n - 1]) < tiny) dd[n - 1] = copysign(tiny, dd[n - 1]);
        for (int i = 0; i < n; ++i) dd[i] = 1.0 / dd[i];  // solves multiply by 1/pivot
        double* xs = sw + n;  // the iterate, in shared memory
        auto X = [&](int i) -> double& { return xs[i]; };
        for (int i = 0; i < n; ++i) X(i) = 1.0 + 0.01 * ((i * 7 + j * 13) % 17);
        for (int pass = 0; pass < 3; ++pass) {
            for (int i = 0; i + 1 < n; ++i) {  // L^{-1} with the interchanges
                if (sw[i] == 0.0) {
                    X(i + 1) -= dl[i] * X(i);
                } else {
                    const double t = X(i);
                    X(i) = X(i + 1);
                    X(i + 1) = t - dl[i] * X(i);
                }
            }
            double nrm = 0.0;
            for (int i = n - 1; i >= 0; --i) {  // U^{-1}
                double sum = X(i);
                if (i + 1 < n) sum -= du[i] * X(i + 1);
                if (i + 2 < n) sum -= du2[i] * X(i + 2);
                sum *= dd[i];
                X(i) = sum;
                nrm = fmax(nrm, fabs(sum));
            }
            const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
            for (int i = 0; i < n; ++i) X(i) *= inv;
        }
        double s2 = 0.0;
        for (int i = 0; i < n; ++i) s2 = fma(X(i), X(i), s2);
        const double inv = 1.0 / sqrt(s2);
        for (int i = 0; i < n; ++i) X(i) *= inv;
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) z[static_cast<int64_t>(i) * ldz + j] = work[warp * 6 * n + 5 * n + i];
}

// ---- 3. orthonormalisation: Z <- Z (3I - Z^T Z) / 2, twice -----------------------------
// Z (n x n, global, row stride ldz) <- Z (3I - Z^T Z) / 2, twice. Phase a holds
// Z in shared memory to form S = (3I - Z^T Z)/2 (written to global scratch);
// phase b holds S in shared memory while each warp streams one row of Z
// through registers. A step whose S is already I to 1e-15 is skipped.
__global__ void __launch_bounds__(kTbiThreads, 1)
tbi_orth_kernel(double* __restrict__ z, int n, int ldz, double* __restrict__ S,
                const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double osm[];
    __shared__ int s_dev;
    const int lds = n | 1;
    double* M = osm;  // Z (phase a) or S (phase b), n x lds
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int step = 0; step < 2; ++step) {
        if (threadIdx.x == 0) s_dev = 0;
        load_square(M, lds, z, ldz, n);
        __syncthreads();
        // S(a, b) for b >= a: warp per a, lanes over b
        for (int a = warp; a < n; a += nwarp) {
            for (int b = a + lane; b < n; b += 32) {
                double acc = 0.0;
                for (int t = 0; t < n; ++t) acc = fma(M[t * lds + a], M[t * lds + b], acc);
                const double v = 0.5 * ((a == b ? 3.0 : 0.0) - acc);
                const double dev = fabs(v - (a == b ? 1.0 : 0.0));
                if (dev > (step == 0 ? 1e-15 : 1e-10)) s_dev = 1;
                S[a * n + b] = v;
                S[b * n + a] = v;
            }
        }
        __syncthreads();
        if (s_dev == 0) break;
        load_square(M, lds, S, n, n);
        __syncthreads();
        const int nb = (n + 31) / 32;
        for (int i = warp; i < n; i += nwarp) {
            double zr[8], out[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int col = lane + 32 * q;
                zr[q] = (q < nb && col < n) ? z[static_cast<int64_t>(i) * ldz + col] : 0.0;
                out[q] = 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q >= nb) break;
                for (int tl = 0; tl < 32; ++tl) {
                    const int t = 32 * q + tl;
                    if (t >= n) break;
                    const double zt = __shfl_sync(0xffffffffu, zr[q], tl);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int col = lane + 32 * c;
                        if (c < nb && col < n) out[c] = fma(zt, M[t * lds + col], out[c]);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int col = lane + 32 * c;
                if (c < nb && col < n) z[static_cast<int64_t>(i) * ldz + col] = out[c];
            }
        }
        __syncthreads();
    }
}

// ---- 4. back-transform: V = H_0 H_1 ... H_{n-3} Z, one warp per column -------------
constexpr int kBtWarps = 16;

__global__ void __launch_bounds__(32 * kBtWarps, 1)
tbi_backtransform_kernel(const double* __restrict__ hv, const double* __restrict__ tau,
                         const double* __restrict__ z, int n, int ldz, double* __restrict__ vecs, int ldv,
                         const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double bsm[];
    double* H = bsm;                     // all reflectors, n x n (row k = v_k)
    double* T = H + static_cast<size_t>(n) * n;  // tau, n
    double* X = T + n;                   // kBtWarps x n columns being transformed
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    load_square(H, n, hv, n, n);
    for (int x = threadIdx.x; x < n; x += blockDim.x) T[x] = tau[x];
    const int col = blockIdx.x * kBtWarps + warp;
    double* x = X + warp * n;
    if (col < n)
        for (int i = lane; i < n; i += 32) x[i] = z[static_cast<int64_t>(i) * ldz + col];
    __syncthreads();
    if (col >= n) return;
    for (int k = n - 3; k >= 0; --k) {
        const double t = T[k];
        if (t == 0.0) continue;
        const double* vk = H + static_cast<size_t>(k) * n;
        double s = 0.0;
        for (int i = k + 1 + lane; i < n; i += 32) s = fma(vk[i], x[i], s);
        s = warp_sum(s) * t;
        for (int i = k + 1 + lane; i < n; i += 32) x[i] = fma(-s, vk[i], x[i]);
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) vecs[static_cast<int64_t>(i) * ldv + col] = x[i];
}

__global__ void tbi_clear_kernel(int32_t* flag) { *flag = 0; }

}  // namespace

bool tbi_supported(int l) { return l >= 3 && l <= 160; }

size_t tbi_workspace_bytes(int l) {
    const size_t n = l;
    return sizeof(double) * (n * n /*hv*/ + n /*tau*/ + 2 * n /*d,e*/ + 2 * n * n /*z, S*/) + 64;
}

// Runs the tridiagonal path; sets *clustered (device) when the spectrum needs
// the Jacobi fallback. Writes w.lam / w.vecs (stride w.lp) like jacobi_eig.
void tbi_eig(const double* g, EigWorkspace& w, void* tbi_ws, int32_t* clustered, const int32_t* gate,
             cudaStream_t stream) {
    const int n = w.l;
    double* hv = static_cast<double*>(tbi_ws);
    double* tau = hv + static_cast<size_t>(n) * n;
    double* d = tau + n;
    double* e = d + n;
    double* z = e + n;
    tbi_clear_kernel<<<1, 1, 0, stream>>>(clustered);
    DSVD_LAUNCH_CHECK();
    const int lda = n | 1;
    const size_t s1 = sizeof(double) * (static_cast<size_t>(n) * lda + 2 * n);
    const size_t s3 = sizeof(double) * static_cast<size_t>(n) * lda;
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s1)));
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_orth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s3)));
    tbi_tridiag_kernel<<<1, kTbiThreads, s1, stream>>>(g, n, d, e, hv, tau, gate, nullptr);
    DSVD_LAUNCH_CHECK();
    const size_t s2 = sizeof(double) * (3 * static_cast<size_t>(n) + kTbiWarps * 6 * static_cast<size_t>(n));
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s2)));
    tbi_eig_kernel<<<static_cast<unsigned>(ceil_div(n, kTbiWarps)), 32 * kTbiWarps, s2, stream>>>(
        d, e, n, w.lam, z, n, clustered, gate, nullptr);
    DSVD_LAUNCH_CHECK();
    tbi_orth_kernel<<<1, kTbiThreads, s3, stream>>>(z, n, n, z + static_cast<size_t>(n) * n, gate,
                                                    clustered);
    DSVD_LAUNCH_CHECK();
    const size_t s4 = sizeof(double) * (static_cast<size_t>(n) * n + n + kBtWarps * static_cast<size_t>(n));
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_backtransform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s4)));
    tbi_backtransform_kernel<<<static_cast<unsigned>(ceil_div(n, kBtWarps)), 32 * kBtWarps, s4, stream>>>(
        hv, tau, z, n, n, w.vecs, w.lp, gate, clustered);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
