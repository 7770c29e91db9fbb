// Tridiagonal eigensolver path for eigSVD's l x l Gram matrix on sm_100a:
//
//   1. tbi_tridiag_kernel  — Householder reduction A = Q T Q^T on one SM (the
//      reference's first stage, sym_eig.cpp:19-74, parallelised per step:
//      warp reductions for the norm, warp-per-row for p = tau A v, a
//      symmetric rank-2 update of the lower triangle in shared memory).
//   2. tbi_eig_kernel      — one warp per eigenvalue: 33-way multisection on
//      Sturm counts (each lane evaluates one point) to full precision, then
//      inverse iteration with a partially pivoted tridiagonal LU (lane 0).
//   3. tbi_ns_kernel       — two Newton-Schulz polar steps Z <- Z (3I - Z^T Z)/2
//      (four small GEMMs on all SMs) make the eigenvectors orthonormal to
//      working precision.
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
// lda = n | 1 (odd: a warp reading 32 consecutive rows of one column hits 32
// distinct banks pairs). Outputs d (n), e (n-1), reflectors hv[k*n + i]
// (i > k) and tau[k]. Step k, three block barriers:
//   B  warp 0 derives the reflector of column k (alpha, tau, v0) while warps
//      1..15 form p = A22 x with x = column k as stored: one lane per row,
//      the columns split into chunks across warps (partial sums per chunk);
//   C1 one thread per row: p += (v0 - x0) A(:, k+1) (the v0 substitution),
//      w = tau p, v; the products w_i v_i are warp-reduced for K;
//   C2 A22 -= v w^T + (w - 2K v) v^T, one warp per 32 x 32 lower tile, one
//      lane per row (column k+1, the next reflector's source, included).
// The per-step fixed latency (reflector: norm, sqrt, division) overlaps the
// matvec instead of serialising with the update (tools/micro/tridiag_probe.cu).
constexpr int kTridThreads = 512;
constexpr int kTridWarps = kTridThreads / 32;

#ifdef DSVD_TRID_PROBE  // tools/micro/tridiag_probe.cu: per-step phase clocks
__device__ long long g_trid_probe[192][4];
#define TRID_PROBE(k, slot)                                                   \
    do {                                                                      \
        if (threadIdx.x == 0 || (slot) == 3) g_trid_probe[k][slot] = clock64(); \
    } while (0)
#else
#define TRID_PROBE(k, slot) \
    do {                    \
    } while (0)
#endif

struct Reflector {
    double tau, v0, x0, alpha;
};

// Householder reflector of column c (rows c+1 .. n-1), evaluated by one warp.
__device__ __forceinline__ Reflector make_reflector(const double* A, int lda, int n, int c, int lane) {
    double sig = 0.0;
    for (int i = c + 1 + lane; i < n; i += 32) {
        const double x = A[i * lda + c];
        sig = fma(x, x, sig);
    }
    sig = warp_sum(sig);
    Reflector r;
    r.x0 = A[(c + 1) * lda + c];
    r.alpha = r.x0;
    r.tau = 0.0;
    r.v0 = r.x0;
    const double tail = sig - r.x0 * r.x0;  // sum of squares below the first entry
    if (tail > 0.0) {
        r.alpha = -copysign(sqrt(sig), r.x0);
        r.v0 = r.x0 - r.alpha;
        r.tau = 2.0 / (tail + r.v0 * r.v0);
    }
    return r;
}

__global__ void __launch_bounds__(kTridThreads, 1)
tbi_tridiag_kernel(const double* __restrict__ g, int n, double* __restrict__ d, double* __restrict__ e,
                   double* __restrict__ hv, double* __restrict__ tau_out, const int32_t* __restrict__ gate,
                   const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ __align__(16) double tsm[];
    const int lda = n | 1;
    double* A = tsm;                                   // n x lda
    double2* vw = reinterpret_cast<double2*>(A + n * lda + (n * lda & 1));  // n: (v_i, w_i)
    double* part = reinterpret_cast<double*>(vw + n);  // (kTridWarps - 1) x n matvec partials
    __shared__ Reflector s_ref;
    __shared__ double s_ksum[kTridWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_square(A, lda, g, n, n);
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
        const int k1 = k + 1, m = n - k1;
        const int G = (m + 31) >> 5;  // 32-row groups of the trailing block
        TRID_PROBE(k, 0);
        // ---- B ----
        __syncwarp();  // reconverge (lanes past row n - 1 skipped parts of C2)
        if (warp == 0) {
            const Reflector r = make_reflector(A, lda, n, k, lane);
            if (lane == 0) {
                s_ref = r;
                tau_out[k] = r.tau;
                e[k] = r.alpha;
                d[k] = A[k * lda + k];
            }
            TRID_PROBE(k, 3);
        } else {
            const int C = (kTridWarps - 1) / G;  // column chunks
            const int item = warp - 1, grp = item % G, c = item / G;
            if (c < C) {
                const int i = k1 + 32 * grp + lane;
                const int len = (m + C - 1) / C;
                const int j0 = k1 + c * len, j1 = min(n, j0 + len);
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                if (i < n) {
                    const double* xk = A + k;  // x_j = A(j, k)
                    auto el = [&](int j) { return j <= i ? A[i * lda + j] : A[j * lda + i]; };
                    int j = j0;
                    for (; j + 3 < j1; j += 4) {
                        a0 = fma(el(j), xk[j * lda], a0);
                        a1 = fma(el(j + 1), xk[(j + 1) * lda], a1);
                        a2 = fma(el(j + 2), xk[(j + 2) * lda], a2);
                        a3 = fma(el(j + 3), xk[(j + 3) * lda], a3);
                    }
                    for (; j < j1; ++j) a0 = fma(el(j), xk[j * lda], a0);
                    part[c * n + i] = (a0 + a1) + (a2 + a3);
                }
            }
        }
        __syncthreads();
        TRID_PROBE(k, 1);
        // ---- C1 ----
        __syncwarp();
        const Reflector ref = s_ref;
        {
            double t = 0.0;
            if (tid < m) {
                const int i = k1 + tid;
                const int C = (kTridWarps - 1) / G;
                double p = 0.0;
                for (int c = 0; c < C; ++c) p += part[c * n + i];
                p = fma(ref.v0 - ref.x0, A[i * lda + k1], p);
                const double vi = i == k1 ? ref.v0 : A[i * lda + k];
                const double wi = ref.tau * p;
                vw[i] = make_double2(vi, wi);
                hv[static_cast<int64_t>(k) * n + i] = vi;
                t = wi * vi;
            }
            if (warp < G) {
                t = warp_sum(t);
                if (lane == 0) s_ksum[warp] = t;
            }
        }
        __syncthreads();
        TRID_PROBE(k, 2);
        // ---- C2 ----
        {
            double ks = 0.0;
            for (int q = 0; q < G; ++q) ks += s_ksum[q];
            const double K2 = ref.tau * ks;  // 2K
            // lower 32 x 32 tiles (gr >= gc) of the trailing block, one per warp
            int gr = 0, t = warp;
            while (gr < G && t > gr) {
                t -= gr + 1;
                ++gr;
            }
            if (gr < G) {
                const int gc = t;
                const int i = k1 + 32 * gr + lane;
                if (i < n) {
                    const double2 pi = vw[i];
                    const double vi = pi.x, wi = fma(-K2, pi.x, pi.y);
                    double* row = A + i * lda;
                    const int jb = k1 + 32 * gc;
                    const int je = min(gr == gc ? i + 1 : jb + 32, n);
                    int j = jb;
                    for (; j + 3 < je; j += 4) {
                        const double2 q0 = vw[j], q1 = vw[j + 1], q2 = vw[j + 2], q3 = vw[j + 3];
                        const double e0 = row[j], e1 = row[j + 1], e2 = row[j + 2], e3 = row[j + 3];
                        row[j] = fma(-vi, q0.y, fma(-wi, q0.x, e0));
                        row[j + 1] = fma(-vi, q1.y, fma(-wi, q1.x, e1));
                        row[j + 2] = fma(-vi, q2.y, fma(-wi, q2.x, e2));
                        row[j + 3] = fma(-vi, q3.y, fma(-wi, q3.x, e3));
                    }
                    for (; j < je; ++j) {
                        const double2 q0 = vw[j];
                        row[j] = fma(-vi, q0.y, fma(-wi, q0.x, row[j]));
                    }
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = A[(n - 2) * lda + (n - 2)];
            e[n - 2] = A[(n - 1) * lda + (n - 2)];
        }
        d[n - 1] = A[(n - 1) * lda + (n - 1)];
    }
}

size_t tridiag_smem_bytes(int n) {
    const size_t lda = n | 1;
    return sizeof(double) * (n * lda + 1 + 2 * n + (kTridWarps - 1) * static_cast<size_t>(n));
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
// Each Newton-Schulz step is two small GEMMs over all SMs: 16 x 16 output tiles,
// the two n x 16 operand panels staged in shared memory. mode 0: C = A B;
// mode 1: C = (3I - A^T B) / 2 (the polar step's S). The operand layout:
// A(t, i) = trans_a ? a[t * n + i] : a[i * n + t], B(t, j) = b[t * n + j].
constexpr int kNsTile = 16;
constexpr int kNsMaxN = 160;

__global__ void __launch_bounds__(kNsTile * kNsTile)
tbi_ns_kernel(const double* __restrict__ a, int trans_a, const double* __restrict__ b, double* __restrict__ c,
              int n, int mode, const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    __shared__ double as[kNsMaxN][kNsTile + 1];
    __shared__ double bs[kNsMaxN][kNsTile];
    const int i0 = blockIdx.y * kNsTile, j0 = blockIdx.x * kNsTile, tid = threadIdx.x;
    for (int x = tid; x < n * kNsTile; x += blockDim.x) {
        int t, ii;
        if (trans_a) { t = x / kNsTile; ii = x % kNsTile; }
        else { ii = x / n; t = x % n; }
        const int i = i0 + ii;
        as[t][ii] = i < n ? (trans_a ? a[t * n + i] : a[i * n + t]) : 0.0;
        const int tb = x / kNsTile, jj = x % kNsTile, j = j0 + jj;
        bs[tb][jj] = j < n ? b[tb * n + j] : 0.0;
    }
    __syncthreads();
    const int ty = tid / kNsTile, tx = tid % kNsTile;
    double a0 = 0.0, a1 = 0.0;
    int t = 0;
    for (; t + 1 < n; t += 2) {
        a0 = fma(as[t][ty], bs[t][tx], a0);
        a1 = fma(as[t + 1][ty], bs[t + 1][tx], a1);
    }
    if (t < n) a0 = fma(as[t][ty], bs[t][tx], a0);
    const int i = i0 + ty, j = j0 + tx;
    if (i < n && j < n) {
        const double acc = a0 + a1;
        c[i * n + j] = mode == 0 ? acc : 0.5 * ((i == j ? 3.0 : 0.0) - acc);
    }
}

// ---- 4. back-transform: V = H_0 H_1 ... H_{n-3} Z, one warp per column -------------
// The column lives in registers (lane owns rows lane + 32q); the reflectors are
// staged in shared memory once per CTA.
constexpr int kBtWarps = 8;
constexpr int kBtRegs = (kNsMaxN + 31) / 32;

__global__ void __launch_bounds__(32 * kBtWarps, 1)
tbi_backtransform_kernel(const double* __restrict__ hv, const double* __restrict__ tau,
                         const double* __restrict__ z, int n, int ldz, double* __restrict__ vecs, int ldv,
                         const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double bsm[];
    double* H = bsm;                              // all reflectors, n x n (row k = v_k)
    double* T = H + static_cast<size_t>(n) * n;   // tau, n
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    load_square(H, n, hv, n, n);
    for (int x = threadIdx.x; x < n; x += blockDim.x) T[x] = tau[x];
    const int col = blockIdx.x * kBtWarps + warp;
    double x[kBtRegs];
#pragma unroll
    for (int q = 0; q < kBtRegs; ++q) {
        const int i = lane + 32 * q;
        x[q] = (col < n && i < n) ? z[static_cast<int64_t>(i) * ldz + col] : 0.0;
    }
    __syncthreads();
    if (col >= n) return;
    for (int k = n - 3; k >= 0; --k) {
        const double t = T[k];
        if (t == 0.0) continue;
        const double* vk = H + static_cast<size_t>(k) * n;
        double vr[kBtRegs];
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kBtRegs; ++q) {
            const int i = lane + 32 * q;
            vr[q] = (i > k && i < n) ? vk[i] : 0.0;
            s = fma(vr[q], x[q], s);
        }
        s = warp_sum(s) * t;
#pragma unroll
        for (int q = 0; q < kBtRegs; ++q) x[q] = fma(-s, vr[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < kBtRegs; ++q) {
        const int i = lane + 32 * q;
        if (i < n) vecs[static_cast<int64_t>(i) * ldv + col] = x[q];
    }
}

__global__ void tbi_clear_kernel(int32_t* flag) { *flag = 0; }

}  // namespace

bool tbi_supported(int l) { return l >= 3 && l <= 160; }

size_t tbi_workspace_bytes(int l) {
    const size_t n = l;
    return sizeof(double) * (n * n /*hv*/ + n /*tau*/ + 2 * n /*d,e*/ + 3 * n * n /*z, S, z2*/) + 64;
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
    double* S = z + static_cast<size_t>(n) * n;
    double* z2 = S + static_cast<size_t>(n) * n;
    tbi_clear_kernel<<<1, 1, 0, stream>>>(clustered);
    DSVD_LAUNCH_CHECK();
    const size_t s1 = tridiag_smem_bytes(n);
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s1)));
    tbi_tridiag_kernel<<<1, kTridThreads, s1, stream>>>(g, n, d, e, hv, tau, gate, nullptr);
    DSVD_LAUNCH_CHECK();
    const size_t s2 = sizeof(double) * (3 * static_cast<size_t>(n) + kTbiWarps * 6 * static_cast<size_t>(n));
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s2)));
    tbi_eig_kernel<<<static_cast<unsigned>(ceil_div(n, kTbiWarps)), 32 * kTbiWarps, s2, stream>>>(
        d, e, n, w.lam, z, n, clustered, gate, nullptr);
    DSVD_LAUNCH_CHECK();
    const dim3 ns_grid(static_cast<unsigned>(ceil_div(n, kNsTile)), static_cast<unsigned>(ceil_div(n, kNsTile)));
    for (int step = 0; step < 2; ++step) {
        double* zi = step == 0 ? z : z2;
        double* zo = step == 0 ? z2 : z;
        tbi_ns_kernel<<<ns_grid, kNsTile * kNsTile, 0, stream>>>(zi, 1, zi, S, n, 1, gate, clustered);
        DSVD_LAUNCH_CHECK();
        tbi_ns_kernel<<<ns_grid, kNsTile * kNsTile, 0, stream>>>(zi, 0, S, zo, n, 0, gate, clustered);
        DSVD_LAUNCH_CHECK();
    }
    const size_t s4 = sizeof(double) * (static_cast<size_t>(n) * n + n);
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_backtransform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s4)));
    tbi_backtransform_kernel<<<static_cast<unsigned>(ceil_div(n, kBtWarps)), 32 * kBtWarps, s4, stream>>>(
        hv, tau, z, n, n, w.vecs, w.lp, gate, clustered);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
