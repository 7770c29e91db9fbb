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

// Minimum eigenvalue gap (relative to ||T||) for the twisted-factorisation
// vectors: a pair closer than gap has its two vectors accurate only to an angle
// ~ eps / gap inside the pair's 2-D eigenspace; at 1e-12 that is ~1e-4, which
// the two Newton-Schulz steps remove (1e-4 -> 1e-8 -> 1e-16), and the mixing
// inside the pair changes the factorisation by ~angle x gap ~ 1e-16 ||T||.
// Tighter clusters (e.g. repeated eigenvalues) take the Jacobi fallback.
constexpr double kTbiGap = 1e-12;

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

// sqrt and reciprocal from the hardware approximations plus Newton steps
// (within an ulp; the step's critical path is the reflector, and the IEEE
// sequences were ~40% of its latency, tools/micro/tridiag_probe.cu)
__device__ __forceinline__ double sqrt_nr(double a) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    const double ha = 0.5 * a;
    r = r * fma(-ha * r, r, 1.5);
    r = r * fma(-ha * r, r, 1.5);
    const double s = a * r;
    return fma(0.5 * r, fma(-s, s, a), s);
}
__device__ __forceinline__ double rcp_nr(double a) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    r = r * fma(-a, r, 2.0);
    r = r * fma(-a, r, 2.0);
    return fma(r, fma(-a, r, 1.0), r);
}

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
        r.alpha = -copysign(sqrt_nr(sig), r.x0);
        r.v0 = r.x0 - r.alpha;
        r.tau = 2.0 * rcp_nr(tail + r.v0 * r.v0);
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
            const int C = min((kTridWarps - 1) / G, max(1, (m + 15) / 16));  // column chunks of >= ~16
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
                const int C = min((kTridWarps - 1) / G, max(1, (m + 15) / 16));
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
                __syncwarp();  // lanes past row n - 1 skipped the block above
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

// Wide variant (n > kTridSmemMaxN, up to 320): A no longer fits in shared
// memory, so the full symmetric matrix lives in global memory (L2-resident,
// 0.8 MB at n = 320), element (i, j) at A[j * n + i], and every access is
// lane-per-row, i.e. coalesced. Same three phases per step with 32 warps:
// B (reflector on warp 0, p = A22 x on the rest: 32-row groups x column
// chunks, eight loads in flight per lane), C1 (v, w, K), C2 (the symmetric
// rank-2 update A22 -= v u^T + u v^T, u = w - K v, on all m x m entries with
// the two products added before the subtraction, so A stays exactly
// symmetric).
constexpr int kTridBigThreads = 1024;
constexpr int kTridBigWarps = kTridBigThreads / 32;

__global__ void __launch_bounds__(kTridBigThreads, 1)
tbi_tridiag_big_kernel(const double* __restrict__ g, int n, double* __restrict__ A, double* __restrict__ d,
                       double* __restrict__ e, double* __restrict__ hv, double* __restrict__ tau_out,
                       const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ __align__(16) double tbm[];
    double2* vw = reinterpret_cast<double2*>(tbm);     // n: (v_i, u_i)
    double* xk = tbm + 2 * n;                          // n: column k (x)
    double* part = xk + n;                             // (kTridBigWarps - 1) x n matvec partials
    __shared__ Reflector s_ref;
    __shared__ double s_ksum[kTridBigWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int x = tid; x < n * n; x += blockDim.x) A[x] = g[x];  // g row-major symmetric: same layout
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
        const int k1 = k + 1, m = n - k1;
        const int G = (m + 31) >> 5;
        const int C = min((kTridBigWarps - 1) / G, max(1, (m + 15) / 16));
        for (int j = k1 + tid; j < n; j += blockDim.x) xk[j] = A[k * n + j];
        __syncthreads();
        // ---- B ----
        if (warp == 0) {
            double sig = 0.0;
            for (int i = k1 + lane; i < n; i += 32) sig = fma(xk[i], xk[i], sig);
            sig = warp_sum(sig);
            if (lane == 0) {
                Reflector r;
                r.x0 = xk[k1];
                r.alpha = r.x0;
                r.tau = 0.0;
                r.v0 = r.x0;
                const double tail = sig - r.x0 * r.x0;
                if (tail > 0.0) {
                    r.alpha = -copysign(sqrt(sig), r.x0);
                    r.v0 = r.x0 - r.alpha;
                    r.tau = 2.0 / (tail + r.v0 * r.v0);
                }
                s_ref = r;
                tau_out[k] = r.tau;
                e[k] = r.alpha;
                d[k] = A[k * n + k];
            }
        } else {
            const int item = warp - 1, grp = item % G, c = item / G;
            if (c < C) {
                const int i = k1 + 32 * grp + lane;
                const int len = (m + C - 1) / C;
                const int j0 = k1 + c * len, j1 = min(n, j0 + len);
                double acc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] = 0.0;
                if (i < n) {
                    int j = j0;
                    for (; j + 7 < j1; j += 8) {
                        double a[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) a[u] = A[(j + u) * n + i];
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[u] = fma(a[u], xk[j + u], acc[u]);
                    }
                    for (; j < j1; ++j) acc[0] = fma(A[j * n + i], xk[j], acc[0]);
                    part[c * n + i] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
                }
            }
        }
        __syncthreads();
        // ---- C1 ----
        const Reflector ref = s_ref;
        {
            double t = 0.0;
            if (tid < m) {
                const int i = k1 + tid;
                double p = 0.0;
                for (int c = 0; c < C; ++c) p += part[c * n + i];
                p = fma(ref.v0 - ref.x0, A[k1 * n + i], p);  // x -> v: first entry v0
                const double vi = i == k1 ? ref.v0 : xk[i];
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
        // ---- C2: A22 -= v u^T + u v^T, u = w - (tau K / 2) v -------------------------
        {
            double ks = 0.0;
            for (int q = 0; q < G; ++q) ks += s_ksum[q];
            const double hk = 0.5 * ref.tau * ks;
            const int ntile = G * G;
            for (int tile = warp; tile < ntile; tile += kTridBigWarps) {
                const int gr = tile % G, gc = tile / G;
                const int i = k1 + 32 * gr + lane;
                if (i >= n) continue;
                const double2 pi = vw[i];
                const double vi = pi.x, ui = fma(-hk, pi.x, pi.y);
                const int jb = k1 + 32 * gc, je = min(jb + 32, n);
                for (int j = jb; j < je; ++j) {
                    const double2 q = vw[j];
                    const double uj = fma(-hk, q.x, q.y);
                    A[j * n + i] -= vi * uj + ui * q.x;
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = A[(n - 2) * n + (n - 2)];
            e[n - 2] = A[(n - 2) * n + (n - 1)];
        }
        d[n - 1] = A[(n - 1) * n + (n - 1)];
    }
}

size_t tridiag_big_smem_bytes(int n) { return sizeof(double) * (3 * static_cast<size_t>(n) + (kTridBigWarps - 1) * static_cast<size_t>(n)); }

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

// Two Sturm counts at once: independent recurrences interleaved, so the
// dependent-latency chain is paid once for both points.
__device__ __forceinline__ void sturm_count2(const double* d, const double* e2, int n, double x0, double x1,
                                             double pivmin, int& c0, int& c1) {
    double q0 = d[0] - x0, q1 = d[0] - x1;
    if (fabs(q0) < pivmin) q0 = -pivmin;
    if (fabs(q1) < pivmin) q1 = -pivmin;
    int a0 = q0 < 0.0, a1 = q1 < 0.0;
    for (int i = 1; i < n; ++i) {
        const double di = d[i], ei = e2[i - 1];
        q0 = (di - x0) - ei * rcp_fast(q0);
        q1 = (di - x1) - ei * rcp_fast(q1);
        if (fabs(q0) < pivmin) q0 = -pivmin;
        if (fabs(q1) < pivmin) q1 = -pivmin;
        a0 += q0 < 0.0;
        a1 += q1 < 0.0;
    }
    c0 = a0;
    c1 = a1;
}

// 1/q to full double precision (approximation + two Newton steps); the LU of
// the inverse iteration only needs a backward-stable factorisation
__device__ __forceinline__ double rcp_nr2(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    r = r * fma(-q, r, 2.0);
    return r * fma(-q, r, 2.0);
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
constexpr int kGridPts = 2048;  // shared Sturm-count grid (tbi_grid_kernel)

#ifdef DSVD_EIG_PROBE  // tools/micro/eig_probe.cu: per-eigenvalue phase clocks
__device__ long long g_eig_probe[256][6];
#define EIG_PROBE(j, slot)                                             \
    do {                                                               \
        if ((threadIdx.x & 31) == 0) g_eig_probe[j][slot] = clock64(); \
    } while (0)
#else
#define EIG_PROBE(j, slot) \
    do {                   \
    } while (0)
#endif

// Gershgorin bounds, pivmin and ||T|| of the tridiagonal (d, e), one warp.
struct TriBounds {
    double gl, gu, pivmin, tnorm;
};
__device__ TriBounds tri_bounds(const double* d, const double* e, const double* e2, int n, int lane) {
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
    const double pad = 2.0 * DBL_EPSILON * fmax(fabs(gl), fabs(gu)) + 1e-300;
    return {gl - pad, gu + pad, DBL_MIN * fmax(1.0, emax), tn};
}

// Grid point t of the shared count grid: 0 -> gl, 1 .. kGridPts-1 geometric
// from gu * 2^-70 up to gu (the Gram spectrum is non-negative and spans many
// decades), so every eigenvalue above gu * 2^-70 starts bracketed to ~2.4%.
__device__ __forceinline__ double grid_x(int t, double gl, double gu) {
    if (t == 0 || gu <= 0.0) return gl + (gu - gl) * t / (kGridPts - 1);
    return gu * exp2(-70.0 * (kGridPts - 1 - t) / (kGridPts - 2));
}

__device__ __forceinline__ void load_tri(const double* dg, const double* eg, int n, double* d, double* e,
                                         double* e2) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        d[i] = dg[i];
        const double ei = i + 1 < n ? eg[i] : 0.0;
        e[i] = ei;
        e2[i] = ei * ei;
    }
}

// counts[t] = number of eigenvalues below grid_x(t), two points per thread.
__global__ void __launch_bounds__(256)
tbi_grid_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n, int32_t* __restrict__ counts,
                const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double gsm2[];
    double* d = gsm2;
    double* e = d + n;
    double* e2 = e + n;
    load_tri(dg, eg, n, d, e, e2);
    __syncthreads();
    const TriBounds b = tri_bounds(d, e, e2, n, threadIdx.x & 31);
    const int t0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (t0 >= kGridPts) return;
    int c0, c1;
    sturm_count2(d, e2, n, grid_x(t0, b.gl, b.gu), grid_x(t0 + 1, b.gl, b.gu), b.pivmin, c0, c1);
    counts[t0] = c0;
    counts[t0 + 1] = c1;
}

// One warp per eigenvalue j (ascending): bracket from the count grid, 65-way
// multisection on Sturm counts to full precision, then the eigenvector from a
// twisted factorization of T - lambda I (Dhillon-Parlett): forward and
// backward pivots D+ / D- (lanes 0 and 1), twist index r = argmin |gamma_r|,
// gamma_r = D+_r + D-_r - (d_r - lambda), and z from z_r = 1 outwards with the
// ratios -e/D+ and -e/D- (one pass; no inverse-iteration sweeps). Lane 2 checks
// the gap to the next eigenvalue at the same time.
__global__ void __launch_bounds__(32 * kTbiWarps)
tbi_eig_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
               const int32_t* __restrict__ counts, double* __restrict__ lam, double* __restrict__ z, int ldz,
               int32_t* __restrict__ clustered, const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double esm[];
    double* d = esm;        // n
    double* e = d + n;      // n
    double* e2 = e + n;     // n
    double* work = e2 + n;  // kTbiWarps x 3n: D+, D-, z
    __shared__ int s_cnt[kGridPts];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_tri(dg, eg, n, d, e, e2);
    for (int t = tid; t < kGridPts; t += blockDim.x) s_cnt[t] = counts[t];
    __syncthreads();
    const int j = blockIdx.x * kTbiWarps + warp;
    if (j >= n) return;
    const TriBounds b = tri_bounds(d, e, e2, n, lane);
    const double pivmin = b.pivmin, tnorm = b.tnorm;
    EIG_PROBE(j, 0);
    // bracket: last grid point with count <= j, first with count > j
    double lo = b.gl, hi = b.gu;
    {
        int tl = -1, th = kGridPts;  // count(x_tl) <= j < count(x_th); counts are monotone in t
        for (int t = lane; t < kGridPts; t += 32) {
            if (s_cnt[t] <= j) tl = max(tl, t);
            else th = min(th, t);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            tl = max(tl, __shfl_xor_sync(0xffffffffu, tl, o));
            th = min(th, __shfl_xor_sync(0xffffffffu, th, o));
        }
        if (tl >= 0) lo = grid_x(tl, b.gl, b.gu);
        if (th < kGridPts) hi = grid_x(th, b.gl, b.gu);
    }
    for (int it = 0; it < 40; ++it) {
        const double width = hi - lo;
        if (width <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin) break;
        const double x0 = lo + width * (2 * lane + 1) / 65.0;
        const double x1 = lo + width * (2 * lane + 2) / 65.0;
        int c0, c1;
        sturm_count2(d, e2, n, x0, x1, pivmin, c0, c1);
        const unsigned a0 = __ballot_sync(0xffffffffu, c0 > j), a1 = __ballot_sync(0xffffffffu, c1 > j);
        // point t = 2L + p (p = 0, 1); counts are monotone in t
        const unsigned any = a0 | a1;
        const int fl = any ? __ffs(any) - 1 : 32;  // lane holding the first point above
        const int ft = fl == 32 ? 64 : 2 * fl + (((a0 >> fl) & 1u) ? 0 : 1);
        auto xat = [&](int t) {  // x of point t (0 .. 63): lane t/2, slot t%2
            const double v0 = __shfl_sync(0xffffffffu, x0, t >> 1), v1 = __shfl_sync(0xffffffffu, x1, t >> 1);
            return (t & 1) ? v1 : v0;
        };
        const double xf = xat(ft < 64 ? ft : 63);
        const double xp = xat(ft > 0 ? ft - 1 : 0);
        if (ft < 64) hi = xf;
        if (ft > 0) lo = xp;
        if (ft == 64) lo = xf;  // all points below: root in (x_63, hi]
    }
    const double lmb = 0.5 * (lo + hi);
    EIG_PROBE(j, 1);
    if (lane == 0) lam[j] = lmb;
    double* Dp = work + warp * 3 * n;
    double* Dm = Dp + n;
    double* zs = Dm + n;
    if (lane == 0) {
        double q = d[0] - lmb;
        if (fabs(q) < pivmin) q = -pivmin;
        Dp[0] = q;
        for (int i = 1; i < n; ++i) {
            q = (d[i] - lmb) - e2[i - 1] * rcp_fast(q);
            if (fabs(q) < pivmin) q = -pivmin;
            Dp[i] = q;
        }
    } else if (lane == 1) {
        double q = d[n - 1] - lmb;
        if (fabs(q) < pivmin) q = -pivmin;
        Dm[n - 1] = q;
        for (int i = n - 2; i >= 0; --i) {
            q = (d[i] - lmb) - e2[i] * rcp_fast(q);
            if (fabs(q) < pivmin) q = -pivmin;
            Dm[i] = q;
        }
    } else if (lane == 2 && j + 1 < n) {
        // neighbours closer than kTbiGap ||T||: vectors from one shift are not reliable
        const int c = sturm_count(d, e2, n, lmb + kTbiGap * tnorm, pivmin);
        if (c > j + 1) atomicExch(clustered, 1);
    }
    __syncwarp();
    // twist index: argmin |gamma_r| (ties: smallest r)
    double gbest = DBL_MAX;
    int rbest = 0;
    for (int r = lane; r < n; r += 32) {
        const double g = fabs(Dp[r] + Dm[r] - (d[r] - lmb));
        if (g < gbest) {
            gbest = g;
            rbest = r;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double go = __shfl_xor_sync(0xffffffffu, gbest, o);
        const int ro = __shfl_xor_sync(0xffffffffu, rbest, o);
        if (go < gbest || (go == gbest && ro < rbest)) {
            gbest = go;
            rbest = ro;
        }
    }
    const int r = rbest;
    // ratios in parallel: z_i = ratio_i z_{i+1} (i < r), z_i = ratio_i z_{i-1} (i > r)
    for (int i = lane; i < n; i += 32)
        zs[i] = i < r ? -e[i] * rcp_nr2(Dp[i]) : (i > r ? -e[i - 1] * rcp_nr2(Dm[i]) : 1.0);
    __syncwarp();
    if (lane == 0) {
        double zi = 1.0;
        for (int i = r - 1; i >= 0; --i) {
            zi *= zs[i];
            zs[i] = zi;
        }
    } else if (lane == 1) {
        double zi = 1.0;
        for (int i = r + 1; i < n; ++i) {
            zi *= zs[i];
            zs[i] = zi;
        }
    }
    __syncwarp();
    double s2 = 0.0;
    for (int i = lane; i < n; i += 32) s2 = fma(zs[i], zs[i], s2);
    s2 = warp_sum(s2);
    const double inv = 1.0 / sqrt(s2);
    EIG_PROBE(j, 2);
    for (int i = lane; i < n; i += 32) z[static_cast<int64_t>(i) * ldz + j] = zs[i] * inv;
}

// ---- 3. orthonormalisation: Z <- Z (3I - Z^T Z) / 2, twice -----------------------------
// Each Newton-Schulz step is two small GEMMs over all SMs: 16 x 16 output tiles,
// the two n x 16 operand panels staged in shared memory. mode 0: C = A B;
// mode 1: C = (3I - A^T B) / 2 (the polar step's S). The operand layout:
// A(t, i) = trans_a ? a[t * n + i] : a[i * n + t], B(t, j) = b[t * n + j].
constexpr int kNsTile = 16;
constexpr int kNsChunk = 160;  // t-panel staged per pass (n <= 160: one pass)
constexpr int kNsMaxN = 320;

__global__ void __launch_bounds__(kNsTile * kNsTile)
tbi_ns_kernel(const double* __restrict__ a, int trans_a, const double* __restrict__ b, double* __restrict__ c,
              int n, int mode, const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    __shared__ double as[kNsChunk][kNsTile + 1];
    __shared__ double bs[kNsChunk][kNsTile];
    const int i0 = blockIdx.y * kNsTile, j0 = blockIdx.x * kNsTile, tid = threadIdx.x;
    const int ty = tid / kNsTile, tx = tid % kNsTile;
    double a0 = 0.0, a1 = 0.0;
    for (int t0 = 0; t0 < n; t0 += kNsChunk) {
        const int tn = min(kNsChunk, n - t0);
        if (t0 > 0) __syncthreads();
        for (int x = tid; x < tn * kNsTile; x += blockDim.x) {
            int t, ii;
            if (trans_a) { t = x / kNsTile; ii = x % kNsTile; }
            else { ii = x / tn; t = x % tn; }
            const int i = i0 + ii;
            as[t][ii] = i < n ? (trans_a ? a[(t0 + t) * n + i] : a[i * n + t0 + t]) : 0.0;
            const int tb = x / kNsTile, jj = x % kNsTile, j = j0 + jj;
            bs[tb][jj] = j < n ? b[(t0 + tb) * n + j] : 0.0;
        }
        __syncthreads();
        int t = 0;
        for (; t + 1 < tn; t += 2) {
            a0 = fma(as[t][ty], bs[t][tx], a0);
            a1 = fma(as[t + 1][ty], bs[t + 1][tx], a1);
        }
        if (t < tn) a0 = fma(as[t][ty], bs[t][tx], a0);
    }
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

// R: registers per lane (n <= 32 R); SMEM: reflectors staged in shared memory
// (n <= 160) or read from global / L2 (wider n, 0.8 MB of reflectors at 320)
template <int R, bool SMEM>
__global__ void __launch_bounds__(32 * kBtWarps)
tbi_backtransform_kernel(const double* __restrict__ hv, const double* __restrict__ tau,
                         const double* __restrict__ z, int n, int ldz, double* __restrict__ vecs, int ldv,
                         const int32_t* __restrict__ gate, const int32_t* __restrict__ skip) {
    if ((gate != nullptr && *gate != 0) || (skip != nullptr && *skip != 0)) return;
    extern __shared__ double bsm[];
    const double* H = hv;  // all reflectors, n x n (row k = v_k)
    const double* T = tau;
    if (SMEM) {
        double* Hs = bsm;
        double* Ts = Hs + static_cast<size_t>(n) * n;
        load_square(Hs, n, hv, n, n);
        for (int x = threadIdx.x; x < n; x += blockDim.x) Ts[x] = tau[x];
        H = Hs;
        T = Ts;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = blockIdx.x * kBtWarps + warp;
    double x[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        x[q] = (col < n && i < n) ? z[static_cast<int64_t>(i) * ldz + col] : 0.0;
    }
    if (SMEM) __syncthreads();
    if (col >= n) return;
    for (int k = n - 3; k >= 0; --k) {
        const double t = T[k];
        if (t == 0.0) continue;
        const double* vk = H + static_cast<size_t>(k) * n;
        double vr[R];
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int i = lane + 32 * q;
            vr[q] = (i > k && i < n) ? vk[i] : 0.0;
            s = fma(vr[q], x[q], s);
        }
        s = warp_sum(s) * t;
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = fma(-s, vr[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i < n) vecs[static_cast<int64_t>(i) * ldv + col] = x[q];
    }
}

__global__ void tbi_clear_kernel(int32_t* flag) { *flag = 0; }

}  // namespace

constexpr int kTridSmemMaxN = 160;  // tbi_tridiag_kernel / the staged back-transform

bool tbi_supported(int l) { return l >= 3 && l <= kNsMaxN; }

size_t tbi_workspace_bytes(int l) {
    const size_t n = l;
    return sizeof(double) * (n * n /*hv*/ + n /*tau*/ + 2 * n /*d,e*/ + 3 * n * n /*z, S, z2*/ +
                             (l > kTridSmemMaxN ? n * n : 0) /*A for the wide tridiagonalisation*/) +
           sizeof(int32_t) * kGridPts /*count grid*/ + 64;
}

// Runs the tridiagonal path; sets *clustered (device) when the spectrum needs
// the Jacobi fallback. Writes w.lam / w.vecs (stride w.lp) like jacobi_eig.
void tbi_eig(const double* g, EigWorkspace& w, void* tbi_ws, int32_t* clustered, const int32_t* gate,
             cudaStream_t stream, int phase) {
    const int n = w.l;
    double* hv = static_cast<double*>(tbi_ws);
    double* tau = hv + static_cast<size_t>(n) * n;
    double* d = tau + n;
    double* e = d + n;
    double* z = e + n;
    double* S = z + static_cast<size_t>(n) * n;
    double* z2 = S + static_cast<size_t>(n) * n;
    int32_t* counts = reinterpret_cast<int32_t*>(z2 + static_cast<size_t>(n) * n);
    if (phase != 2) {
    tbi_clear_kernel<<<1, 1, 0, stream>>>(clustered);
    DSVD_LAUNCH_CHECK();
    if (n <= kTridSmemMaxN) {
        const size_t s1 = tridiag_smem_bytes(n);
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(s1)));
        tbi_tridiag_kernel<<<1, kTridThreads, s1, stream>>>(g, n, d, e, hv, tau, gate, nullptr);
    } else {
        double* Aw = reinterpret_cast<double*>(counts + kGridPts);  // n x n, after the count grid
        const size_t s1 = tridiag_big_smem_bytes(n);
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_tridiag_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(s1)));
        tbi_tridiag_big_kernel<<<1, kTridBigThreads, s1, stream>>>(g, n, Aw, d, e, hv, tau, gate, nullptr);
    }
    DSVD_LAUNCH_CHECK();
    }
    if (phase == 1) return;
    tbi_grid_kernel<<<kGridPts / 512, 256, sizeof(double) * 3 * n, stream>>>(d, e, n, counts, gate, nullptr);
    DSVD_LAUNCH_CHECK();
    const size_t s2 = sizeof(double) * (3 * static_cast<size_t>(n) + kTbiWarps * 3 * static_cast<size_t>(n));
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(s2)));
    tbi_eig_kernel<<<static_cast<unsigned>(ceil_div(n, kTbiWarps)), 32 * kTbiWarps, s2, stream>>>(
        d, e, n, counts, w.lam, z, n, clustered, gate, nullptr);
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
    const unsigned bt_grid = static_cast<unsigned>(ceil_div(n, kBtWarps));
    if (n <= kTridSmemMaxN) {
        const size_t s4 = sizeof(double) * (static_cast<size_t>(n) * n + n);
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(tbi_backtransform_kernel<5, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s4)));
        tbi_backtransform_kernel<5, true><<<bt_grid, 32 * kBtWarps, s4, stream>>>(hv, tau, z, n, n, w.vecs, w.lp,
                                                                                  gate, clustered);
    } else {
        tbi_backtransform_kernel<10, false><<<bt_grid, 32 * kBtWarps, 0, stream>>>(hv, tau, z, n, n, w.vecs, w.lp,
                                                                                   gate, clustered);
    }
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
