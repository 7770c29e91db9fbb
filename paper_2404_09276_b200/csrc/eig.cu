// Symmetric l x l eigensolver for eigSVD on sm_100a: parallel cyclic
// (round-robin) two-sided Jacobi in ONE CTA of 1024 threads with G resident
// in shared memory (up to l = 164; larger l keeps G in global/L2).
//
// The reference uses Householder + implicit QL (sym_eig.cpp:19-130), a serial
// algorithm. Jacobi computes the same eigenpairs to roundoff, with high
// relative accuracy for the positive semidefinite Gram matrices it sees here,
// and converges in few sweeps late in the power loop where G is nearly
// diagonal. Each round applies l/2 disjoint rotations as independent 2x2
// block updates G <- J^T G J (upper blocks computed once and mirrored, so G
// stays exactly symmetric). Rotations are logged and a second kernel replays
// them on the rows of V = I * J_1 * J_2 * ... in parallel (rows of V are
// independent under right multiplication), keeping V out of the CTA's
// shared-memory budget.
//
// eig_svd_finish then applies the reference's eigSVD rules exactly
// (decompositions.cpp:52-73): descending order, rank floor
// max(rows, l) * eps * sqrt(lambda_max), s = sqrt(lambda), the sign
// convention on V (:21-35), and for loop iterations the trace, the PVE stop
// rule (solver.cpp:38-50) and the shift update (:34-36), evaluated with the
// reference's operand order.
#include <cfloat>

#include "eig.cuh"

namespace dsvd {

namespace {

constexpr int kEigThreads = 1024;
constexpr int kMaxPairs = 256;  // lp <= 512
constexpr double kJacobiTol = 1e-15;
constexpr double kBigRatio2 = 1e-16;  // (1e-8)^2: sweep-level convergence test
constexpr int kSmemLimit = 227 * 1024;

__device__ __forceinline__ void pair_of(int round, int k, int lp, int& p, int& q) {
    const int m = lp - 1;
    if (k == 0) {
        p = m;
        q = round;
    } else {
        p = (round + k) % m;
        q = (round - k + m) % m;
    }
}

__global__ void __launch_bounds__(kEigThreads, 1)
jacobi_kernel(const double* __restrict__ g_in, int l, int lp, double* __restrict__ gbuf,
              int use_smem, double2* __restrict__ rot_log, int max_sweeps,
              double* __restrict__ lam, Control* ctrl, const int32_t* __restrict__ gate,
              const int32_t* __restrict__ need) {
    if (gate != nullptr && *gate != 0) return;
    if (need != nullptr && *need == 0) return;
    extern __shared__ double smem[];
    __shared__ double cs_c[kMaxPairs], cs_s[kMaxPairs], cs_t[kMaxPairs];
    __shared__ int pp[kMaxPairs], qq[kMaxPairs];
    __shared__ int rotated;
    double* G = use_smem ? smem : gbuf;
    const int tid = threadIdx.x;
    const int half = lp / 2;
    const int nblocks = half * (half + 1) / 2;
    // (kp, kr) of every upper 2x2 block, decoded once (fixed across rounds)
    uint16_t* blk = reinterpret_cast<uint16_t*>(use_smem ? smem + lp * lp : smem);
    for (int e = tid; e < lp * lp; e += blockDim.x) {
        const int i = e / lp, j = e % lp;
        G[e] = (i < l && j < l) ? g_in[i * l + j] : 0.0;
    }
    for (int kp = tid; kp < half; kp += blockDim.x) {
        const int base = kp * half - kp * (kp - 1) / 2;  // blocks before row kp
        for (int kr = kp; kr < half; ++kr) blk[base + (kr - kp)] = static_cast<uint16_t>((kp << 8) | kr);
    }
    __syncthreads();
    int sweep = 0;
    bool converged = false;
    for (; sweep < max_sweeps; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < lp - 1; ++round) {
            for (int k = tid; k < half; k += blockDim.x) {
                int p, q;
                pair_of(round, k, lp, p, q);
                const double a = G[p * lp + p], d = G[q * lp + q], b = G[p * lp + q];
                double c = 1.0, s = 0.0, t = 0.0;
                if (fabs(b) > kJacobiTol * sqrt(fabs(a)) * sqrt(fabs(d)) && fabs(b) > 1e-300) {
                    const double theta = (d - a) / (2.0 * b);
                    if (fabs(theta) > 1e150) {
                        t = 0.5 / theta;
                    } else {
                        t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
                    }
                    c = 1.0 / sqrt(fma(t, t, 1.0));
                    s = t * c;
                    if (s != 0.0) rotated = 1;
                }
                cs_c[k] = c;
                cs_s[k] = s;
                cs_t[k] = t;
                pp[k] = p;
                qq[k] = q;
                rot_log[(static_cast<int64_t>(sweep) * (lp - 1) + round) * half + k] = make_double2(c, s);
            }
            __syncthreads();
            for (int e = tid; e < nblocks; e += blockDim.x) {
                const int code = blk[e];
                const int kp = code >> 8, kr = code & 0xff;
                const double s1 = cs_s[kp], s2 = cs_s[kr];
                const int p = pp[kp], q = qq[kp];
                if (kp == kr) {
                    if (s1 != 0.0) {
                        const double t = cs_t[kp];
                        const double b = G[p * lp + q];
                        G[p * lp + p] -= t * b;
                        G[q * lp + q] += t * b;
                        G[p * lp + q] = 0.0;
                        G[q * lp + p] = 0.0;
                    }
                    continue;
                }
                if (s1 == 0.0 && s2 == 0.0) continue;
                const double c1 = cs_c[kp], c2 = cs_c[kr];
                const int r = pp[kr], s = qq[kr];
                const double xpr = G[p * lp + r], xps = G[p * lp + s];
                const double xqr = G[q * lp + r], xqs = G[q * lp + s];
                // columns (r, s) by J(kr), then rows (p, q) by J(kp)^T
                const double ypr = c2 * xpr - s2 * xps, yps = s2 * xpr + c2 * xps;
                const double yqr = c2 * xqr - s2 * xqs, yqs = s2 * xqr + c2 * xqs;
                const double zpr = c1 * ypr - s1 * yqr, zqr = s1 * ypr + c1 * yqr;
                const double zps = c1 * yps - s1 * yqs, zqs = s1 * yps + c1 * yqs;
                G[p * lp + r] = zpr;
                G[r * lp + p] = zpr;
                G[p * lp + s] = zps;
                G[s * lp + p] = zps;
                G[q * lp + r] = zqr;
                G[r * lp + q] = zqr;
                G[q * lp + s] = zqs;
                G[s * lp + q] = zqs;
            }
            __syncthreads();
        }
        if (rotated == 0) {
            converged = true;
            ++sweep;
            break;
        }
        __syncthreads();
    }
    for (int i = tid; i < lp; i += blockDim.x) lam[i] = G[i * lp + i];
    if (tid == 0) {
        ctrl->eig_sweeps = sweep;
        ctrl->total_sweeps += sweep;
        if (!converged && ctrl->status == DSVD_OK) {
            ctrl->status = DSVD_NUMERICAL;
            ctrl->stopped = 1;
        }
    }
}

// V = I * J_1 * ... replayed on one row of V per warp.
__global__ void jacobi_replay_kernel(const double2* __restrict__ rot_log, int l, int lp,
                                     const Control* ctrl, double* __restrict__ vecs,
                                     const int32_t* __restrict__ gate, const int32_t* __restrict__ need) {
    if (gate != nullptr && *gate != 0) return;
    if (need != nullptr && *need == 0) return;
    extern __shared__ double vrow_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + warp;
    if (row >= lp) return;
    double* v = vrow_all + warp * lp;
    for (int j = lane; j < lp; j += 32) v[j] = (j == row) ? 1.0 : 0.0;
    __syncwarp();
    const int sweeps = ctrl->eig_sweeps;
    const int half = lp / 2;
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int round = 0; round < lp - 1; ++round) {
            const double2* lg = rot_log + (static_cast<int64_t>(sw) * (lp - 1) + round) * half;
            for (int k = lane; k < half; k += 32) {
                const double2 cs = lg[k];
                if (cs.y != 0.0) {
                    int p, q;
                    pair_of(round, k, lp, p, q);
                    const double vp = v[p], vq = v[q];
                    v[p] = cs.x * vp - cs.y * vq;
                    v[q] = cs.y * vp + cs.x * vq;
                }
            }
            __syncwarp();
        }
    }
    for (int j = lane; j < lp; j += 32) vecs[static_cast<int64_t>(row) * lp + j] = v[j];
}


// ---- two-CTA cluster variant -----------------------------------------------------
// CTA 0 runs the Jacobi rounds on G (shared memory) exactly as jacobi_kernel;
// after computing a round's rotations it writes them straight into CTA 1's
// shared memory (DSMEM) and signals an mbarrier there. CTA 1 holds V and applies
// each round's rotations V <- V J while CTA 0 is already on the next rounds: the
// accumulation of eigenvectors runs concurrently on a second SM instead of in a
// replay kernel afterwards. A kClRing-slot ring with full/empty mbarriers (the
// empty ones live in CTA 0 and are signalled remotely) decouples the two.
constexpr int kClRing = 8;

__device__ __forceinline__ unsigned s_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(s_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_arrive(unsigned addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void cl_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(s_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                     : "memory");
}

__device__ __forceinline__ void cl_expect_tx_remote(unsigned addr, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;\n" ::"r"(addr),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cl_bulk_copy(unsigned remote_dst, const void* local_src, unsigned bytes,
                                             unsigned remote_bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            remote_dst),
        "r"(s_u32(local_src)), "r"(bytes), "r"(remote_bar)
        : "memory");
}

// Shared memory of each CTA: M (lp x lds, lds = lp + 1 odd so row and column
// strides hit distinct banks), the rotation ring (payload per round: half
// (c, s) pairs + a header {continue?, 0}), the local staging ring of CTA 0,
// mbarriers, and the block table.
size_t cluster_smem_bytes(int lp) {
    const size_t half = lp / 2, lds = lp + 1;
    return sizeof(double) * lp * lds + 2 * sizeof(double2) * kClRing * (half + 1) +
           2 * kClRing * sizeof(uint64_t) + sizeof(uint16_t) * half * (half + 1) / 2 + 128;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kEigThreads, 1)
jacobi_cluster_kernel(const double* __restrict__ g_in, int l, int lp, int max_sweeps,
                      double* __restrict__ lam, double* __restrict__ vecs, Control* ctrl,
                      const int32_t* __restrict__ gate, const int32_t* __restrict__ need) {
    // the gates are read by both CTAs before any cluster traffic, so both exit together
    if (gate != nullptr && *gate != 0) return;
    if (need != nullptr && *need == 0) return;
    extern __shared__ __align__(16) double cl_smem[];
    __shared__ double cs_c[kMaxPairs], cs_s[kMaxPairs], cs_t[kMaxPairs];
    __shared__ int pp[kMaxPairs], qq[kMaxPairs];
    __shared__ int rotated, big;
    const int half = lp / 2, lds = lp + 1;
    const int pay = half + 1;                                           // double2 per round
    double* M = cl_smem;                                                // G (rank 0) or V (rank 1)
    double2* ring = reinterpret_cast<double2*>(M + ((lp * lds + 1) & ~1));  // [kClRing][pay] (rank 1)
    double2* stage = ring + kClRing * pay;                              // [kClRing][pay] (rank 0)
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + kClRing * pay);  // rank 1
    uint64_t* empty = full + kClRing;                                   // rank 0
    uint16_t* blk = reinterpret_cast<uint16_t*>(empty + kClRing);       // rank 0
    const unsigned rank = cl_rank();
    const int tid = threadIdx.x;
    auto UP = [&](int i, int j) -> double& { return i <= j ? M[i * lds + j] : M[j * lds + i]; };
    const unsigned pay_bytes = static_cast<unsigned>(sizeof(double2) * pay);
    if (tid == 0) {
        for (int sl = 0; sl < kClRing; ++sl) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(&full[sl])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(&empty[sl])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cl_sync();

    if (rank == 0) {
        const int nblocks = half * (half + 1) / 2;
        for (int e = tid; e < lp * lp; e += blockDim.x) {
            const int i = e / lp, j = e % lp;
            M[i * lds + j] = (i < l && j < l) ? g_in[i * l + j] : 0.0;
        }
        for (int kp = tid; kp < half; kp += blockDim.x) {
            const int base = kp * half - kp * (kp - 1) / 2;
            for (int kr = kp; kr < half; ++kr) blk[base + (kr - kp)] = static_cast<uint16_t>((kp << 8) | kr);
        }
        __syncthreads();
        // hand round rg's payload (already in stage[sl]) to the V-CTA
        auto send = [&](int64_t rg) {
            const int sl = static_cast<int>(rg % kClRing);
            cl_wait(&empty[sl], static_cast<unsigned>(((rg / kClRing) & 1) ^ 1));
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const unsigned bar = cl_map(&full[sl], 1);
            cl_expect_tx_remote(bar, pay_bytes);
            cl_bulk_copy(cl_map(&ring[sl * pay], 1), &stage[sl * pay], pay_bytes, bar);
        };
        int64_t rg = 0;
        int sweep = 0;
        bool converged = false;
        for (; sweep < max_sweeps && !converged; ++sweep) {
            if (tid == 0) {
                rotated = 0;
                big = 0;
            }
            __syncthreads();
            for (int round = 0; round < lp - 1; ++round, ++rg) {
                const int sl = static_cast<int>(rg % kClRing);
                if (tid == 0)  // the staging slot is reusable once the V-CTA released it
                    cl_wait(&empty[sl], static_cast<unsigned>(((rg / kClRing) & 1) ^ 1));
                __syncthreads();
                for (int k = tid; k < half; k += blockDim.x) {
                    int p, q;
                    pair_of(round, k, lp, p, q);
                    const double a = M[p * lds + p], d = M[q * lds + q], b = UP(p, q);
                    double c = 1.0, s = 0.0, t = 0.0;
                    const double b2 = b * b, ad = fabs(a * d);
                    if (b2 > kBigRatio2 * ad) big = 1;
                    if (b2 > kJacobiTol * kJacobiTol * ad && fabs(b) > 1e-300) {
                        // t = tan(phi) = sgn(d - a) 2b / (|d - a| + sqrt((d - a)^2 + 4b^2))
                        const double dm = d - a, tb = 2.0 * b;
                        const double den = fabs(dm) + sqrt(fma(dm, dm, tb * tb));
                        t = (dm >= 0.0 ? tb : -tb) / den;
                        c = rsqrt(fma(t, t, 1.0));
                        s = t * c;
                        if (s != 0.0) rotated = 1;
                    }
                    cs_c[k] = c;
                    cs_s[k] = s;
                    cs_t[k] = t;
                    pp[k] = p;
                    qq[k] = q;
                    stage[sl * pay + k] = make_double2(c, s);
                    if (k == 0) stage[sl * pay + half] = make_double2(1.0, 0.0);  // header: continue
                    // make the generic-proxy writes visible to the bulk copy (async proxy)
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                }
                __syncthreads();
                if (tid == kEigThreads - 32) {
                    send(rg);  // the last warp forwards the round while the others update G
                } else if (tid < kEigThreads - 32) {
                    for (int e = tid; e < nblocks; e += kEigThreads - 32) {
                        const int code = blk[e];
                        const int kp = code >> 8, kr = code & 0xff;
                        const double s1 = cs_s[kp], s2 = cs_s[kr];
                        const int p = pp[kp], q = qq[kp];
                        if (kp == kr) {
                            if (s1 != 0.0) {
                                const double t = cs_t[kp];
                                double& bpq = UP(p, q);
                                const double bb = bpq;
                                M[p * lds + p] -= t * bb;
                                M[q * lds + q] += t * bb;
                                bpq = 0.0;
                            }
                            continue;
                        }
                        if (s1 == 0.0 && s2 == 0.0) continue;
                        const double c1 = cs_c[kp], c2 = cs_c[kr];
                        const int r = pp[kr], s = qq[kr];
                        // G is kept as its upper triangle only: every entry is read and
                        // written once per round (half the traffic of a mirrored update)
                        double& gpr = UP(p, r);
                        double& gps = UP(p, s);
                        double& gqr = UP(q, r);
                        double& gqs = UP(q, s);
                        const double xpr = gpr, xps = gps, xqr = gqr, xqs = gqs;
                        const double ypr = c2 * xpr - s2 * xps, yps = s2 * xpr + c2 * xps;
                        const double yqr = c2 * xqr - s2 * xqs, yqs = s2 * xqr + c2 * xqs;
                        gpr = c1 * ypr - s1 * yqr;
                        gqr = s1 * ypr + c1 * yqr;
                        gps = c1 * yps - s1 * yqs;
                        gqs = s1 * yps + c1 * yqs;
                    }
                }
                __syncthreads();
            }
            // quadratic convergence: once every off-diagonal entry seen in a sweep
            // was below 1e-8 of sqrt(g_pp g_qq), the sweep left them at ~1e-16
            converged = rotated == 0 || big == 0;
            __syncthreads();
        }
        if (tid == 0) {  // stop marker
            const int sl = static_cast<int>(rg % kClRing);
            cl_wait(&empty[sl], static_cast<unsigned>(((rg / kClRing) & 1) ^ 1));
            stage[sl * pay + half] = make_double2(0.0, 0.0);
            send(rg);
        }
        for (int i = tid; i < lp; i += blockDim.x) lam[i] = M[i * lds + i];
        if (tid == 0) {
            ctrl->eig_sweeps = sweep;
            ctrl->total_sweeps += sweep;
            if (!converged && ctrl->status == DSVD_OK) {
                ctrl->status = DSVD_NUMERICAL;
                ctrl->stopped = 1;
            }
        }
    } else {
        for (int e = tid; e < lp * lp; e += blockDim.x) {
            const int i = e / lp, j = e % lp;
            M[i * lds + j] = (i == j) ? 1.0 : 0.0;
        }
        __syncthreads();
        const int groups = blockDim.x / half;  // row groups (>= 1: half <= 82 here)
        const int k = tid % half, grp = tid / half;
        const int rows_per = (lp + groups - 1) / groups;
        for (int64_t rg = 0;; ++rg) {
            const int sl = static_cast<int>(rg % kClRing);
            // one thread acquires at cluster scope (each cluster-scope acquire
            // invalidates L1), the CTA barrier hands the slot to the others
            if (tid == 0) cl_wait(&full[sl], static_cast<unsigned>((rg / kClRing) & 1));
            __syncthreads();
            const double2* rot = ring + sl * pay;
            if (rot[half].x == 0.0) break;
            const int round = static_cast<int>(rg % (lp - 1));
            // thread -> (pair k, strip of rows): one rotation, several rows
            if (grp < groups) {
                const double2 cs = rot[k];
                if (cs.y != 0.0) {
                    int p, q;
                    pair_of(round, k, lp, p, q);
                    const int r0 = grp * rows_per, r1 = min(lp, r0 + rows_per);
                    for (int r = r0; r < r1; ++r) {
                        const double vp = M[r * lds + p], vq = M[r * lds + q];
                        M[r * lds + p] = cs.x * vp - cs.y * vq;
                        M[r * lds + q] = cs.y * vp + cs.x * vq;
                    }
                }
            }
            __syncthreads();
            if (tid == 0) cl_arrive(cl_map(&empty[sl], 0));
        }
        for (int e = tid; e < lp * lp; e += blockDim.x) {
            const int i = e / lp, j = e % lp;
            vecs[e] = M[i * lds + j];
        }
    }
    cl_sync();  // keep both CTAs' shared memory alive until all remote traffic is done
}

constexpr int kFinishThreads = 512;

__global__ void __launch_bounds__(kFinishThreads)
eig_svd_finish_kernel(const double* __restrict__ lam, const double* __restrict__ vecs, int l,
                      int lp, int64_t rows, double* __restrict__ W, int64_t ldw,
                      double* __restrict__ s_out, double* __restrict__ inv_s, Control* ctrl,
                      int loop_mode, LoopStep loop, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    __shared__ int perm[2 * kMaxPairs];
    __shared__ double sv[2 * kMaxPairs];
    __shared__ int first_bad;
    __shared__ int all_small;
    __shared__ double floor2_s;
    const int tid = threadIdx.x;
    if (tid == 0) {
        first_bad = l;
        all_small = 1;
    }
    __syncthreads();
    for (int i = tid; i < l; i += blockDim.x) {
        perm[i] = i;
        if (!(lam[i] == lam[i])) first_bad = 0;  // NaN: reported as NumericalError below
    }
    __syncthreads();
    if (first_bad == 0) {
        if (tid == 0) {
            if (ctrl->status == DSVD_OK) ctrl->status = DSVD_NUMERICAL;
            ctrl->stopped = 1;
        }
        return;
    }
    __syncthreads();
    // descending order; ties keep the reverse of the stable ascending order
    for (int i = tid; i < l; i += blockDim.x) {
        const double li = lam[i];
        int rank = 0;
        for (int j = 0; j < l; ++j) {
            const double lj = lam[j];
            rank += (lj > li) || (lj == li && j > i);
        }
        perm[rank] = i;
    }
    __syncthreads();
    if (tid == 0) {
        const double lmax = fmax(lam[perm[0]], 0.0);
        const double fl = static_cast<double>(rows > l ? rows : l) * DBL_EPSILON * sqrt(lmax);
        floor2_s = fl * fl;
    }
    __syncthreads();
    for (int r = tid; r < l; r += blockDim.x) {
        const double lr = lam[perm[r]];
        if (!(lr > floor2_s)) atomicMin(&first_bad, r);  // NaN also lands here
    }
    __syncthreads();
    if (first_bad < l) {
        if (tid == 0) {
            const double lr = lam[perm[first_bad]];
            if (ctrl->status == DSVD_OK) {
                ctrl->status = (lr == lr) ? DSVD_RANK_DEFICIENT : DSVD_NUMERICAL;
                ctrl->status_index = first_bad;
            }
            ctrl->stopped = 1;
        }
        return;
    }
    for (int r = tid; r < l; r += blockDim.x) {
        const int src = perm[r];
        const double s = sqrt(lam[src]);
        sv[r] = s;
        s_out[r] = s;
        inv_s[r] = 1.0 / s;
        double lead = 0.0;
        for (int t = 0; t < l; ++t) {
            const double x = vecs[static_cast<int64_t>(t) * lp + src];
            if (x != 0.0) {
                lead = x;
                break;
            }
        }
        const bool flip = lead < 0.0;
        for (int t = 0; t < l; ++t) {
            const double x = vecs[static_cast<int64_t>(t) * lp + src];
            W[static_cast<int64_t>(t) * ldw + r] = flip ? -x : x;
        }
    }
    if (!loop_mode) return;
    __syncthreads();
    // ---- power-loop bookkeeping, solver.cpp:97-112 -----------------------
    const int64_t j = ctrl->iteration + 1;
    const double alpha = ctrl->alpha;
    if (j - 1 < loop.cap) {
        if (tid == 0 && loop.alphas) loop.alphas[j - 1] = alpha;
        if (loop.s_hat)
            for (int r = tid; r < l; r += blockDim.x) loop.s_hat[(j - 1) * l + r] = sv[r];
    }
    if (loop.alg == DSVD_ALG_BASIC) {  // basic_core: trace only, no shift (solver.cpp:130-136)
        if (tid == 0) ctrl->iteration = j;
        return;
    }
    bool stop = false;
    if (loop.alg == DSVD_ALG_DASH) {
        // pve_stop_check(s_stored, alpha_stored, s, alpha, k, tol): operand order as written
        const double denom = sv[loop.k] + alpha;
        const double ap = ctrl->alpha_stored;
        for (int i = tid; i < loop.k; i += blockDim.x) {
            const double change = fabs(loop.s_stored[i] + ap - sv[i] - alpha);
            if (!(change / denom <= loop.tol)) all_small = 0;
        }
        __syncthreads();
        stop = all_small != 0;
    }
    __syncthreads();
    if (stop) {
        if (tid == 0) {
            ctrl->iteration = j;
            ctrl->stop_pending = 1;
        }
        return;
    }
    for (int r = tid; r < l; r += blockDim.x) loop.s_stored[r] = sv[r];
    if (tid == 0) {
        double a = alpha;
        if (loop.alg != DSVD_ALG_FIXED_SHIFT || j == 1) {
            const double s_ll = sv[l - 1];
            a = s_ll > a ? (s_ll + a) / 2.0 : a;  // update_shift
        }
        ctrl->alpha = a;
        ctrl->alpha_stored = a;
        ctrl->iteration = j;
    }
}

__global__ void sym_finish_kernel(const double* __restrict__ lam, const double* __restrict__ vecs,
                                  int l, int lp, double* __restrict__ values,
                                  double* __restrict__ vectors) {
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        const double li = lam[i];
        int rank = 0;
        for (int j = 0; j < l; ++j) {
            const double lj = lam[j];
            rank += (lj < li) || (lj == li && j < i);
        }
        values[rank] = li;
        for (int t = 0; t < l; ++t)
            vectors[static_cast<int64_t>(rank) * l + t] = vecs[static_cast<int64_t>(t) * lp + i];
    }
}

__global__ void loop_begin_kernel(Control* ctrl) {
    if (ctrl->stop_pending) ctrl->stopped = 1;
}

__global__ void control_init_kernel(Control* ctrl, double* s_stored, int l) {
    for (int i = threadIdx.x; i < l; i += blockDim.x) s_stored[i] = 0.0;
    if (threadIdx.x == 0) {
        ctrl->alpha = 0.0;
        ctrl->alpha_stored = 0.0;
        ctrl->iteration = 0;
        ctrl->status_index = -1;
        ctrl->total_sweeps = 0;
        ctrl->stopped = 0;
        ctrl->stop_pending = 0;
        ctrl->status = DSVD_OK;
        ctrl->status_src = 0;
        ctrl->eig_sweeps = 0;
    }
}

int padded_order(int l) { return (l + 1) & ~1; }

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t eig_workspace_bytes(int l, int max_sweeps) {
    const size_t lp = padded_order(l);
    const size_t half = lp / 2;
    return al(sizeof(double) * lp * lp) + al(sizeof(double2) * max_sweeps * (lp - 1) * half) +
           al(sizeof(double) * lp) + al(sizeof(double) * lp * lp);
}

void eig_workspace_bind(EigWorkspace& w, int l, int max_sweeps, void* mem) {
    w.l = l;
    w.lp = padded_order(l);
    w.max_sweeps = max_sweeps;
    const size_t lp = w.lp, half = lp / 2;
    char* p = static_cast<char*>(mem);
    w.gbuf = reinterpret_cast<double*>(p);
    p += al(sizeof(double) * lp * lp);
    w.rot_log = reinterpret_cast<double2*>(p);
    p += al(sizeof(double2) * max_sweeps * (lp - 1) * half);
    w.lam = reinterpret_cast<double*>(p);
    p += al(sizeof(double) * lp);
    w.vecs = reinterpret_cast<double*>(p);
}

void jacobi_eig(const double* g, EigWorkspace& w, Control* ctrl, const int32_t* gate,
                cudaStream_t stream, const int32_t* need) {
    if (w.lp > 2 * kMaxPairs) fail(DSVD_UNSUPPORTED, "eigensolver: l > 512 is not supported");
    const size_t csmem = cluster_smem_bytes(w.lp);
    if (csmem <= static_cast<size_t>(kSmemLimit) - 12 * 1024 && w.lp >= 4) {
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(jacobi_cluster_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(csmem)));
        jacobi_cluster_kernel<<<2, kEigThreads, csmem, stream>>>(g, w.l, w.lp, w.max_sweeps, w.lam,
                                                                 w.vecs, ctrl, gate, need);
        DSVD_LAUNCH_CHECK();
        return;
    }
    const size_t half = w.lp / 2;
    const size_t table = sizeof(uint16_t) * half * (half + 1) / 2;
    const size_t gbytes = sizeof(double) * w.lp * w.lp;
    const int use_smem = gbytes + table <= static_cast<size_t>(kSmemLimit) - 16 * 1024;
    const size_t smem = (use_smem ? gbytes : 0) + table;
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemLimit - 16 * 1024));
    jacobi_kernel<<<1, kEigThreads, smem, stream>>>(
        g, w.l, w.lp, w.gbuf, use_smem, w.rot_log, w.max_sweeps, w.lam, ctrl, gate, need);
    DSVD_LAUNCH_CHECK();
    const int warps = 8;
    jacobi_replay_kernel<<<static_cast<unsigned>(ceil_div(w.lp, warps)), 32 * warps,
                           sizeof(double) * warps * w.lp, stream>>>(w.rot_log, w.l, w.lp, ctrl,
                                                                    w.vecs, gate, need);
    DSVD_LAUNCH_CHECK();
}

void eig_svd_finish(const EigWorkspace& w, int64_t rows, double* W, int64_t ldw, double* s,
                    double* inv_s, Control* ctrl, const LoopStep* loop, const int32_t* gate,
                    cudaStream_t stream) {
    LoopStep ls;
    if (loop) ls = *loop;
    eig_svd_finish_kernel<<<1, kFinishThreads, 0, stream>>>(w.lam, w.vecs, w.l, w.lp, rows, W, ldw,
                                                            s, inv_s, ctrl, loop ? 1 : 0, ls, gate);
    DSVD_LAUNCH_CHECK();
}

void sym_eig_finish(const EigWorkspace& w, double* values, double* vectors_colmajor,
                    cudaStream_t stream) {
    sym_finish_kernel<<<1, 256, 0, stream>>>(w.lam, w.vecs, w.l, w.lp, values, vectors_colmajor);
    DSVD_LAUNCH_CHECK();
}

__global__ void trace_basic_kernel(Control* ctrl, double* alphas, int64_t cap) {
    const int64_t j = ctrl->iteration + 1;
    if (alphas != nullptr && j - 1 < cap) alphas[j - 1] = 0.0;
    ctrl->iteration = j;
}

void trace_basic_iteration(Control* ctrl, double* alphas, int64_t cap, cudaStream_t stream) {
    trace_basic_kernel<<<1, 1, 0, stream>>>(ctrl, alphas, cap);
    DSVD_LAUNCH_CHECK();
}

void loop_begin(Control* ctrl, cudaStream_t stream) {
    loop_begin_kernel<<<1, 1, 0, stream>>>(ctrl);
    DSVD_LAUNCH_CHECK();
}

void control_init(Control* ctrl, double* s_stored, int l, cudaStream_t stream) {
    control_init_kernel<<<1, 256, 0, stream>>>(ctrl, s_stored, l);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
