// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) kernels for the two dense
// products of every power iteration (eigSVD, decompositions.cpp:52-73):
//
//   gram_dmma    G = C^T C for row-major C (n x l): one warp per 4x4 tile of
//                8x8 blocks on and above the diagonal (16 DMMAs per 8 fragment
//                loads per 4-row k-step); C is staged 32 rows at a time by
//                cp.async; per-CTA partial triangles are summed in a fixed
//                order (deterministic, not the reference's single FMA chain;
//                the eigensolver is not bitwise either).
//   rescale_dmma out = C (W diag(scale)) for the 150-wide tall-skinny blocks:
//                CTA tile 128 rows x 32 columns, the W column block resident
//                in shared memory (pre-transposed, scale folded in), C staged
//                16 k at a time through a 4-deep cp.async ring with an XOR
//                swizzle so every fragment load is one conflict-free LDS.128.
//
// B200 runs DMMA and DFMA at the same peak (~37 TFLOP/s measured,
// tools/micro/dmma_tput.cu) but one DMMA carries 256 FMAs, which leaves issue
// slots for the operand loads; the register-tiled DFMA kernels these replace
// reached ~26% of the FP64 pipe.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dense.cuh"

namespace dsvd {

namespace {

__device__ __forceinline__ void dmma884(double2& d, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d.x), "+d"(d.y)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa16z(void* dst, const void* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
// 2-D TMA tile load (box of the tensor map at column x, row y) into shared memory
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
}
// 1-D bulk copy global -> shared (bytes a multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(su32(bar))
        : "memory");
}

// ---- rescale ----------------------------------------------------------------------
constexpr int kRsBM = 128, kRsBN = 32, kRsBK = 16, kRsStages = 4, kRsThreads = 256;
constexpr int kRsMaxK = 320;  // W block (32 x (K+8)) + the ring fit in shared memory

// wt[nn][k] = (k < K && nn < ncol) ? w[k][nn] * scale[nn] : 0, nn < npad, k < ldb
__global__ void rescale_prep_kernel(const double* __restrict__ w, int64_t ldw, const double* __restrict__ scale,
                                    int K, int ncol, int npad, int ldb, double* __restrict__ wt,
                                    const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < npad * ldb; e += gridDim.x * blockDim.x) {
        const int nn = e / ldb, k = e - nn * ldb;
        double v = 0.0;
        if (k < K && nn < ncol) v = w[static_cast<int64_t>(k) * ldw + nn] * (scale != nullptr ? scale[nn] : 1.0);
        wt[e] = v;
    }
}

template <bool kPeers>
__global__ void __launch_bounds__(kRsThreads, 2)
rescale_dmma_kernel(const double* __restrict__ c, int64_t n, int K, int64_t ldc, const double* __restrict__ wt,
                    int ldb, int ncol, double* __restrict__ out, int64_t ld_out, int out_colmajor,
                    const int32_t* __restrict__ gate, double* __restrict__ out2, int out2_w,
                   const PeerOut peers) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ __align__(16) double rsm[];
    double* Bt = rsm;                // [32][ldb]: W block, transposed
    double* As = rsm + kRsBN * ldb;  // [stages][128][16], 8-double halves XOR-swizzled by row parity
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int j0 = blockIdx.x * kRsBN;
    const int nk = (K + kRsBK - 1) / kRsBK;
    const int64_t nrb = (n + kRsBM - 1) / kRsBM;
    for (int e = tid; e < kRsBN * ldb / 2; e += kRsThreads)
        cpa16z(Bt + 2 * e, wt + static_cast<int64_t>(j0) * ldb + 2 * e, true);
    cpa_commit();
    for (int64_t rb = blockIdx.y; rb < nrb; rb += gridDim.y) {
        const int64_t r0 = rb * kRsBM;
        auto load_a = [&](int slot, int kc) {
            double* dst = As + slot * (kRsBM * kRsBK);
            const int k0 = kc * kRsBK;
            for (int e = tid; e < kRsBM * (kRsBK / 2); e += kRsThreads) {
                const int r = e >> 3, ch = e & 7;
                const int64_t gr = r0 + r;
                const int k = k0 + 2 * ch;
                const bool ok = gr < n && k < ldc;
                double* d = dst + r * kRsBK + ((((ch >> 2) ^ (r & 1)) << 3) | ((2 * ch) & 7));
                cpa16z(d, ok ? c + gr * ldc + k : c, ok);
            }
        };
        for (int s = 0; s < kRsStages - 1; ++s) {
            if (s < nk) load_a(s, s);
            cpa_commit();
        }
        double2 acc[2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
        for (int kc = 0; kc < nk; ++kc) {
            cpa_wait<kRsStages - 2>();
            __syncthreads();
            const int pf = kc + kRsStages - 1;
            if (pf < nk) load_a(pf % kRsStages, pf);
            cpa_commit();
            const double* A = As + (kc % kRsStages) * (kRsBM * kRsBK);
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                double2 af[2], bf[4];
#pragma unroll
                for (int mb = 0; mb < 2; ++mb) {
                    const int r = warp * 16 + mb * 8 + g;
                    af[mb] = *reinterpret_cast<const double2*>(A + r * kRsBK + ((p ^ (r & 1)) << 3) + 2 * q);
                }
                const int kg = kc * kRsBK + p * 8 + 2 * q;
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
                    bf[nb] = *reinterpret_cast<const double2*>(Bt + (nb * 8 + g) * ldb + kg);
                // the two k-halves of each accumulator are eight DMMAs apart
#pragma unroll
                for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) dmma884(acc[mb][nb], af[mb].x, bf[nb].x);
#pragma unroll
                for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) dmma884(acc[mb][nb], af[mb].y, bf[nb].y);
            }
        }
        cpa_wait<0>();
        __syncthreads();  // the ring is reused by the next row block
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
            const int64_t r = r0 + warp * 16 + mb * 8 + g;
            if (r >= n) continue;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const int j = j0 + nb * 8 + 2 * q;
                const double2 v = acc[mb][nb];
                if (out_colmajor) {
                    if (j < ncol) out[static_cast<int64_t>(j) * n + r] = v.x;
                    if (j + 1 < ncol) out[static_cast<int64_t>(j + 1) * n + r] = v.y;
                } else if (j + 1 < ld_out) {
                    *reinterpret_cast<double2*>(out + r * ld_out + j) = v;
                    if (out2 != nullptr)  // the slab-major copy (j even: j, j + 1 share a slab)
                        *reinterpret_cast<double2*>(out2 + ((j / out2_w) * n + r) * out2_w + j % out2_w) = v;
#pragma unroll
                    for (int pp = 0; pp < kMaxPeerOut; ++pp)  // the other ranks' copies of these rows
                        if (kPeers && pp < peers.n) *reinterpret_cast<double2*>(peers.p[pp] + r * ld_out + j) = v;
                } else if (j < ld_out) {
                    out[r * ld_out + j] = v.x;
                    if (out2 != nullptr) out2[((j / out2_w) * n + r) * out2_w + j % out2_w] = v.x;
#pragma unroll
                    for (int pp = 0; pp < kMaxPeerOut; ++pp)
                        if (kPeers && pp < peers.n) peers.p[pp][r * ld_out + j] = v.x;
                }
            }
        }
    }
}

// One 16-deep k chunk of a warp's 16 x 32 tile (2 x NB 8x8 DMMA tiles), the C
// chunk in the TMA ring's 128-byte-swizzled layout.
template <int NB>
__device__ __forceinline__ void rs_ksteps(const double* A, const double* Bt, int ldb, int kc, int warp, int g, int q,
                                          double2 (&acc)[2][4]) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        double2 af[2], bf[4];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
            const int r = warp * 16 + mb * 8 + g;
            af[mb] = *reinterpret_cast<const double2*>(A + r * kRsBK + (((4 * p + q) ^ (r & 7)) << 1));
        }
        const int kg = kc * kRsBK + p * 8 + 2 * q;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) bf[nb] = *reinterpret_cast<const double2*>(Bt + (nb * 8 + g) * ldb + kg);
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) dmma884(acc[mb][nb], af[mb].x, bf[nb].x);
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) dmma884(acc[mb][nb], af[mb].y, bf[nb].y);
    }
}

// TMA-fed variant: one thread streams the C tiles (128 rows x 16 k, 128-byte
// swizzle) into a kRsStages ring with mbarriers and bulk-copies the W block;
// fragment addresses follow the swizzle (16-byte chunk c of row r lives at
// chunk c ^ (r & 7)). Removes the per-thread cp.async address arithmetic,
// which was ~45% of the issued instructions of rescale_dmma_kernel.
template <int ST, bool kPeers>
__global__ void __launch_bounds__(kRsThreads, 2)
rescale_tma_kernel(const __grid_constant__ CUtensorMap cmap, int64_t n, int K, const double* __restrict__ wt,
                   int ldb, int ncol, double* __restrict__ out, int64_t ld_out, int out_colmajor,
                   const int32_t* __restrict__ gate, double* __restrict__ out2, int out2_w,
                   const PeerOut peers) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ __align__(1024) unsigned char rsm_raw[];
    // 1024-byte aligned ring first (128B-swizzle requirement), then W, then barriers
    double* As = reinterpret_cast<double*>(rsm_raw + ((1024 - (su32(rsm_raw) & 1023)) & 1023));
    double* Bt = As + ST * kRsBM * kRsBK;
    uint64_t* full = reinterpret_cast<uint64_t*>(Bt + kRsBN * ldb);
    uint64_t* wbar = full + ST;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int j0 = blockIdx.x * kRsBN;
    const int nk = (K + kRsBK - 1) / kRsBK;
    const int64_t nrb = (n + kRsBM - 1) / kRsBM;
    constexpr unsigned kTileBytes = kRsBM * kRsBK * sizeof(double);
    const int width = out_colmajor ? ncol : static_cast<int>(ld_out);
    const int nbv = min(4, (width - j0 + 7) / 8);  // 8-column tiles with columns in range
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) bar_init(&full[s], 1);
        bar_init(wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned wbytes = static_cast<unsigned>(kRsBN * ldb * sizeof(double));
        bar_expect_tx(wbar, wbytes);
        bulk_load(Bt, wt + static_cast<int64_t>(j0) * ldb, wbytes, wbar);
    }
    bar_wait(wbar, 0);
    unsigned use = 0;  // chunks consumed so far (ring position and mbarrier phase)
    for (int64_t rb = blockIdx.y; rb < nrb; rb += gridDim.y) {
        const int y0 = static_cast<int>(rb * kRsBM);
        if (tid == 0) {
            for (int s = 0; s < ST - 1 && s < nk; ++s) {
                const unsigned slot = (use + s) % ST;
                bar_expect_tx(&full[slot], kTileBytes);
                tma_load_2d(As + slot * (kRsBM * kRsBK), &cmap, s * kRsBK, y0, &full[slot]);
            }
        }
        double2 acc[2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
        for (int kc = 0; kc < nk; ++kc, ++use) {
            __syncthreads();  // every warp is done with the slot refilled below
            if (tid == 0 && kc + ST - 1 < nk) {
                const unsigned slot = (use + ST - 1) % ST;
                bar_expect_tx(&full[slot], kTileBytes);
                tma_load_2d(As + slot * (kRsBM * kRsBK), &cmap, (kc + ST - 1) * kRsBK, y0, &full[slot]);
            }
            const unsigned slot = use % ST;
            bar_wait(&full[slot], (use / ST) & 1);
            const double* A = As + slot * (kRsBM * kRsBK);
            // the last column block forms only its in-range 8-column tiles
            if (nbv == 4) rs_ksteps<4>(A, Bt, ldb, kc, warp, g, q, acc);
            else if (nbv == 3) rs_ksteps<3>(A, Bt, ldb, kc, warp, g, q, acc);
            else if (nbv == 2) rs_ksteps<2>(A, Bt, ldb, kc, warp, g, q, acc);
            else rs_ksteps<1>(A, Bt, ldb, kc, warp, g, q, acc);
        }
        const int64_t r0 = rb * kRsBM;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
            const int64_t r = r0 + warp * 16 + mb * 8 + g;
            if (r >= n) continue;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const int j = j0 + nb * 8 + 2 * q;
                const double2 v = acc[mb][nb];
                if (out_colmajor) {
                    if (j < ncol) out[static_cast<int64_t>(j) * n + r] = v.x;
                    if (j + 1 < ncol) out[static_cast<int64_t>(j + 1) * n + r] = v.y;
                } else if (j + 1 < ld_out) {
                    *reinterpret_cast<double2*>(out + r * ld_out + j) = v;
                    if (out2 != nullptr)  // the slab-major copy (j even: j, j + 1 share a slab)
                        *reinterpret_cast<double2*>(out2 + ((j / out2_w) * n + r) * out2_w + j % out2_w) = v;
#pragma unroll
                    for (int pp = 0; pp < kMaxPeerOut; ++pp)  // the other ranks' copies of these rows
                        if (kPeers && pp < peers.n) *reinterpret_cast<double2*>(peers.p[pp] + r * ld_out + j) = v;
                } else if (j < ld_out) {
                    out[r * ld_out + j] = v.x;
                    if (out2 != nullptr) out2[((j / out2_w) * n + r) * out2_w + j % out2_w] = v.x;
#pragma unroll
                    for (int pp = 0; pp < kMaxPeerOut; ++pp)
                        if (kPeers && pp < peers.n) peers.p[pp][r * ld_out + j] = v.x;
                }
            }
        }
    }
}

// 2-D tensor map over a row-major (rows x ld) fp64 block: box of 16 columns x
// 128 rows, 128-byte swizzle, out-of-range elements read as zero.
CUtensorMap make_cmap(const double* c, int64_t rows, int64_t ld) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (encode == nullptr) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        DSVD_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
        if (fn == nullptr || qr != cudaDriverEntryPointSuccess) fail(DSVD_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    CUtensorMap map;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * sizeof(double))};
    const cuuint32_t box[2] = {kRsBK, kRsBM};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(c), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(DSVD_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return map;
}

// ---- gram -------------------------------------------------------------------------
// 1: skip the DMMAs of padding / below-diagonal 8x8 blocks (predicated per warp).
// Measured on C4: the predicated issue made the wide Gram slower (596 vs 538 ms
// per solve), so it is off.
constexpr int kGramSkip = 0;
constexpr int kGmRows = 32, kGmStages = 4;

__host__ __device__ constexpr int gm_pairs(int nb) { return nb * (nb + 1) / 2; }
__device__ __forceinline__ int gm_tri(int a, int j, int nb) { return a * nb - a * (a - 1) / 2 + (j - a); }

// 4x4 register-blocked Gram: the 8x8-block grid (padded to NB4*4 blocks) is
// covered by NB4(NB4+1)/2 tiles of 4x4 blocks on and above the diagonal, one
// warp each; per 4-row k-step a warp loads 8 fragments (4 on diagonal tiles)
// for 16 DMMAs.
// Row stride of the staged block: 2 * stride == 8 (mod 32) banks, so the four
// rows (q = lane & 3) of a half-warp's 64-bit fragment loads hit distinct banks
__host__ __device__ constexpr int gm4_stride(int nb4) { return 32 * nb4 + 4; }

template <int NB4>
__global__ void __launch_bounds__(32 * NB4 * (NB4 + 1) / 2, NB4 >= 5 ? 1 : (NB4 == 4 ? 2 : (NB4 == 3 ? 3 : 4)))
gram_dmma_kernel(const double* __restrict__ c, int64_t n, int64_t ld, int nb, int64_t rows_per_block,
                 double* __restrict__ partial, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    constexpr int S = gm4_stride(NB4);
    extern __shared__ __align__(16) double gsm[];  // [stages][kGmRows][S]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    int I = 0, t = warp;  // tile (I, J), I <= J, row-major over the upper triangle
    while (t >= NB4 - I) {
        t -= NB4 - I;
        ++I;
    }
    const int J = I + t;
    const int64_t r_beg = static_cast<int64_t>(blockIdx.x) * rows_per_block;
    const int64_t r_end = min(n, r_beg + rows_per_block);
    const int vec = static_cast<int>(ld / 2);
    // columns [ld, S) are never written by cp.async: zero them once
    for (int e = tid; e < kGmStages * kGmRows * (S - 2 * vec); e += blockDim.x) {
        const int row = e / (S - 2 * vec), col = 2 * vec + e % (S - 2 * vec);
        gsm[row * S + col] = 0.0;
    }
    const int nwarp = blockDim.x >> 5;
    auto stage = [&](int slot, int64_t rr0) {  // warp per row, lanes along the row
        double* dst = gsm + slot * kGmRows * S;
        for (int r = warp; r < kGmRows; r += nwarp) {
            const int64_t gr = rr0 + r;
            const bool ok = gr < r_end;
            const double* src = c + (ok ? gr * ld : 0);
            for (int v = lane; v < vec; v += 32) cpa16z(dst + r * S + 2 * v, src + 2 * v, ok);
        }
    };
    const int nst = static_cast<int>(((r_end > r_beg ? r_end - r_beg : int64_t(0)) + kGmRows - 1) / kGmRows);
    for (int st = 0; st < kGmStages - 1; ++st) {
        if (st < nst) stage(st, r_beg + st * kGmRows);
        cpa_commit();
    }
    double2 acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = make_double2(0.0, 0.0);
    const bool diag = I == J;
    // 8x8 blocks this warp must form: inside the nb x nb grid and on or above
    // the diagonal (diagonal tiles skip their 6 lower blocks, padding tiles the
    // blocks past nb): DMMA issue slots the other warps of the SM get instead
    // (NB4 >= 5 only: the smaller instances have no registers to spare for it)
    unsigned live = NB4 >= 5 ? 0u : 0xffffu;
    if (NB4 >= 5) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (4 * I + u < nb && 4 * J + v < nb && (!diag || u <= v)) live |= 1u << (4 * u + v);
    }
    for (int st = 0; st < nst; ++st) {
        cpa_wait<kGmStages - 2>();
        __syncthreads();
        const int pf = st + kGmStages - 1;
        if (pf < nst) stage(pf % kGmStages, r_beg + static_cast<int64_t>(pf) * kGmRows);
        cpa_commit();
        const double* C = gsm + (st % kGmStages) * kGmRows * S;
#pragma unroll 2
        for (int ks = 0; ks < kGmRows / 4; ++ks) {
            const double* row = C + (4 * ks + q) * S + g;
            double fa[4], fb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) fa[u] = row[8 * (4 * I + u)];
            if (diag) {
#pragma unroll
                for (int v = 0; v < 4; ++v) fb[v] = fa[v];
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) fb[v] = row[8 * (4 * J + v)];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    if (kGramSkip == 0 || (live & (1u << (4 * u + v)))) dmma884(acc[u][v], fa[u], fb[v]);
        }
    }
    cpa_wait<0>();
    double* out = partial + static_cast<int64_t>(blockIdx.x) * gm_pairs(nb) * 64;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int bi = 4 * I + u, bj = 4 * J + v;
            if (bi <= bj && bj < nb)
                *reinterpret_cast<double2*>(out + gm_tri(bi, bj, nb) * 64 + g * 8 + 2 * q) = acc[u][v];
        }
}

// G(i, j) = G(j, i) = sum over CTAs of the partial block entry: 256 threads per
// 8x8 block, four interleaved partial sums combined in a fixed order.
__global__ void __launch_bounds__(256)
gram_dmma_reduce_kernel(const double* __restrict__ partial, int nblk, int nb, int64_t l, double* __restrict__ g,
                        const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    __shared__ double red[4][64];
    const int t = blockIdx.x, npair = nb * (nb + 1) / 2;
    const int w = threadIdx.x & 63, part = threadIdx.x >> 6;
    double s0 = 0.0, s1 = 0.0;
    int bb = part;
    for (; bb + 4 < nblk; bb += 8) {
        s0 += partial[(static_cast<int64_t>(bb) * npair + t) * 64 + w];
        s1 += partial[(static_cast<int64_t>(bb + 4) * npair + t) * 64 + w];
    }
    if (bb < nblk) s0 += partial[(static_cast<int64_t>(bb) * npair + t) * 64 + w];
    red[part][w] = s0 + s1;
    __syncthreads();
    if (part != 0) return;
    const double s = (red[0][w] + red[1][w]) + (red[2][w] + red[3][w]);
    int ta = 0, rem = t;
    while (rem >= nb - ta) {
        rem -= nb - ta;
        ++ta;
    }
    const int64_t i = 8 * ta + w / 8, j = 8 * (ta + rem) + w % 8;
    if (i >= l || j >= l || i > j) return;
    g[i * l + j] = s;
    g[j * l + i] = s;
}

// Wide Gram (l > 160, e.g. C4's l = 300): the 32-column strips are split in
// two halves H0 = [0, h), H1 = [h, NS); a CTA "kind" is the triangle of 4x4
// tiles inside one half, or a piece of the H0 x H1 rectangle at most 16 tiles
// big (one warp per tile, 16 warps), so the kinds carry near-equal tile counts
// (C4: 15, 15, 15, 10). A CTA (kind, row slab) stages only the columns of its
// one or two strip segments. blockIdx.x (the kind) varies fastest so the CTAs
// of one slab share it in L2. Same partial layout as gram_dmma_kernel (one
// triangle of 8x8 blocks per slab).
constexpr int kGwRows = 32, kGwStages = 3, kGwStride = 260;  // 2 * 260 == 8 (mod 32) banks: conflict-free
constexpr int kGwMaxKinds = 8;

struct GwKinds {
    int8_t sa0[kGwMaxKinds], sa1[kGwMaxKinds], sb0[kGwMaxKinds], sb1[kGwMaxKinds];
};

// One stage (kGwRows rows) of a warp's 4x4 tile of 8x8 blocks: fragment loads
// and the DMMAs of the blocks the tile shape forms (kDiag: u <= v only; NV
// block columns in range).
template <bool kDiag, int NV>
__device__ __forceinline__ void gw_ksteps(const double* C, int q, int g, int ia, int jb, double2 (&acc)[4][4]) {
#pragma unroll
    for (int ks = 0; ks < kGwRows / 4; ++ks) {
        const double* row = C + (4 * ks + q) * kGwStride + g;
        double fa[4], fb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (!kDiag || u < NV) fa[u] = row[ia + 8 * u];
#pragma unroll
        for (int v = 0; v < NV; ++v) fb[v] = row[jb + 8 * v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (!kDiag || u <= v) dmma884(acc[u][v], fa[u], fb[v]);
    }
}

__global__ void __launch_bounds__(512, 1)
gram_dmma_wide_kernel(const double* __restrict__ c, int64_t n, int64_t ld, int nb, int64_t rows_per_block,
                      const GwKinds kinds, double* __restrict__ partial, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ __align__(16) double wsm[];  // [stages][kGwRows][kGwStride]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int kd = blockIdx.x;
    const int sa0 = kinds.sa0[kd], nA = kinds.sa1[kd] - sa0, sb0 = kinds.sb0[kd], nB = kinds.sb1[kd] - sb0;
    const bool tri = nB == 0;
    int I, J;
    bool active;
    if (tri) {  // upper triangle of the nA x nA strip tiles, row-major
        int t = warp, i = 0;
        while (i < nA && t >= nA - i) {
            t -= nA - i;
            ++i;
        }
        active = i < nA;
        I = sa0 + i;
        J = sa0 + i + t;
    } else {
        active = warp < nA * nB;
        I = sa0 + warp / max(nB, 1);
        J = sb0 + warp % max(nB, 1);
    }
    const int64_t r_beg = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t r_end = min(n, r_beg + rows_per_block);
    // staging: 32 rows x up to 128 16-byte chunks per stage, eight per thread
    // at rows (tid >> 7) + 4u of one fixed chunk (addresses set up once)
    const int ch = tid & 127, r0t = tid >> 7;
    const int64_t col = ch < 16 * nA ? 32 * sa0 + 2 * ch : 32 * sb0 + 2 * (ch - 16 * nA);
    const bool col_ok = ch < 16 * (nA + nB) && col < ld;
    const double* src0 = c + (col_ok ? col : 0);
    double* dst0 = wsm + r0t * kGwStride + 2 * ch;
    auto stage = [&](int slot, int64_t rr0) {
        double* dst = dst0 + slot * kGwRows * kGwStride;
#pragma unroll
        for (int u = 0; u < kGwRows / 4; ++u) {
            const int64_t gr = rr0 + r0t + 4 * u;
            const bool ok = col_ok && gr < r_end;
            cpa16z(dst + 4 * u * kGwStride, ok ? src0 + gr * ld : c, ok);
        }
    };
    const int nst = static_cast<int>(((r_end > r_beg ? r_end - r_beg : int64_t(0)) + kGwRows - 1) / kGwRows);
    for (int st = 0; st < kGwStages - 1; ++st) {
        if (st < nst) stage(st, r_beg + st * kGwRows);
        cpa_commit();
    }
    double2 acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = make_double2(0.0, 0.0);
    const int ia = 32 * (I - sa0), jb = tri ? 32 * (J - sa0) : 32 * (nA + J - sb0);
    // (Forming only the in-range, on-or-above-diagonal 8x8 blocks of each tile —
    // predicated DMMAs, or per-shape DMMA sequences — was measured on C4 and did
    // not shorten the kernel: 553 vs 552 ms per solve.)
    for (int st = 0; st < nst; ++st) {
        cpa_wait<kGwStages - 2>();
        __syncthreads();
        const int pf = st + kGwStages - 1;
        if (pf < nst) stage(pf % kGwStages, r_beg + static_cast<int64_t>(pf) * kGwRows);
        cpa_commit();
        if (!active) continue;
        const double* C = wsm + (st % kGwStages) * kGwRows * kGwStride;
        gw_ksteps<false, 4>(C, q, g, ia, jb, acc);
    }
    cpa_wait<0>();
    if (!active) return;
    double* out = partial + static_cast<int64_t>(blockIdx.y) * gm_pairs(nb) * 64;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int bi = 4 * I + u, bj = 4 * J + v;
            if (bi <= bj && bj < nb)
                *reinterpret_cast<double2*>(out + gm_tri(bi, bj, nb) * 64 + g * 8 + 2 * q) = acc[u][v];
        }
}

// Wide Gram, 2x2 tiles: the same kinds-of-CTA scheme as gram_dmma_wide_kernel,
// but over 16-column tiles of 2x2 8x8 blocks, up to four tiles per warp
// (tiles w, w + 16, w + 32, w + 48 of the kind). At l = 300 (38 blocks, 19 tiles)
// the 190 tiles on and above the diagonal issue 741 block products per k-step,
// every one of them useful (the 4x4 tiles issue 880: 320-column padding and the
// lower halves of the diagonal tiles). Kind encoding as GwKinds, in tile units.
constexpr int kGw2Tiles = 4;  // tiles per warp
#ifndef DSVD_GW2_UNROLL
#define DSVD_GW2_UNROLL 8
#endif
constexpr int kGw2Unroll = DSVD_GW2_UNROLL;  // k-steps unrolled in gw2_ksteps (C4 Gram per solve: 2 -> 274.5 ms, 4 -> 272.5, 8 -> 269.4; profiles/r02_ab_gw2_unroll.txt)

// One stage (kGwRows rows) of a warp's NT 2x2 tiles: per k-step four fragment
// loads and four DMMAs per tile
template <int NT>
__device__ __forceinline__ void gw2_ksteps(const double* C, int q, int g, const int (&ia)[kGw2Tiles],
                                           const int (&jb)[kGw2Tiles], double2 (&acc)[kGw2Tiles][2][2]) {
#pragma unroll kGw2Unroll
    for (int ks = 0; ks < kGwRows / 4; ++ks) {
        const double* row = C + (4 * ks + q) * kGwStride + g;
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const double fa0 = row[ia[s]], fa1 = row[ia[s] + 8];
            const double fb0 = row[jb[s]], fb1 = row[jb[s] + 8];
            dmma884(acc[s][0][0], fa0, fb0);
            dmma884(acc[s][1][0], fa1, fb0);
            dmma884(acc[s][0][1], fa0, fb1);
            dmma884(acc[s][1][1], fa1, fb1);
        }
    }
}

__global__ void __launch_bounds__(512, 1)
gram_dmma_wide2_kernel(const double* __restrict__ c, int64_t n, int64_t ld, int nb, int64_t rows_per_block,
                       const GwKinds kinds, double* __restrict__ partial, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ __align__(16) double wsm[];  // [stages][kGwRows][kGwStride]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int kd = blockIdx.x;
    const int a0 = kinds.sa0[kd], nA = kinds.sa1[kd] - a0, b0 = kinds.sb0[kd], nB = kinds.sb1[kd] - b0;
    const bool tri = nB == 0;
    const int ntile = tri ? nA * (nA + 1) / 2 : nA * nB;
    // this warp's tiles: global tile coordinates, staged column offsets
    int ia[kGw2Tiles], jb[kGw2Tiles], ti[kGw2Tiles], tj[kGw2Tiles];
    bool has[kGw2Tiles];
#pragma unroll
    for (int s = 0; s < kGw2Tiles; ++s) {
        const int t = warp + 16 * s;
        has[s] = t < ntile;
        int i = 0, j = 0;
        if (tri) {
            int r = t;
            while (i < nA && r >= nA - i) {
                r -= nA - i;
                ++i;
            }
            j = i + r;
        } else {
            i = t / max(nB, 1);
            j = t % max(nB, 1);
        }
        if (!has[s]) i = j = 0;  // (an absent slot before the last would compute tile (0, 0) unused)
        ti[s] = a0 + i;
        tj[s] = tri ? a0 + j : b0 + j;
        ia[s] = 16 * i;
        jb[s] = tri ? 16 * j : 16 * (nA + j);
    }
    const int ntw = (ntile > warp) ? min(kGw2Tiles, (ntile - warp + 15) / 16) : 0;  // tiles of this warp
    const int64_t r_beg = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t r_end = min(n, r_beg + rows_per_block);
    // staging as gram_dmma_wide_kernel: 32 rows x up to 128 16-byte chunks
    const int ch = tid & 127, r0t = tid >> 7;
    const int64_t col = ch < 8 * nA ? 16 * a0 + 2 * ch : 16 * b0 + 2 * (ch - 8 * nA);
    const bool col_ok = ch < 8 * (nA + nB) && col < ld;
    const double* src0 = c + (col_ok ? col : 0);
    double* dst0 = wsm + r0t * kGwStride + 2 * ch;
    auto stage = [&](int slot, int64_t rr0) {
        double* dst = dst0 + slot * kGwRows * kGwStride;
#pragma unroll
        for (int u = 0; u < kGwRows / 4; ++u) {
            const int64_t gr = rr0 + r0t + 4 * u;
            const bool ok = col_ok && gr < r_end;
            cpa16z(dst + 4 * u * kGwStride, ok ? src0 + gr * ld : c, ok);
        }
    };
    const int nst = static_cast<int>(((r_end > r_beg ? r_end - r_beg : int64_t(0)) + kGwRows - 1) / kGwRows);
    for (int st = 0; st < kGwStages - 1; ++st) {
        if (st < nst) stage(st, r_beg + st * kGwRows);
        cpa_commit();
    }
    double2 acc[kGw2Tiles][2][2];
#pragma unroll
    for (int s = 0; s < kGw2Tiles; ++s)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) acc[s][u][v] = make_double2(0.0, 0.0);
    for (int st = 0; st < nst; ++st) {
        cpa_wait<kGwStages - 2>();
        __syncthreads();
        const int pf = st + kGwStages - 1;
        if (pf < nst) stage(pf % kGwStages, r_beg + static_cast<int64_t>(pf) * kGwRows);
        cpa_commit();
        const double* C = wsm + (st % kGwStages) * kGwRows * kGwStride;
        // every tile forms its four block products (a diagonal tile's lower
        // block, 19 of 760 at l = 300, is not stored); one warp-uniform branch
        // per stage on the warp's tile count
        if (ntw == 4) gw2_ksteps<4>(C, q, g, ia, jb, acc);
        else if (ntw == 3) gw2_ksteps<3>(C, q, g, ia, jb, acc);
        else if (ntw == 2) gw2_ksteps<2>(C, q, g, ia, jb, acc);
        else if (ntw == 1) gw2_ksteps<1>(C, q, g, ia, jb, acc);
    }
    cpa_wait<0>();
    double* out = partial + static_cast<int64_t>(blockIdx.y) * gm_pairs(nb) * 64;
#pragma unroll
    for (int s = 0; s < kGw2Tiles; ++s) {
        if (!has[s]) continue;
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int bi = 2 * ti[s] + u, bj = 2 * tj[s] + v;
                if (bi <= bj && bj < nb)
                    *reinterpret_cast<double2*>(out + gm_tri(bi, bj, nb) * 64 + g * 8 + 2 * q) = acc[s][u][v];
            }
    }
}

template <int NB4>
void launch_gram_dmma(const double* c, int64_t n, int64_t ld, int nb, int nblk, int64_t rpb, double* partial,
                      const int32_t* gate, cudaStream_t stream) {
    const size_t smem = sizeof(double) * kGmStages * kGmRows * gm4_stride(NB4);
    DSVD_CUDA_CHECK(cudaFuncSetAttribute(gram_dmma_kernel<NB4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    gram_dmma_kernel<NB4><<<nblk, 32 * NB4 * (NB4 + 1) / 2, smem, stream>>>(c, n, ld, nb, rpb, partial, gate);
    DSVD_LAUNCH_CHECK();
}

struct GramDmmaPlan {
    int nb = 0, nblk = 0;
    int64_t rpb = 0;
};

// CTA kinds of gram_dmma_wide_kernel for NS strips of 32 columns (NS <= 10)
struct GwPlan {
    GwKinds k{};
    int n = 0;
};
GwPlan gw_kinds(int ns) {
    GwPlan p;
    auto add = [&](int a0, int a1, int b0, int b1) {
        p.k.sa0[p.n] = static_cast<int8_t>(a0);
        p.k.sa1[p.n] = static_cast<int8_t>(a1);
        p.k.sb0[p.n] = static_cast<int8_t>(b0);
        p.k.sb1[p.n] = static_cast<int8_t>(b1);
        ++p.n;
    };
    const int h = (ns + 1) / 2;
    add(0, h, 0, 0);
    if (ns > h) add(h, ns, h, h);
    const int cw = std::max(1, 16 / h);
    for (int b0 = h; b0 < ns; b0 += cw) add(0, h, b0, std::min(ns, b0 + cw));
    return p;
}
// CTA kinds of gram_dmma_wide2_kernel for nt 16-column tiles (nt <= 20): the
// two half triangles and the rectangle between them in pieces of at most 64
// tiles whose staged columns fit 256
GwPlan gw2_kinds(int nt) {
    GwPlan p;
    auto add = [&](int a0, int a1, int b0, int b1) {
        p.k.sa0[p.n] = static_cast<int8_t>(a0);
        p.k.sa1[p.n] = static_cast<int8_t>(a1);
        p.k.sb0[p.n] = static_cast<int8_t>(b0);
        p.k.sb1[p.n] = static_cast<int8_t>(b1);
        ++p.n;
    };
    const int h = (nt + 1) / 2;
    add(0, h, 0, 0);
    if (nt > h) add(h, nt, h, h);
    const int cw = std::max(1, std::min(16 * kGw2Tiles / h, 16 - h));
    for (int b0 = h; b0 < nt; b0 += cw) add(0, h, b0, std::min(nt, b0 + cw));
    return p;
}
int gram_wide_tiles = 2;  // 2: gram_dmma_wide2_kernel (default), 4: gram_dmma_wide_kernel
int gram_wide_waves = 24;  // CTAs of the wide Gram: about this many per SM (C4: 6 -> 24 = 519 -> 485 ms per solve)
constexpr int kGramNarrowMaxNb = 20;  // gram_dmma_kernel<NB4 <= 5>: l <= 160
constexpr int kGramWideMaxNb = 40;    // gram_dmma_wide_kernel: l <= 320 (<= 10 strips)

GramDmmaPlan gram_dmma_plan(int64_t n, int64_t l) {
    GramDmmaPlan p;
    p.nb = static_cast<int>((l + 7) / 8);
    if (p.nb > kGramNarrowMaxNb) {
        // wide: kinds x slabs, ~6 waves of one CTA per SM
        const int nkinds = gram_wide_tiles == 2 ? gw2_kinds((p.nb + 1) / 2).n : gw_kinds((p.nb + 3) / 4).n;
        p.nblk = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(gram_wide_waves * kNumSMs, nkinds), ceil_div(n, 8 * kGwRows))));
        p.rpb = ceil_div(ceil_div(n, p.nblk), kGwRows) * kGwRows;
        p.nblk = static_cast<int>(std::max<int64_t>(1, ceil_div(n, p.rpb)));
        return p;
    }
    const int nb4 = (p.nb + 3) / 4;  // CTAs per SM as in the launch bounds
    p.nblk = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(kNumSMs * (nb4 >= 5 ? 1 : (nb4 == 4 ? 2 : (nb4 == 3 ? 3 : 4))), ceil_div(n, 64))));
    p.rpb = ceil_div(ceil_div(n, p.nblk), kGmRows) * kGmRows;
    p.nblk = static_cast<int>(std::max<int64_t>(1, ceil_div(n, p.rpb)));
    return p;
}

}  // namespace

void set_gram_wide_tiles(int t) { gram_wide_tiles = t == 4 ? 4 : 2; }
void set_gram_wide_waves(int w) { gram_wide_waves = w < 1 ? 1 : w; }

bool gram_dmma_supported(int64_t l, int64_t ld) {
    return l >= 1 && (l + 7) / 8 <= kGramWideMaxNb && ld % 2 == 0 && ld >= l;
}

size_t gram_dmma_workspace_bytes(int64_t n, int64_t l) {
    const GramDmmaPlan p = gram_dmma_plan(n, l);
    return sizeof(double) * static_cast<size_t>(p.nblk) * gm_pairs(p.nb) * 64;
}

void gram_dmma(const double* c, int64_t n, int64_t l, int64_t ld, double* g, void* ws, const int32_t* gate,
               cudaStream_t stream) {
    const GramDmmaPlan p = gram_dmma_plan(n, l);
    double* partial = static_cast<double*>(ws);
    if (p.nb > kGramNarrowMaxNb) {
        const bool t2 = gram_wide_tiles == 2;
        const GwPlan kp = t2 ? gw2_kinds((p.nb + 1) / 2) : gw_kinds((p.nb + 3) / 4);
        const size_t smem = sizeof(double) * kGwStages * kGwRows * kGwStride;
        auto kern = t2 ? gram_dmma_wide2_kernel : gram_dmma_wide_kernel;
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        const dim3 grid(static_cast<unsigned>(kp.n), static_cast<unsigned>(p.nblk));
        kern<<<grid, 512, smem, stream>>>(c, n, ld, p.nb, p.rpb, kp.k, partial, gate);
        DSVD_LAUNCH_CHECK();
        gram_dmma_reduce_kernel<<<gm_pairs(p.nb), 256, 0, stream>>>(partial, p.nblk, p.nb, l, g, gate);
        DSVD_LAUNCH_CHECK();
        return;
    }
    switch ((p.nb + 3) / 4) {
        case 1: launch_gram_dmma<1>(c, n, ld, p.nb, p.nblk, p.rpb, partial, gate, stream); break;
        case 2: launch_gram_dmma<2>(c, n, ld, p.nb, p.nblk, p.rpb, partial, gate, stream); break;
        case 3: launch_gram_dmma<3>(c, n, ld, p.nb, p.nblk, p.rpb, partial, gate, stream); break;
        case 4: launch_gram_dmma<4>(c, n, ld, p.nb, p.nblk, p.rpb, partial, gate, stream); break;
        case 5: launch_gram_dmma<5>(c, n, ld, p.nb, p.nblk, p.rpb, partial, gate, stream); break;
        default: fail(DSVD_OTHER, "gram_dmma: unsupported width");
    }
    gram_dmma_reduce_kernel<<<gm_pairs(p.nb), 256, 0, stream>>>(partial, p.nblk, p.nb, l, g, gate);
    DSVD_LAUNCH_CHECK();
}

bool rescale_use_tma = true;
int64_t rescale_max_row_ctas = 4096;  // grid.y cap: CTAs loop over row blocks beyond it (C4: 815 -> 798 ms per solve vs 65535: one W load per CTA serves 8 row blocks)
void set_rescale_row_ctas(int64_t c) { rescale_max_row_ctas = c < 1 ? 1 : std::min<int64_t>(c, 65535); }

bool rescale_dmma_supported(int64_t K, int64_t ldc, int64_t ld_out, int out_colmajor) {
    return K >= 1 && K <= kRsMaxK && ldc % 2 == 0 && ldc >= K && (out_colmajor || ld_out % 2 == 0);
}

size_t rescale_dmma_workspace_bytes(int64_t K, int64_t width) {
    const int64_t kpad = ceil_div(K, kRsBK) * kRsBK;
    const int64_t ldb = kpad + 8;
    return sizeof(double) * static_cast<size_t>(ceil_div(width, kRsBN) * kRsBN * ldb);
}

void rescale_dmma(const double* c, int64_t n, int64_t K, int64_t ldc, const double* w, int64_t ldw,
                  const double* scale, int64_t ncol, double* out, int64_t ld_out, int out_colmajor, void* ws,
                  const int32_t* gate, cudaStream_t stream, double* out2, int out2_w, const PeerOut* peers) {
    if (out2 != nullptr && (out_colmajor || out2_w <= 0 || out2_w % 2 != 0)) fail(DSVD_OTHER, "rescale: bad second output");
    PeerOut po{};
    if (peers != nullptr) {
        if (out_colmajor || peers->n > kMaxPeerOut) fail(DSVD_OTHER, "rescale: bad peer outputs");
        po = *peers;
    }
    if (n == 0) return;
    const int64_t width = out_colmajor ? ncol : ld_out;
    const int ncb = static_cast<int>(ceil_div(width, kRsBN));
    const int ldb = static_cast<int>(ceil_div(K, kRsBK) * kRsBK + 8);  // == 8 (mod 16): conflict-free B loads
    double* wt = static_cast<double*>(ws);
    const int npad = ncb * kRsBN;
    rescale_prep_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(npad) * ldb, 256)), 256, 0, stream>>>(
        w, ldw, scale, static_cast<int>(K), static_cast<int>(ncol), npad, ldb, wt, gate);
    DSVD_LAUNCH_CHECK();
    const int64_t nrb = ceil_div(n, kRsBM);
    const dim3 grid(static_cast<unsigned>(ncb), static_cast<unsigned>(std::min<int64_t>(nrb, rescale_max_row_ctas)));
    const bool tma = rescale_use_tma && (reinterpret_cast<uintptr_t>(c) % 16) == 0 && (ldc * 8) % 16 == 0;
    if (tma) {
        // K > 160: a 2-deep ring keeps two CTAs per SM (the W block grows with K)
        const int st = K > 160 ? 2 : kRsStages;
        const size_t smem = 1024 + sizeof(double) * (st * kRsBM * kRsBK + static_cast<size_t>(kRsBN) * ldb) +
                            sizeof(uint64_t) * (st + 1);
        auto kern = po.n > 0 ? (st == 2 ? rescale_tma_kernel<2, true> : rescale_tma_kernel<kRsStages, true>)
                             : (st == 2 ? rescale_tma_kernel<2, false> : rescale_tma_kernel<kRsStages, false>);
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        const CUtensorMap cmap = make_cmap(c, n, ldc);
        kern<<<grid, kRsThreads, smem, stream>>>(cmap, n, static_cast<int>(K), wt, ldb, static_cast<int>(ncol), out,
                                                 ld_out, out_colmajor, gate, out2, out2_w, po);
    } else {
        const size_t smem = sizeof(double) * (static_cast<size_t>(kRsBN) * ldb + kRsStages * kRsBM * kRsBK);
        auto kd = po.n > 0 ? rescale_dmma_kernel<true> : rescale_dmma_kernel<false>;
        DSVD_CUDA_CHECK(cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem)));
        kd<<<grid, kRsThreads, smem, stream>>>(c, n, static_cast<int>(K), ldc, wt, ldb,
                                                                static_cast<int>(ncol), out, ld_out, out_colmajor,
                                                                gate, out2, out2_w, po);
    }
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
