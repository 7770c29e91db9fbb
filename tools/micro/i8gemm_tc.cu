// Harness for a hand-written tcgen05 INT8 GEMM (the building block of an
// Ozaki-style FP64 emulation): C[M x N] (int32) = A[M x K] * B[N x K]^T with
// int8 A, B both K-major in global memory, TMA (128-byte swizzle) into a
// 2-stage shared-memory ring, one elected thread issuing
// tcgen05.mma.cta_group::1.kind::i8 into a TMEM accumulator (128 lanes x N
// columns), four warps draining it with tcgen05.ld. Checks exactness against
// a CPU GEMM and reports the throughput.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e = (x);                                                                       \
        if (e != cudaSuccess) {                                                                    \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
            exit(1);                                                                               \
        }                                                                                          \
    } while (0)

constexpr int BM = 128, BK = 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t sdesc(const void* smem) {
    const uint64_t addr = su32(smem);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor: s32 accumulate, s8 x s8, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

template <int BN, int STAGES, int MINB>
__global__ void __launch_bounds__(128, MINB)
i8gemm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int K,
              int32_t* __restrict__ C, int ldc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
    uint8_t* sa = base;                       // [STAGES][BM][BK]
    uint8_t* sb = base + STAGES * BM * BK;    // [STAGES][BN][BK]
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * BN * BK);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    __shared__ uint32_t tmem_base_sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    constexpr uint32_t kCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : BN <= 256 ? 256 : 512;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_sh)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    const int nk = K / BK;
    if (warp == 0 && lane == 0) {  // TMA producer
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
            mbar_expect_tx(&full[s], (BM + BN) * BK);
            tma2d(sa + s * BM * BK, &amap, kb * BK, m0, &full[s]);
            tma2d(sb + s * BN * BK, &bmap, kb * BK, n0, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {  // MMA issuer
        constexpr uint32_t id = idesc_i8(BM, BN);
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t ad = sdesc(sa + s * BM * BK), bd = sdesc(sb + s * BN * BK);
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk) {
                const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                // advance the start address by 32 bytes of K per step (2 x 16-byte units)
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(id), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&empty[s]))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(done))
                     : "memory");
    }
    __syncwarp();
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: warp w reads TMEM lanes 32w .. 32w + 31 (= C rows), 8 columns per load
    const int row = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; ++j) C[static_cast<int64_t>(row) * ldc + n0 + c0 + j] = static_cast<int32_t>(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static CUtensorMap map_i8(const int8_t* ptr, int64_t rows, int64_t K, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K)};
    const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("tensor map encode failed %d\n", r);
        exit(1);
    }
    return m;
}

template <int BN, int STAGES = 2, int MINB = 1>
static void run(int M, int N, int K, bool check) {
    std::vector<int8_t> ha(static_cast<size_t>(M) * K), hb(static_cast<size_t>(N) * K);
    uint64_t s = 12345;
    auto rnd = [&] {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return static_cast<int8_t>(static_cast<int>(s % 129) - 64);  // digits in [-64, 64]
    };
    for (auto& x : ha) x = rnd();
    for (auto& x : hb) x = rnd();
    int8_t *da, *db;
    int32_t* dc;
    CK(cudaMalloc(&da, ha.size()));
    CK(cudaMalloc(&db, hb.size()));
    CK(cudaMalloc(&dc, sizeof(int32_t) * M * N));
    CK(cudaMemcpy(da, ha.data(), ha.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb.data(), hb.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dc, 0, sizeof(int32_t) * M * N));
    const CUtensorMap am = map_i8(da, M, K, BM), bm = map_i8(db, N, K, BN);
    const size_t smem = 1024 + STAGES * (BM + BN) * BK + 64;
    CK(cudaFuncSetAttribute(i8gemm_kernel<BN, STAGES, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    dim3 grid(M / BM, N / BN);
    i8gemm_kernel<BN, STAGES, MINB><<<grid, 128, smem>>>(am, bm, K, dc, N);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (check) {
        std::vector<int32_t> hc(static_cast<size_t>(M) * N);
        CK(cudaMemcpy(hc.data(), dc, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost));
        long bad = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                int32_t acc = 0;
                for (int k = 0; k < K; ++k) acc += static_cast<int32_t>(ha[(size_t)i * K + k]) * hb[(size_t)j * K + k];
                if (acc != hc[(size_t)i * N + j]) {
                    if (bad < 5) printf("  mismatch (%d,%d): %d vs %d\n", i, j, hc[(size_t)i * N + j], acc);
                    ++bad;
                }
            }
        printf("check M=%d N=%d K=%d BN=%d: %ld mismatches\n", M, N, K, BN, bad);
    } else {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            i8gemm_kernel<BN, STAGES, MINB><<<grid, 128, smem>>>(am, bm, K, dc, N);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("perf M=%d N=%d K=%d BN=%d stages=%d ctas/SM=%d: %.3f ms, %.1f TOPS (int8 MAC = 2 ops)\n", M, N, K,
               BN, STAGES, MINB, best,
               2.0 * M * N * K / best / 1e9);
    }
    cudaFree(da);
    cudaFree(db);
    cudaFree(dc);
}

int main() {
    run<64>(128, 64, 128, true);
    run<64>(256, 128, 512, true);
    run<128>(512, 256, 1024, true);
    run<256>(256, 256, 384, true);
    run<128, 4, 2>(512, 256, 1024, true);
    run<256, 3, 2>(512, 512, 1024, true);
    run<256>(18944, 256, 8192, false);
    run<128>(18944, 256, 8192, false);
    run<128, 4, 1>(18944, 512, 8192, false);
    run<128, 4, 2>(18944, 512, 8192, false);
    run<256, 3, 1>(18944, 512, 8192, false);
    run<256, 3, 2>(18944, 512, 8192, false);
    run<256, 4, 1>(37888, 512, 8192, false);
    run<128, 6, 1>(37888, 512, 8192, false);
    return 0;
}
