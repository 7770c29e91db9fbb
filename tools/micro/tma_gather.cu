// Microbenchmark: TMA tile::gather4 throughput on sm_100a.
// One producer thread per CTA streams random row indices into gather4 copies
// (box = W doubles x 1 row, 4 rows per instruction) through an S-stage ring of
// 32-row stages; one consumer warp waits for each stage and releases it.
// Reports bytes/s for one CTA and for the whole chip (2 CTAs/SM).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void expect(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, unsigned ph) {
    asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* m, int c, int4 r, uint64_t* b) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(su(dst)), "l"((uint64_t)m), "r"(c), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su(b)) : "memory");
}

template <int W, int S, int LANES>
__global__ void __launch_bounds__(64) bench(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                            int nstage, double* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    double* data = (double*)sm;
    uint64_t* full = (uint64_t*)(data + S * 32 * W);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { init(&full[s], 1); init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;\nfence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int* my = idx + (size_t)blockIdx.x * nstage * 32;
    double acc = 0;
    if (warp == 0) {
        for (int st = 0; st < nstage; ++st) {
            const int s = st % S;
            wait(&empty[s], ((st / S) & 1) ^ 1);
            if (lane == 0) expect(&full[s], 32 * W * 8);
            __syncwarp();
            if (lane < 8) {
                const int per = 8 / LANES;
                if (lane % per == 0 || LANES == 8)
                    for (int g = lane; g < lane + (LANES == 8 ? 1 : per); ++g) {
                        int4 r = ((const int4*)(my + st * 32))[g];
                        g4(data + (s * 32 + 4 * g) * W, &map, 0, r, &full[s]);
                    }
            }
        }
    } else {
        for (int st = 0; st < nstage; ++st) {
            const int s = st % S;
            wait(&full[s], (st / S) & 1);
            acc += data[(s * 32 + (lane & 31)) * W];
            __syncwarp();
            if (lane == 0) arrive(&empty[s]);
        }
        if (acc == 1234.5) out[0] = acc;
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const long rows = 200000, ld = 152;
    double* x;
    cudaMalloc(&x, rows * ld * 8);
    cudaMemset(x, 0, rows * ld * 8);
    const int nstage = 2000, maxcta = 296;
    std::vector<int> h((size_t)maxcta * nstage * 32);
    uint64_t s = 88172645463325252ull;
    for (auto& v : h) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; v = s % rows; }
    int* idx;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, 8);
    auto run = [&](auto kern, int W, int S, const char* name) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows}, str[1] = {(cuuint64_t)ld * 8};
        cuuint32_t box[2] = {(cuuint32_t)W, 1}, es[2] = {1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        size_t smem = (size_t)S * 32 * W * 8 + 2 * S * 8 + 64;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int ctas : {1, 148, 296}) {
            kern<<<ctas, 64, smem>>>(m, idx, nstage, out);
            cudaEventRecord(a);
            kern<<<ctas, 64, smem>>>(m, idx, nstage, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double bytes = (double)ctas * nstage * 32 * W * 8;
            printf("%-22s W=%3d S=%2d ctas=%3d: %8.1f GB/s  (%.1f cycles/row per CTA @1.965GHz) err=%s\n", name, W, S,
                   ctas, bytes / ms / 1e6, ms * 1.965e6 / (nstage * 32.0), cudaGetErrorString(cudaGetLastError()));
        }
    };
    run(bench<64, 6, 8>, 64, 6, "8 lanes issue");
    run(bench<64, 6, 1>, 64, 6, "1 lane issues all");
    run(bench<64, 12, 8>, 64, 12, "8 lanes, 12 stages");
    run(bench<32, 12, 8>, 32, 12, "8 lanes, W32 S12");
    run(bench<32, 24, 8>, 32, 24, "8 lanes, W32 S24");
    run(bench<128, 5, 8>, 128, 5, "8 lanes, W128 S5");
    run(bench<152, 4, 8>, 152, 4, "8 lanes, W152 S4");
    return 0;
}
