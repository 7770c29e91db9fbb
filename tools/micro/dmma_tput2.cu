// DMMA m8n8k4 f64 throughput variants: accumulator count, fresh A/B operand
// registers per DMMA (loaded from shared memory), warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}
template <int ACC, bool LOAD>
__global__ void k(double* out, int n) {
    __shared__ double sm[32 * 64];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) sm[i] = i * 1e-3;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double2 c[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = make_double2(0, 0);
    double a = sm[lane], b = sm[lane + 32];
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) {
            if (LOAD) {
                a = sm[(i & 7) * 64 + lane];
                b = sm[((i + 3) & 7) * 64 + 32 + lane];
            }
            dmma(c[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i].x + c[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ACC, bool LOAD>
void run(double* out, int warps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int n = 2000;
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k<ACC, LOAD><<<148, 32 * warps>>>(out, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const double dm = double(n) * ACC * warps * 148;
    printf("acc %2d %s warps/SM %2d: %.1f TF/s (%.1f cycles per DMMA per SMSP at 1.965 GHz)\n", ACC,
           LOAD ? "smem operands" : "reg operands ", warps, dm * 512 / ms / 1e9,
           ms * 1e-3 * 1.965e9 / (dm / (148 * 4)));
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * 8);
    for (int w : {4, 8, 16}) {
        run<8, false>(out, w);
        run<8, true>(out, w);
        run<20, false>(out, w);
        run<20, true>(out, w);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
