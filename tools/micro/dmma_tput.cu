// Microbenchmark: FP64 tensor-core (mma.sync m8n8k4 f64) vs DFMA throughput
// on sm_100a, whole GPU, cycles + wall time.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int ACC>
__global__ void mma_loop(double* out, int n) {
    double a = out[threadIdx.x] + 1.0, b = a * 0.5;
    double c[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fma_loop(double* out, int n) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = out[threadIdx.x] + i;
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999, 1e-3);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 1024 * 8);
    cudaMemset(out, 0, 148 * 8 * 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 20000;
    for (int warps : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            mma_loop<8><<<148 * 2, 32 * warps / 2>>>(out, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * double(n) * 148 * warps;
        printf("DMMA m8n8k4, %2d warps/SM, 8 acc: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            fma_loop<<<148 * 2, 32 * warps / 2>>>(out, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * 32 * double(n) * 148 * warps;
        printf("DFMA,          %2d warps/SM, 8 chains: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
