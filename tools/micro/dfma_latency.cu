// Microbenchmark: dependent DFMA chain latency and issue rate on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, double a, double b, int n, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fma(a, x, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chains4(double* out, double a, double b, int n, long long* cyc) {
    double x0 = out[threadIdx.x], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) { x0 = fma(a, x0, b); x1 = fma(a, x1, b); x2 = fma(a, x2, b); x3 = fma(a, x3, b); }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x0 + x1 + x2 + x3;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1024 * 8); cudaMemset(out, 0, 1024 * 8); cudaMalloc(&cyc, 8);
    const int n = 4096;
    for (int warps : {1, 4, 8, 16, 32}) {
        chain<<<1, 32 * warps>>>(out, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
        chain<<<1, 32 * warps>>>(out, 0.999, 1e-3, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("1 chain/thread, %2d warps: %.2f cycles per dependent DFMA\n", warps, double(h) / (n * 16));
        chains4<<<1, 32 * warps>>>(out, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
        chains4<<<1, 32 * warps>>>(out, 0.999, 1e-3, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("4 chains/thread, %2d warps: %.2f cycles per 4 DFMA step\n", warps, double(h) / (n * 16));
    }
    return 0;
}
