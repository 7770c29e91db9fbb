// Microbenchmark: do the FP64 tensor pipe (DMMA m8n8k4) and the FP64 vector
// pipe (DFMA) add up on sm_100a, or is it one set of units?  One CTA per SM of
// 32 warps; the first `mw` warps of every SM sub-partition group issue DMMAs,
// the rest DFMAs.  Prints each side's rate alone and together.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// warps with (warp / 4) < mw4 run DMMA (mw4 warps per sub-partition), the others DFMA;
// n_mma / n_fma = loop counts (0 = that kind of warp exits at once).
__global__ void __launch_bounds__(1024, 1) mix(double* out, int mw4, int n_mma, int n_fma) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if ((warp >> 2) < mw4) {
        double a = out[threadIdx.x] + 1.0, b = a * 0.5;
        double c[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
        for (int it = 0; it < n_mma; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    } else {
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = out[threadIdx.x] + i;
        for (int it = 0; it < n_fma; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999, 1e-3);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += x[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMemset(out, 0, 148 * 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](int mw4, int n_mma, int n_fma) {
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            mix<<<148, 1024>>>(out, mw4, n_mma, n_fma);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        return ms;
    };
    const int n = 40000;
    for (int mw4 : {1, 2, 4}) {
        const int mma_warps = 4 * mw4, fma_warps = 32 - mma_warps;
        const double f_mma = 2.0 * 256 * 8 * double(n) * 148 * mma_warps;
        // give the DFMA warps about the same duration as the DMMA warps alone
        const float t_mma = run(mw4, n, 0);
        const float t_fma1 = run(mw4, 0, n);
        const int n_fma = int(double(n) * t_mma / t_fma1);
        const double f_fma = 2.0 * 8 * 32 * double(n_fma) * 148 * fma_warps;
        const float t_fma = run(mw4, 0, n_fma);
        const float t_both = run(mw4, n, n_fma);
        printf("%2d DMMA warps + %2d DFMA warps per SM: DMMA alone %.1f TF/s (%.2f ms), DFMA alone %.1f TF/s (%.2f ms), "
               "together %.2f ms -> %.1f TF/s combined\n",
               mma_warps, fma_warps, f_mma / t_mma / 1e9, t_mma, f_fma / t_fma / 1e9, t_fma, t_both,
               (f_mma + f_fma) / t_both / 1e9);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
