// Microbenchmark: random row gathers (warp loads one 8*W-byte row slab per
// index) from an X of `rows` x 152 doubles, all SMs. Reports GB/s of gathered
// bytes for an L2-resident and a DRAM-sized X.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void gather(const double* __restrict__ x, const int* __restrict__ idx, long n, int ld,
                       double* out) {
    const int lane = threadIdx.x & 31;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double2 acc = make_double2(0, 0);
    for (long p = w * 32; p < n; p += nw * 32) {
        int c = idx[p + lane];
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
            int cj = __shfl_sync(0xffffffff, c, j);
            double2 v = __ldg(reinterpret_cast<const double2*>(x + (long)cj * ld) + lane);
            acc.x += v.x; acc.y += v.y;
        }
    }
    if (acc.x == 12345.0) out[0] = acc.y;
}
int main() {
    const int ld = 152;
    const long n = 1 << 24;
    int* idx; cudaMalloc(&idx, n * 4);
    double* out; cudaMalloc(&out, 8);
    for (long rows : {40000L, 200000L, 2000000L}) {
        double* x; cudaMalloc(&x, rows * ld * 8); cudaMemset(x, 0, rows * ld * 8);
        int* h = new int[n]; uint64_t s = 88172645463325252ull;
        for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % rows; }
        cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice); delete[] h;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int blocks : {148 * 8, 148 * 16, 148 * 32}) {
            gather<<<blocks, 256>>>(x, idx, n, ld, out);
            cudaEventRecord(a); gather<<<blocks, 256>>>(x, idx, n, ld, out); cudaEventRecord(b);
            cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
            printf("X %7.1f MB, blocks %5d: %.1f GB/s of 512-B gathers (%.3f ms)\n", rows * ld * 8 / 1e6,
                   blocks, n * 512.0 / ms / 1e6, ms);
        }
        cudaFree(x);
    }
    return 0;
}
