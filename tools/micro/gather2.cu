// Microbenchmark: warp-per-index random row gathers on all SMs, 128-bit vs
// 256-bit loads per lane, uniform vs Zipf(1.1) row popularity, X from
// L1-sized to DRAM-sized. Reports TB/s of gathered bytes.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int V>  // doubles per lane per load: 2 (LDG.128) or 4 (LDG.256)
__global__ void gather(const double* __restrict__ x, const int* __restrict__ idx, long n, int ld, double* out) {
    const int lane = threadIdx.x & 31;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (long p = w * 32; p < n; p += nw * 32) {
        int c = idx[p + lane];
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
            int cj = __shfl_sync(0xffffffff, c, j);
            const double* src = x + (long)cj * ld + V * lane;
            if constexpr (V == 2) {
                double2 v = __ldg(reinterpret_cast<const double2*>(src));
                acc += v.x + v.y;
            } else {
                double a, b, cc, d;
                asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(cc), "=d"(d) : "l"(src));
                acc += (a + b) + (cc + d);
            }
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    const int ld = 152;
    const long n = 1 << 24;
    int* idx;
    cudaMalloc(&idx, n * 4);
    double* out;
    cudaMalloc(&out, 8);
    std::vector<int> h(n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (long rows : {256L, 4000L, 40000L, 100000L, 200000L, 2000000L}) {
        double* x;
        cudaMalloc(&x, rows * ld * 8);
        cudaMemset(x, 0, rows * ld * 8);
        for (int dist = 0; dist < 2; ++dist) {
            uint64_t s = 88172645463325252ull;
            // Zipf(1.1) via inverse CDF on a table
            std::vector<double> cdf;
            if (dist == 1) {
                cdf.resize(rows);
                double t = 0;
                for (long r = 0; r < rows; ++r) cdf[r] = (t += 1.0 / std::pow(r + 1.0, 1.1));
                for (auto& v : cdf) v /= t;
            }
            for (long i = 0; i < n; ++i) {
                s ^= s << 13; s ^= s >> 7; s ^= s << 17;
                if (dist == 0) {
                    h[i] = s % rows;
                } else {
                    double u = (s >> 11) * (1.0 / 9007199254740992.0);
                    long lo = 0, hi = rows - 1;
                    while (lo < hi) { long m = (lo + hi) / 2; if (cdf[m] < u) lo = m + 1; else hi = m; }
                    h[i] = static_cast<int>((lo * 2654435761ull) % rows);  // scatter hot rows
                }
            }
            cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
            for (int v : {2, 4}) {
                float best = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    if (v == 2) gather<2><<<148 * 8, 256>>>(x, idx, n, ld, out);
                    else gather<4><<<148 * 8, 256>>>(x, idx, n, ld, out);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("X %8.1f MB %-7s LDG.%d: %5.1f TB/s (%d B per gather)\n", rows * ld * 8 / 1e6,
                       dist ? "zipf" : "uniform", 64 * v, n * 32.0 * 8 * v / best / 1e9, 32 * 8 * v);
            }
        }
        cudaFree(x);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
