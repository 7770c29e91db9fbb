// Microbenchmark: 256-byte random gathers (8 lanes x LDG.256, four gathers per
// warp instruction, like spmm_slab_kernel<32>) with the R-MAT scale-22 column
// marginal (each of 22 index bits is 1 with probability b + d = 0.24), from
//   (a) a row-major 4.2M x 300 fp64 block (rows 2,400 B apart: the 32-column
//       slab of a whole-row layout, spread over 10 GB),
//   (b) a slab-major copy (rows 256 B apart: the same slab contiguous, 1.07 GB),
//   (c) (a) with the rows relabelled by popularity (hot rows first),
// plus whole 2,400-byte row gathers from (a) for reference. Separates the
// address-layout effects (TLB reach, DRAM page locality) from the L2 hit rate.
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const double* p, double (&r)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

// 8 lanes per gather of 256 B; stride in doubles between rows
__global__ void __launch_bounds__(256, 4) g256(const double* __restrict__ x, const int* __restrict__ idx, long n,
                                               long stride, double* out) {
    const int lane = threadIdx.x & 31, g = lane >> 3, t = lane & 7;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (long p = w * 32; p < n; p += nw * 32) {
        const int c = idx[p + lane];
#pragma unroll
        for (int j0 = 0; j0 < 8; j0 += 2) {
            double r0[4], r1[4];
            const int c0 = __shfl_sync(0xffffffff, c, 4 * j0 + g);
            const int c1 = __shfl_sync(0xffffffff, c, 4 * (j0 + 1) + g);
            ld256(x + (long)c0 * stride + 4 * t, r0);
            ld256(x + (long)c1 * stride + 4 * t, r1);
            acc += (r0[0] + r0[1]) + (r0[2] + r0[3]) + (r1[0] + r1[1]) + (r1[2] + r1[3]);
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

// whole 2,400-byte rows (lanes 0..31 two LDG.256 + lanes 0..10 one LDG.128 ~ spmm_row_wide)
__global__ void __launch_bounds__(256, 2) grow(const double* __restrict__ x, const int* __restrict__ idx, long n,
                                               long stride, double* out) {
    const int lane = threadIdx.x & 31;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (long p = w * 32; p < n; p += nw * 32) {
        const int c = idx[p + lane];
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            const int cj = __shfl_sync(0xffffffff, c, j);
            double r0[4], r1[4];
            ld256(x + (long)cj * stride + 8 * lane, r0);
            ld256(x + (long)cj * stride + 8 * lane + 4, r1);
            double e = 0;
            if (256 + 2 * lane < 300) e = __ldg(x + (long)cj * stride + 256 + 2 * lane);
            acc += (r0[0] + r0[1]) + (r0[2] + r0[3]) + (r1[0] + r1[1]) + (r1[2] + r1[3]) + e;
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    const int scale = 22;
    const long rows = 1L << scale;
    const long n = 1L << 26;  // gathers per launch
    std::vector<int> h(n), hr(n);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    std::vector<long> count(rows, 0);
    for (long i = 0; i < n; ++i) {
        int c = 0;
        for (int b = 0; b < scale; ++b) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            c = (c << 1) | ((s & 0xffff) < 15729 ? 1 : 0);  // 0.24 * 65536
        }
        h[i] = c;
        ++count[c];
    }
    // popularity relabel: hottest row -> 0
    std::vector<int> order(rows), rank(rows);
    for (long r = 0; r < rows; ++r) order[r] = (int)r;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return count[a] > count[b] || (count[a] == count[b] && a < b); });
    for (long r = 0; r < rows; ++r) rank[order[r]] = (int)r;
    for (long i = 0; i < n; ++i) hr[i] = rank[h[i]];
    int *idx, *idxr;
    double *x, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&idxr, n * 4);
    cudaMalloc(&out, 8);
    cudaMalloc(&x, rows * 300 * 8);
    cudaMemset(x, 0, rows * 300 * 8);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(idxr, hr.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, const int* ix, long stride, double bytes_per) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            kern<<<148 * 8, 256>>>(x, ix, n, stride, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-58s %7.3f ms  %6.2f TB/s gathered\n", name, best, n * bytes_per / best / 1e9);
    };
    run("(a) 256 B gathers, rows 2400 B apart (10 GB span)", g256, idx, 300, 256.0);
    run("(b) 256 B gathers, rows 256 B apart (1.07 GB span)", g256, idx, 32, 256.0);
    run("(c) 256 B gathers, 2400 B apart, hot rows relabelled first", g256, idxr, 300, 256.0);
    run("(d) 256 B gathers, 256 B apart, hot rows relabelled first", g256, idxr, 32, 256.0);
    run("(e) whole 2400 B rows (10 GB span)", grow, idx, 300, 2400.0);
    run("(f) whole 2400 B rows, hot rows relabelled first", grow, idxr, 300, 2400.0);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
