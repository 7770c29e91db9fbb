// Microbenchmark: the real C4 gather stream. The R-MAT scale-22 matrix of
// bench.py's C4 (oracle/inputs_gen.c, seed 4) is flattened into its column
// index sequence in the SpMM kernel's row order (rows by length, longest
// first); 512-byte gathers (16 lanes x LDG.256: one 64-column slab row, two
// rows per warp instruction) replay it from a slab-major 64-column block
// (2.1 GB contiguous), against the same number of i.i.d. draws from the
// matrix's own column distribution (shuffled stream) and from a uniform one.
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <numeric>
#include <cuda_runtime.h>

extern "C" int gen_rmat(int scale, int64_t draws, double a, double b, double c, int uniform, uint64_t seed,
                        int64_t* nnz_out);
extern "C" void gen_fetch(int64_t* off, int64_t* idx, double* val);

__device__ __forceinline__ void ld256(const double* p, double (&r)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

// G lanes per gather of 4*G doubles (G = 16: 512 B), 32/G gathers per instruction, D loads in flight per lane
template <int G, int D>
__global__ void __launch_bounds__(256, 4) gk(const double* __restrict__ x, const int* __restrict__ idx, long n,
                                             double* out) {
    constexpr int R = 32 / G;
    const int lane = threadIdx.x & 31, g = lane / G, t = lane % G;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (long p = w * 32; p < n; p += nw * 32) {
        const int c = idx[p + lane];
#pragma unroll
        for (int j0 = 0; j0 < 32 / R; j0 += D) {
            double r[D][4];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int cj = __shfl_sync(0xffffffff, c, R * (j0 + d) + g);
                ld256(x + (long)cj * (4 * G) + 4 * t, r[d]);
            }
#pragma unroll
            for (int d = 0; d < D; ++d) acc += (r[d][0] + r[d][1]) + (r[d][2] + r[d][3]);
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    int64_t nnz = 0;
    gen_rmat(22, 104000000, 0.57, 0.19, 0.19, 0, 4, &nnz);
    const long rows = 1L << 22;
    std::vector<int64_t> off(rows + 1), idx(nnz);
    std::vector<double> val(nnz);
    gen_fetch(off.data(), idx.data(), val.data());
    std::vector<int> order(rows);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
    const long n = nnz / 32 * 32;
    std::vector<int> seq(nnz), shuf;
    long w = 0;
    for (int r : order)
        for (int64_t p = off[r]; p < off[r + 1]; ++p) seq[w++] = (int)idx[p];
    shuf = seq;
    uint64_t s = 0x9E3779B97F4A7C15ull;
    for (long i = nnz - 1; i > 0; --i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        std::swap(shuf[i], shuf[s % (i + 1)]);
    }
    std::vector<int> uni(nnz);
    for (long i = 0; i < nnz; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; uni[i] = (int)(s % rows); }
    int *d_seq, *d_shuf, *d_uni;
    double *x, *out;
    cudaMalloc(&d_seq, n * 4); cudaMalloc(&d_shuf, n * 4); cudaMalloc(&d_uni, n * 4);
    cudaMemcpy(d_seq, seq.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_shuf, shuf.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_uni, uni.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 8);
    cudaMalloc(&x, rows * 64 * 8);  // one 64-column slab, slab-major
    cudaMemset(x, 0, rows * 64 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, const int* ix, double bytes) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            kern<<<148 * 8, 256>>>(x, ix, n, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-52s %7.3f ms  %6.2f TB/s\n", name, best, n * bytes / best / 1e9);
    };
    printf("nnz %ld, one 64-column slab (%.2f GB), 512 B per gather\n", (long)nnz, rows * 512.0 / 1e9);
    run("real stream, kernel row order, D=2", gk<16, 2>, d_seq, 512.0);
    run("real stream, kernel row order, D=4", gk<16, 4>, d_seq, 512.0);
    run("same indices shuffled, D=2", gk<16, 2>, d_shuf, 512.0);
    run("same indices shuffled, D=4", gk<16, 4>, d_shuf, 512.0);
    run("uniform random rows, D=4", gk<16, 4>, d_uni, 512.0);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
