// Microbenchmark for a "flat stream" column-slab SpMM pass: the rows of the real
// C4 matrix (kernel order: longest first, empty rows dropped) are cut into runs
// of ~T consecutive nonzeros at row boundaries; a 16-lane group walks its run's
// (index, value) stream contiguously with a rolling gather pipeline (U = 2
// 512-byte gathers in flight per lane), keeps the row's FMA chain in CSR order,
// and writes the row's 64-column slab at each row end (row-end flag in bit 30 of
// the index, output row from the run's row list). One 64-column slab of a
// slab-major X; compared with the same kernel doing one row per group.
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

constexpr int G = 16, WARPS = 8;
constexpr unsigned kEnd = 1u << 30;

// one run per group: stream [rs[r], rs[r+1]), its rows' output ids from rid[rr[r] ...]
template <int U, int MB>
__global__ void __launch_bounds__(256, MB) flat_kernel(const double* __restrict__ x, const int* __restrict__ idx,
                                                      const double* __restrict__ val, const int64_t* __restrict__ rs,
                                                      const int* __restrict__ rr, const int* __restrict__ rid,
                                                      int nruns, double* __restrict__ y) {
    const int lane = threadIdx.x & 31, g = lane / G, t = lane % G;
    const int run = (blockIdx.x * WARPS + (threadIdx.x >> 5)) * 2 + g;
    if (run >= nruns) return;
    const int64_t p0 = rs[run], p1 = rs[run + 1];
    int k = rr[run];
    const double* xc = x + 4 * t;
    double acc[4] = {0, 0, 0, 0};
    double xa[U][4], va[U];
    unsigned ca[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (p0 + u < p1) {
            ca[u] = static_cast<unsigned>(idx[p0 + u]);
            va[u] = val[p0 + u];
            ld256(xc + static_cast<int64_t>(ca[u] & (kEnd - 1)) * 64, xa[u]);
        }
    }
    for (int64_t p = p0; p < p1; p += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = p + u;
            if (q < p1) {
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] = fma(va[u], xa[u][j], acc[j]);
                if (ca[u] & kEnd) {
                    double* o = y + static_cast<int64_t>(rid[k]) * 64 + 4 * t;
                    *reinterpret_cast<double2*>(o) = make_double2(acc[0], acc[1]);
                    *reinterpret_cast<double2*>(o + 2) = make_double2(acc[2], acc[3]);
                    acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
                    ++k;
                }
                const int64_t qn = q + U;
                if (qn < p1) {
                    ca[u] = static_cast<unsigned>(idx[qn]);
                    va[u] = val[qn];
                    ld256(xc + static_cast<int64_t>(ca[u] & (kEnd - 1)) * 64, xa[u]);
                }
            }
        }
    }
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
    std::vector<int> sidx;
    std::vector<double> sval;
    std::vector<int> rid;
    sidx.reserve(nnz);
    sval.reserve(nnz);
    for (int r : order) {
        const int64_t b = off[r], e = off[r + 1];
        if (b == e) continue;
        for (int64_t p = b; p < e; ++p) {
            sidx.push_back(static_cast<int>(idx[p]) | (p + 1 == e ? static_cast<int>(kEnd) : 0));
            sval.push_back(val[p]);
        }
        rid.push_back(r);
    }
    const int64_t S = static_cast<int64_t>(sidx.size());
    for (int T : {64}) {
        // runs at row boundaries, ~T nonzeros each (long rows become single runs)
        std::vector<int64_t> rs{0};
        std::vector<int> rr{0};
        int64_t acc = 0;
        int krow = 0;
        for (int64_t p = 0; p < S; ++p) {
            ++acc;
            if (sidx[p] & kEnd) {
                ++krow;
                if (acc >= T) {
                    rs.push_back(p + 1);
                    rr.push_back(krow);
                    acc = 0;
                }
            } else if (acc >= 512) {  // a long row: cut into 512-nonzero pieces (the product's chunks)
                rs.push_back(p + 1);
                rr.push_back(krow);
                acc = 0;
            }
        }
        if (rs.back() != S) {
            rs.push_back(S);
            rr.push_back(krow);
        }
        const int nruns = static_cast<int>(rs.size()) - 1;
        int *d_idx, *d_rr, *d_rid;
        double *d_val, *x, *y;
        int64_t* d_rs;
        cudaMalloc(&d_idx, S * 4);
        cudaMalloc(&d_val, S * 8);
        cudaMalloc(&d_rs, rs.size() * 8);
        cudaMalloc(&d_rr, rr.size() * 4);
        cudaMalloc(&d_rid, rid.size() * 4);
        cudaMalloc(&x, rows * 64 * 8);
        cudaMalloc(&y, rows * 64 * 8);
        cudaMemset(x, 0, rows * 64 * 8);
        cudaMemcpy(d_idx, sidx.data(), S * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(d_val, sval.data(), S * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(d_rs, rs.data(), rs.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(d_rr, rr.data(), rr.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(d_rid, rid.data(), rid.size() * 4, cudaMemcpyHostToDevice);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int blocks = (nruns + 2 * WARPS - 1) / (2 * WARPS);
        auto time = [&](auto kern, const char* name) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(a);
                kern<<<blocks, 32 * WARPS>>>(x, d_idx, d_val, d_rs, d_rr, d_rid, nruns, y);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("T=%5d runs %8d %-14s: one 64-column slab %.3f ms (%.2f TB/s gathered), x5 slabs = %.1f ms per pass\n",
                   T, nruns, name, best, S * 512.0 / best / 1e9, 5 * best);
        };
        time(flat_kernel<2, 4>, "U=2 32 warps");
        time(flat_kernel<4, 4>, "U=4 32 warps");
        time(flat_kernel<4, 3>, "U=4 24 warps");
        time(flat_kernel<8, 2>, "U=8 16 warps");
        time(flat_kernel<8, 3>, "U=8 24 warps");
        cudaFree(d_idx); cudaFree(d_val); cudaFree(d_rs); cudaFree(d_rr); cudaFree(d_rid); cudaFree(x); cudaFree(y);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
