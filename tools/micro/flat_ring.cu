// Microbenchmark: one 64-column slab pass of the C4 SpMM (the rows at most
// 512 nonzeros long, i.e. the non-split rows, longest first) three ways:
//   row    — the product's structure: one row per 16-lane group, the group's
//            (index, value) batches staged two ahead in a shared-memory ring,
//            U gathers in flight, then the group exits (a new warp per 2 rows);
//   flat   — the same ring and gather pipeline run continuously over a run of
//            ~T nonzeros spanning many rows (persistent groups, runs handed out
//            round-robin so the SMs stay together in stream order); a row-end
//            flag in bit 30 of the index ends the FMA chain and stores the row;
//   replay — the same permuted index stream gathered with no FMAs (ceiling).
// Results of row and flat are compared bitwise.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>
#include <numeric>
#include <cuda_runtime.h>

extern "C" int gen_rmat(int scale, int64_t draws, double a, double b, double c, int uniform, uint64_t seed,
                        int64_t* nnz_out);
extern "C" void gen_fetch(int64_t* off, int64_t* idx, double* val);

__device__ __forceinline__ void ld256(const double* p, double (&r)[4]) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                 : "l"(p));
}

constexpr int G = 16, W = 64, WARPS = 8;
constexpr unsigned kEnd = 1u << 30, kMask = kEnd - 1;

// one row per group of GW = WW / 4 lanes (rows r in [0, nrows): stream [pb[r], pb[r+1])), X slab WW wide
template <int U, int MB, bool kStore = true, bool kFma = true, int WW = 64>
__global__ void __launch_bounds__(256, MB) row_kernel(const double* __restrict__ x, const unsigned* __restrict__ idx,
                                                     const double* __restrict__ val, const int64_t* __restrict__ pb,
                                                     const int* __restrict__ rid, int nrows, double* __restrict__ y) {
    constexpr int GW = WW / 4, RW = 32 / GW;
    __shared__ __align__(16) double2 cv[WARPS][RW][2 * (GW + 1)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / GW, t = lane % GW;
    const int r = (blockIdx.x * WARPS + warp) * RW + g;
    int64_t beg = 0, end = 0;
    if (r < nrows) {
        beg = pb[r];
        end = pb[r + 1];
    }
    const int len = static_cast<int>(end - beg);
    int maxlen = len;
    for (int o = 16; o >= 1; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    const double* xc = x + 4 * t;
    double2* ring = cv[warp][g];
    unsigned cb = 0;
    double vb = 0.0;
    if (t < len) {
        cb = idx[beg + t];
        vb = val[beg + t];
    }
    ring[t] = make_double2(vb, __longlong_as_double(cb));
    cb = 0;
    vb = 0.0;
    if (GW + t < len) {
        cb = idx[beg + GW + t];
        vb = val[beg + GW + t];
    }
    __syncwarp();
    double acc[4] = {0, 0, 0, 0}, xa[U][4], va[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        va[u] = 0.0;
        if (u < len) {
            const double2 e = ring[u];
            va[u] = e.x;
            ld256(xc + static_cast<int64_t>(__double_as_longlong(e.y) & kMask) * WW, xa[u]);
        }
    }
    for (int p = 0; p < maxlen; p += U) {
        if (p % GW == 0) {
            const int b = p / GW;
            __syncwarp();
            ring[((b + 1) & 1) * (GW + 1) + t] = make_double2(vb, __longlong_as_double(cb));
            __syncwarp();
            cb = 0;
            vb = 0.0;
            if ((b + 2) * GW + t < len) {
                cb = idx[beg + (b + 2) * GW + t];
                vb = val[beg + (b + 2) * GW + t];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = p + u;
            if (q < len) {
                if (kFma) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[k] = fma(va[u], xa[u][k], acc[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[k] += xa[u][k];
                }
            }
            const int qn = q + U;
            if (qn < len) {
                const double2 e = ring[((qn / GW) & 1) * (GW + 1) + qn % GW];
                va[u] = e.x;
                ld256(xc + static_cast<int64_t>(__double_as_longlong(e.y) & kMask) * WW, xa[u]);
            }
        }
    }
    if (r >= nrows) return;
    if (!kStore && acc[0] != 12345.0) return;
    double* o = y + static_cast<int64_t>(rid[r]) * WW + 4 * t;
    *reinterpret_cast<double2*>(o) = make_double2(acc[0], acc[1]);
    *reinterpret_cast<double2*>(o + 2) = make_double2(acc[2], acc[3]);
}

// persistent groups over runs: run j = [rs[j], rs[j+1]), its first row rr[j]
template <int U, int MB>
__global__ void __launch_bounds__(256, MB) flat_kernel(const double* __restrict__ x, const unsigned* __restrict__ idx,
                                                      const double* __restrict__ val, const int64_t* __restrict__ rs,
                                                      const int* __restrict__ rr, const int* __restrict__ rid,
                                                      int nruns, double* __restrict__ y) {
    __shared__ __align__(16) double2 cv[WARPS][2][2 * (G + 1)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / G, t = lane % G;
    const int gid = (blockIdx.x * WARPS + warp) * 2 + g, ngroups = gridDim.x * WARPS * 2;
    const double* xc = x + 4 * t;
    double2* ring = cv[warp][g];
    // the warp iterates while either group has a run left
    for (int base = (blockIdx.x * WARPS + warp) * 2; base < nruns; base += ngroups) {
        const int run = base + g;
        int64_t beg = 0, end = 0;
        int k = 0;
        if (run < nruns) {
            beg = rs[run];
            end = rs[run + 1];
            k = rr[run];
        }
        const int len = static_cast<int>(end - beg);
        int maxlen = len;
        for (int o = 16; o >= 1; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
        // output rows of this run, 16 at a time: lane t holds rid[kb + t] (cur) and rid[kb + 16 + t] (next)
        int kb = k;
        int ridc = (run < nruns) ? rid[kb + t] : 0;  // rid is padded by 32 entries
        int ridn = (run < nruns) ? rid[kb + G + t] : 0;
        unsigned cb = 0;
        double vb = 0.0;
        if (t < len) {
            cb = idx[beg + t];
            vb = val[beg + t];
        }
        __syncwarp();
        ring[t] = make_double2(vb, __longlong_as_double(cb));
        cb = 0;
        vb = 0.0;
        if (G + t < len) {
            cb = idx[beg + G + t];
            vb = val[beg + G + t];
        }
        __syncwarp();
        double acc[4] = {0, 0, 0, 0}, xa[U][4], va[U];
        unsigned ca[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            va[u] = 0.0;
            ca[u] = 0;
            if (u < len) {
                const double2 e = ring[u];
                va[u] = e.x;
                ca[u] = static_cast<unsigned>(__double_as_longlong(e.y));
                ld256(xc + static_cast<int64_t>(ca[u] & kMask) * W, xa[u]);
            }
        }
        for (int p = 0; p < maxlen; p += U) {
            if (p % G == 0) {
                const int b = p / G;
                __syncwarp();
                ring[((b + 1) & 1) * (G + 1) + t] = make_double2(vb, __longlong_as_double(cb));
                __syncwarp();
                cb = 0;
                vb = 0.0;
                if ((b + 2) * G + t < len) {
                    cb = idx[beg + (b + 2) * G + t];
                    vb = val[beg + (b + 2) * G + t];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = p + u;
                // (the shuffle outside the divergent row-end branch)
                const int row = __shfl_sync(0xffffffffu, ridc, g * G + (k - kb));
                if (q < len) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = fma(va[u], xa[u][j], acc[j]);
                    if (ca[u] & kEnd) {
                        double* o = y + static_cast<int64_t>(row) * W + 4 * t;
                        *reinterpret_cast<double2*>(o) = make_double2(acc[0], acc[1]);
                        *reinterpret_cast<double2*>(o + 2) = make_double2(acc[2], acc[3]);
                        acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
                        if (++k - kb == G) {
                            kb += G;
                            ridc = ridn;
                            ridn = rid[kb + G + t];
                        }
                    }
                }
                const int qn = q + U;
                if (qn < len) {
                    const double2 e = ring[((qn / G) & 1) * (G + 1) + qn % G];
                    va[u] = e.x;
                    ca[u] = static_cast<unsigned>(__double_as_longlong(e.y));
                    ld256(xc + static_cast<int64_t>(ca[u] & kMask) * W, xa[u]);
                }
            }
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256, 4) replay_kernel(const double* __restrict__ x, const unsigned* __restrict__ idx,
                                                       long n, double* out) {
    const int lane = threadIdx.x & 31, g = lane / G, t = lane % G;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (long p = w * 32; p < n; p += nw * 32) {
        const unsigned c = idx[p + lane] & kMask;
#pragma unroll
        for (int j0 = 0; j0 < 16; j0 += D) {
            double r[D][4];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const unsigned cj = __shfl_sync(0xffffffff, c, 2 * (j0 + d) + g);
                ld256(x + (long)cj * W + 4 * t, r[d]);
            }
#pragma unroll
            for (int d = 0; d < D; ++d) acc += (r[d][0] + r[d][1]) + (r[d][2] + r[d][3]);
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

// replay with each warp walking CH consecutive 32-entry pieces before the
// grid-stride jump: the GPU-wide window of in-flight stream positions grows with CH
template <int CH>
__global__ void __launch_bounds__(256, 4) replay_win_kernel(const double* __restrict__ x,
                                                           const unsigned* __restrict__ idx, long n, double* out) {
    const int lane = threadIdx.x & 31, g = lane / G, t = lane % G;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    double acc = 0;
    for (long p0 = w * 32 * CH; p0 < n; p0 += nw * 32 * CH) {
        for (long p = p0; p < p0 + 32 * CH && p < n; p += 32) {
            const unsigned c = idx[p + lane] & kMask;
#pragma unroll
            for (int j0 = 0; j0 < 16; j0 += 2) {
                double r[2][4];
#pragma unroll
                for (int d = 0; d < 2; ++d) {
                    const unsigned cj = __shfl_sync(0xffffffff, c, 2 * (j0 + d) + g);
                    ld256(x + (long)cj * W + 4 * t, r[d]);
                }
#pragma unroll
                for (int d = 0; d < 2; ++d) acc += (r[d][0] + r[d][1]) + (r[d][2] + r[d][3]);
            }
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

// replay morphs: kVal adds the value loads (8 B per entry, FMAs instead of adds);
// kRows walks whole rows (one row per warp, 128-column slab, 32 coalesced indices
// per step, D = 2 gathers in flight), kPersist grid-strides over rows instead of one
// row per warp, kStore writes the row at its end
template <bool kVal, bool kRows, bool kPersist, bool kStore>
__global__ void __launch_bounds__(256, 4) morph_kernel(const double* __restrict__ x, const unsigned* __restrict__ idx,
                                                      const double* __restrict__ val, const int64_t* __restrict__ pb,
                                                      const int* __restrict__ rid, int nrows, long n,
                                                      double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    long nw = (gridDim.x * (long)blockDim.x) >> 5;
    if (!kRows) {  // replay (x 64-column slab, two gathers per instruction)
        const int g = lane / G, t = lane % G;
        double acc[4] = {0, 0, 0, 0};
        for (long p = w * 32; p < n; p += nw * 32) {
            const unsigned c = idx[p + lane] & kMask;
            const double v = kVal ? val[p + lane] : 1.0;
#pragma unroll
            for (int j0 = 0; j0 < 16; j0 += 2) {
                double r[2][4], vv[2];
#pragma unroll
                for (int d = 0; d < 2; ++d) {
                    const unsigned cj = __shfl_sync(0xffffffff, c, 2 * (j0 + d) + g);
                    vv[d] = __shfl_sync(0xffffffff, v, 2 * (j0 + d) + g);
                    ld256(x + (long)cj * W + 4 * t, r[d]);
                }
#pragma unroll
                for (int d = 0; d < 2; ++d)
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[k] = kVal ? fma(vv[d], r[d][k], acc[k]) : acc[k] + r[d][k];
            }
        }
        if (acc[0] == 12345.0) y[0] = acc[1] + acc[2] + acc[3];
        return;
    }
    for (long r = w; r < nrows; r += kPersist ? nw : nrows) {
        const int64_t beg = pb[r], end = pb[r + 1];
        double acc[4] = {0, 0, 0, 0};
        for (int64_t p = beg; p < end; p += 32) {
            const int m = static_cast<int>(end - p < 32 ? end - p : 32);
            const unsigned c = lane < m ? idx[p + lane] & kMask : 0;
            const double v = lane < m ? (kVal ? val[p + lane] : 1.0) : 0.0;
            for (int j0 = 0; j0 < m; j0 += 2) {
                double rr[2][4], vv[2];
#pragma unroll
                for (int d = 0; d < 2; ++d) {
                    const unsigned cj = __shfl_sync(0xffffffff, c, (j0 + d) & 31);
                    vv[d] = __shfl_sync(0xffffffff, v, (j0 + d) & 31);
                    if (j0 + d < m) ld256(x + (long)cj * 128 + 4 * lane, rr[d]);
                }
#pragma unroll
                for (int d = 0; d < 2; ++d)
                    if (j0 + d < m)
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[k] = kVal ? fma(vv[d], rr[d][k], acc[k]) : acc[k] + rr[d][k];
            }
        }
        if (kStore || acc[0] == 12345.0) {
            double* o = y + static_cast<int64_t>(rid[r]) * 128 + 4 * lane;
            *reinterpret_cast<double2*>(o) = make_double2(acc[0], acc[1]);
            *reinterpret_cast<double2*>(o + 2) = make_double2(acc[2], acc[3]);
        }
    }
}

int main(int argc, char** argv) {
    int64_t nnz = 0;
    gen_rmat(22, 104000000, 0.57, 0.19, 0.19, 0, 4, &nnz);
    const long rows = 1L << 22;
    std::vector<int64_t> off(rows + 1), cidx(nnz);
    std::vector<double> cval(nnz);
    gen_fetch(off.data(), cidx.data(), cval.data());
    // row-length histogram
    {
        const int64_t bounds[] = {1, 2, 4, 8, 16, 32, 64, 128, 512, 1L << 40};
        int64_t cnt[10] = {0}, nz[10] = {0}, empty = 0;
        for (long r = 0; r < rows; ++r) {
            const int64_t L = off[r + 1] - off[r];
            if (L == 0) { ++empty; continue; }
            int b = 0;
            while (L > bounds[b]) ++b;
            ++cnt[b];
            nz[b] += L;
        }
        printf("rows %ld (empty %ld), nnz %ld\n", rows, (long)empty, (long)nnz);
        for (int b = 0; b < 10; ++b)
            printf("  len <= %-8lld rows %8lld  nnz %10lld (%.1f%%)\n", (long long)bounds[b], (long long)cnt[b],
                   (long long)nz[b], 100.0 * nz[b] / nnz);
    }
    std::vector<int> order;
    for (long r = 0; r < rows; ++r) {
        const int64_t L = off[r + 1] - off[r];
        if (L > 0 && L <= 512) order.push_back(static_cast<int>(r));
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
    const int nrows = static_cast<int>(order.size());
    std::vector<unsigned> sidx;
    std::vector<double> sval;
    std::vector<int64_t> pb{0};
    for (int r : order) {
        for (int64_t p = off[r]; p < off[r + 1]; ++p) {
            sidx.push_back(static_cast<unsigned>(cidx[p]) | (p + 1 == off[r + 1] ? kEnd : 0u));
            sval.push_back(cval[p]);
        }
        pb.push_back(static_cast<int64_t>(sidx.size()));
    }
    const int64_t S = static_cast<int64_t>(sidx.size());
    printf("non-split rows %d, their nnz %lld (%.1f%%)\n", nrows, (long long)S, 100.0 * S / nnz);
    std::vector<int> rid(order);
    for (int i = 0; i < 64; ++i) rid.push_back(0);
    unsigned* d_idx;
    double *d_val, *x, *y0, *y1, *out;
    int64_t* d_pb;
    int* d_rid;
    cudaMalloc(&d_idx, S * 4);
    cudaMalloc(&d_val, S * 8);
    cudaMalloc(&d_pb, pb.size() * 8);
    cudaMalloc(&d_rid, rid.size() * 4);
    cudaMalloc(&x, rows * 128 * 8);
    cudaMalloc(&y0, rows * W * 8);
    cudaMalloc(&y1, rows * 128 * 8);
    cudaMalloc(&out, 8);
    {
        std::vector<double> hx(rows * W);
        uint64_t s = 88172645463325252ull;
        for (auto& v : hx) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            v = static_cast<double>(s >> 11) * 0x1.0p-53 - 0.5;
        }
        cudaMemcpy(x, hx.data(), rows * W * 8, cudaMemcpyHostToDevice);
    }
    cudaMemcpy(d_idx, sidx.data(), S * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_val, sval.data(), S * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_pb, pb.data(), pb.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rid, rid.data(), rid.size() * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-40s %7.3f ms  %6.2f TB/s gathered\n", name, best, S * 512.0 / best / 1e9);
    };
    const int rblocks = (nrows + 2 * WARPS - 1) / (2 * WARPS);
    cudaMemset(y0, 0, rows * W * 8);
    timeit("row   U=2 32 warps", [&] { row_kernel<2, 4><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y0); });
    timeit("row   U=4 32 warps", [&] { row_kernel<4, 4><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y0); });
    {
        const int rb128 = (nrows + WARPS - 1) / WARPS, rb32 = (nrows + 4 * WARPS - 1) / (4 * WARPS);
        auto tw = [&](const char* nm, double gbytes, auto launch) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("%-40s %7.3f ms  %6.2f TB/s gathered  (per 64 columns %.3f ms)\n", nm, best, S * gbytes / best / 1e9,
                   best * 512.0 / gbytes);
        };
        tw("row W=128 U=2 32 warps", 1024.0, [&] { row_kernel<2, 4, true, true, 128><<<rb128, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
        tw("row W=128 U=1 32 warps", 1024.0, [&] { row_kernel<1, 4, true, true, 128><<<rb128, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
        tw("row W=128 U=4 24 warps", 1024.0, [&] { row_kernel<4, 3, true, true, 128><<<rb128, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
        tw("row W=32 U=2 32 warps", 256.0, [&] { row_kernel<2, 4, true, true, 32><<<rb32, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
        tw("row W=32 U=4 24 warps", 256.0, [&] { row_kernel<4, 3, true, true, 32><<<rb32, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    }
    timeit("row   U=2 32 warps, no stores", [&] { row_kernel<2, 4, false><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    timeit("row   U=2 32 warps, adds not FMAs", [&] { row_kernel<2, 4, true, false><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    timeit("row   U=2 32 warps, neither", [&] { row_kernel<2, 4, false, false><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    timeit("row   U=1 32 warps", [&] { row_kernel<1, 4><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    timeit("row   U=2 24 warps", [&] { row_kernel<2, 3><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    timeit("row   U=2 16 warps", [&] { row_kernel<2, 2><<<rblocks, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, y1); });
    std::vector<double> h0(rows * W), h1(rows * W);
    cudaMemcpy(h0.data(), y0, rows * W * 8, cudaMemcpyDeviceToHost);
    for (int T : {64}) {
        std::vector<int64_t> rs{0};
        std::vector<int> rr{0};
        int64_t acc = 0;
        for (int r = 0; r < nrows; ++r) {
            acc += pb[r + 1] - pb[r];
            if (acc >= T) {
                rs.push_back(pb[r + 1]);
                rr.push_back(r + 1);
                acc = 0;
            }
        }
        if (rs.back() != S) {
            rs.push_back(S);
            rr.push_back(nrows);
        }
        const int nruns = static_cast<int>(rs.size()) - 1;
        int64_t* d_rs;
        int* d_rr;
        cudaMalloc(&d_rs, rs.size() * 8);
        cudaMalloc(&d_rr, rr.size() * 4);
        cudaMemcpy(d_rs, rs.data(), rs.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(d_rr, rr.data(), rr.size() * 4, cudaMemcpyHostToDevice);
        char name[96];
        auto flat = [&](auto kern, int mb, const char* tag) {
            cudaMemset(y1, 0, rows * W * 8);
            snprintf(name, sizeof name, "flat  T=%d %s", T, tag);
            const int blocks = 148 * mb;
            timeit(name, [&] { kern<<<blocks, 256>>>(x, d_idx, d_val, d_rs, d_rr, d_rid, nruns, y1); });
            cudaMemcpy(h1.data(), y1, rows * W * 8, cudaMemcpyDeviceToHost);
            const bool same = std::memcmp(h0.data(), h1.data(), rows * W * 8) == 0;
            printf("      bitwise vs row: %s\n", same ? "yes" : "NO");
        };
        flat(flat_kernel<2, 4>, 4, "U=2 32 warps");
        cudaFree(d_rs);
        cudaFree(d_rr);
    }
    const long n = S / 32 * 32;
    timeit("replay D=2 (no FMAs)", [&] { replay_kernel<2><<<148 * 8, 256>>>(x, d_idx, n, out); });
    timeit("replay D=4 (no FMAs)", [&] { replay_kernel<4><<<148 * 8, 256>>>(x, d_idx, n, out); });
    {
        auto tm = [&](const char* nm, double gb, auto launch) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("%-44s %7.3f ms  %6.2f TB/s gathered\n", nm, best, S * gb / best / 1e9);
        };
        const int nb1 = (nrows + 7) / 8;
        tm("morph replay + values", 512.0, [&] { morph_kernel<true, false, false, false><<<148 * 8, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, n, y1); });
        tm("morph rows W=128 persistent, no vals", 1024.0, [&] { morph_kernel<false, true, true, false><<<148 * 8, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, n, y1); });
        tm("morph rows W=128 persistent + vals", 1024.0, [&] { morph_kernel<true, true, true, false><<<148 * 8, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, n, y1); });
        tm("morph rows W=128 persistent + vals + st", 1024.0, [&] { morph_kernel<true, true, true, true><<<148 * 8, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, n, y1); });
        tm("morph rows W=128 1 row/warp + vals", 1024.0, [&] { morph_kernel<true, true, false, false><<<nb1, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, n, y1); });
        tm("morph rows W=128 1 row/warp + vals + st", 1024.0, [&] { morph_kernel<true, true, false, true><<<nb1, 256>>>(x, d_idx, d_val, d_pb, d_rid, nrows, n, y1); });
    }
    timeit("replay window x2", [&] { replay_win_kernel<2><<<148 * 4, 256>>>(x, d_idx, n, out); });
    timeit("replay window x8", [&] { replay_win_kernel<8><<<148 * 4, 256>>>(x, d_idx, n, out); });
    timeit("replay window x32", [&] { replay_win_kernel<32><<<148 * 4, 256>>>(x, d_idx, n, out); });
    timeit("replay window x128", [&] { replay_win_kernel<128><<<148 * 4, 256>>>(x, d_idx, n, out); });
    timeit("replay window whole stream", [&] { replay_win_kernel<2048><<<148 * 4, 256>>>(x, d_idx, n, out); });
    timeit("replay D=2, 4 blocks/SM grid", [&] { replay_kernel<2><<<148 * 4, 256>>>(x, d_idx, n, out); });
    timeit("replay D=2, 64 blocks/SM grid", [&] { replay_kernel<2><<<148 * 64, 256>>>(x, d_idx, n, out); });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
