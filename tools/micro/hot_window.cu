// Microbenchmark: does an L2 persisting window over the hottest X rows help the
// slab SpMM? The C4 rows of at most 512 nonzeros (longest first) through the
// product-structured row kernel (one row per 16-lane group, U = 2), one 64-column
// slab-major X: (a) as is, (b) X rows relabelled hottest first (column indices
// remapped), (c) (b) + a cudaAccessPolicyWindow (persisting, hitRatio 1) over the
// first H MB of X with the persisting L2 set-aside at its maximum.
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


int main() {
    int64_t nnz = 0;
    gen_rmat(22, 104000000, 0.57, 0.19, 0.19, 0, 4, &nnz);
    const long rows = 1L << 22;
    std::vector<int64_t> off(rows + 1), cidx(nnz);
    std::vector<double> cval(nnz);
    gen_fetch(off.data(), cidx.data(), cval.data());
    std::vector<int> order;
    for (long r = 0; r < rows; ++r) {
        const int64_t L = off[r + 1] - off[r];
        if (L > 0 && L <= 512) order.push_back(static_cast<int>(r));
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
    const int nrows = static_cast<int>(order.size());
    std::vector<unsigned> sidx, ridx;
    std::vector<double> sval;
    std::vector<int64_t> pb{0};
    std::vector<int64_t> deg(rows, 0);
    for (int r : order) {
        for (int64_t p = off[r]; p < off[r + 1]; ++p) {
            sidx.push_back(static_cast<unsigned>(cidx[p]));
            sval.push_back(cval[p]);
            ++deg[cidx[p]];
        }
        pb.push_back(static_cast<int64_t>(sidx.size()));
    }
    const int64_t S = static_cast<int64_t>(sidx.size());
    std::vector<int> byd(rows);
    std::iota(byd.begin(), byd.end(), 0);
    std::stable_sort(byd.begin(), byd.end(), [&](int a, int b) { return deg[a] > deg[b]; });
    std::vector<unsigned> perm(rows);
    for (long i = 0; i < rows; ++i) perm[byd[i]] = static_cast<unsigned>(i);
    ridx.resize(S);
    for (int64_t p = 0; p < S; ++p) ridx[p] = perm[sidx[p]];
    for (int H : {32, 64, 96, 128}) {
        const long k = H * (1L << 20) / 512;
        int64_t hits = 0;
        for (long i = 0; i < k; ++i) hits += deg[byd[i]];
        printf("hottest %ld X rows (%d MB) take %.1f%% of the gathers\n", k, H, 100.0 * hits / S);
    }
    std::vector<int> rid(order);
    for (int i = 0; i < 64; ++i) rid.push_back(0);
    unsigned *d_idx, *d_ridx;
    double *d_val, *x, *y;
    int64_t* d_pb;
    int* d_rid;
    cudaMalloc(&d_idx, S * 4);
    cudaMalloc(&d_ridx, S * 4);
    cudaMalloc(&d_val, S * 8);
    cudaMalloc(&d_pb, pb.size() * 8);
    cudaMalloc(&d_rid, rid.size() * 4);
    cudaMalloc(&x, rows * W * 8);
    cudaMalloc(&y, rows * W * 8);
    cudaMemset(x, 0, rows * W * 8);
    cudaMemcpy(d_idx, sidx.data(), S * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ridx, ridx.data(), S * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_val, sval.data(), S * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_pb, pb.data(), pb.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rid, rid.data(), rid.size() * 4, cudaMemcpyHostToDevice);
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    printf("max persisting L2 %d MB\n", maxp >> 20);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int rblocks = (nrows + 2 * WARPS - 1) / (2 * WARPS);
    auto timeit = [&](const char* name, const unsigned* ix) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a, st);
            row_kernel<2, 4><<<rblocks, 256, 0, st>>>(x, ix, d_val, d_pb, d_rid, nrows, y);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-52s %7.3f ms  %6.2f TB/s gathered\n", name, best, S * 512.0 / best / 1e9);
    };
    timeit("original labels", d_idx);
    timeit("hottest X rows first", d_ridx);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
    for (int H : {32, 64, 96}) {
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.base_ptr = x;
        v.accessPolicyWindow.num_bytes = static_cast<size_t>(H) << 20;
        v.accessPolicyWindow.hitRatio = 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
        char nm[96];
        snprintf(nm, sizeof nm, "hottest first + persisting window %d MB", H);
        timeit(nm, d_ridx);
        snprintf(nm, sizeof nm, "original labels + persisting window %d MB", H);
        timeit(nm, d_idx);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
