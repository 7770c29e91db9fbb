// Dense kernels of the eigSVD re-orthonormalisation on sm_100a (FP64).
//
// B200 FP64 runs at the same rate on the DFMA pipe as on the FP64 tensor
// path, so these are register-tiled DFMA kernels: 64x64 output tiles, 4x4
// accumulators per thread, 16-deep K slabs staged in shared memory. The rescale
// keeps the reference's per-element FMA order (t ascending from 0.0), so given
// the same V and 1/s it is bitwise equal to matmul + scale_columns.
#include "dense.cuh"
#include "rng.cuh"

namespace dsvd {

namespace {

constexpr int kTile = 64;
constexpr int kK = 16;

__global__ void gaussian_kernel(double* __restrict__ out, int64_t rows, int64_t l, int64_t ld,
                                uint64_t seed, int64_t global_rows, int64_t row_offset) {
    const int64_t total = rows * ld;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / ld;
        const int64_t j = e - i * ld;
        out[e] = j < l ? normal_at(seed, static_cast<uint64_t>(j * global_rows + row_offset + i)) : 0.0;
    }
}

__global__ void shift_kernel(double* __restrict__ t, const double* __restrict__ q, int64_t count,
                             const double* __restrict__ alpha_p, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    const double alpha = *alpha_p;
    if (alpha == 0.0) return;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        t[e] = fma(-alpha, q[e], t[e]);
}

// Partial Gram over one row chunk for one upper-triangle 64x64 tile.
__global__ void __launch_bounds__(256)
gram_partial_kernel(const double* __restrict__ c, int64_t n, int64_t l, int64_t ld,
                    int64_t rows_per_chunk, double* __restrict__ partial,
                    const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    __shared__ double As[kK][kTile];
    __shared__ double Bs[kK][kTile];
    // decode tile (bi <= bj) from the linear upper-triangle index
    const int nt = static_cast<int>((l + kTile - 1) / kTile);
    int t = blockIdx.x, bi = 0;
    while (t >= nt - bi) {
        t -= nt - bi;
        ++bi;
    }
    const int bj = bi + t;
    const int64_t i0 = static_cast<int64_t>(bi) * kTile, j0 = static_cast<int64_t>(bj) * kTile;
    const int64_t r_beg = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
    const int64_t r_end = min(n, r_beg + rows_per_chunk);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;

    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

    for (int64_t r0 = r_beg; r0 < r_end; r0 += kK) {
#pragma unroll
        for (int e = threadIdx.x; e < kK * kTile; e += 256) {
            const int kk = e / kTile, cc = e % kTile;
            const int64_t r = r0 + kk;
            const bool okr = r < r_end;
            As[kk][cc] = (okr && i0 + cc < l) ? c[r * ld + i0 + cc] : 0.0;
            Bs[kk][cc] = (okr && j0 + cc < l) ? c[r * ld + j0 + cc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kK; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[kk][ty * 4 + a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx * 4 + b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
    double* out = partial + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * kTile * kTile;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) out[(ty * 4 + a) * kTile + tx * 4 + b] = acc[a][b];
}

// G(i, j) = G(j, i) = sum over chunks (fixed order) of the upper-tile entry.
__global__ void gram_reduce_kernel(const double* __restrict__ partial, int nchunk, int ntiles,
                                   int64_t l, double* __restrict__ g,
                                   const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    const int nt = static_cast<int>((l + kTile - 1) / kTile);
    const int64_t per_tile = kTile * kTile;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
         e < static_cast<int64_t>(ntiles) * per_tile; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int t = static_cast<int>(e / per_tile);
        const int w = static_cast<int>(e % per_tile);
        int bi = 0;
        while (t >= nt - bi) {
            t -= nt - bi;
            ++bi;
        }
        const int bj = bi + t;
        const int64_t i = static_cast<int64_t>(bi) * kTile + w / kTile;
        const int64_t j = static_cast<int64_t>(bj) * kTile + w % kTile;
        if (i >= l || j >= l || i > j) continue;
        const int64_t tile = e / per_tile;
        double s = 0.0;
        for (int ch = 0; ch < nchunk; ++ch) s += partial[(static_cast<int64_t>(ch) * ntiles + tile) * per_tile + w];
        g[i * l + j] = s;
        g[j * l + i] = s;
    }
}

__global__ void __launch_bounds__(256)
rescale_kernel(const double* __restrict__ c, int64_t n, int64_t K, int64_t ldc,
               const double* __restrict__ w, int64_t ldw, const double* __restrict__ scale,
               int64_t ncol, double* __restrict__ out, int64_t ld_out, int out_colmajor,
               const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    __shared__ double As[kK][kTile + 1];
    __shared__ double Ws[kK][kTile];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTile;
    const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kTile;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

    for (int64_t t0 = 0; t0 < K; t0 += kK) {
        const int kmax = static_cast<int>(K - t0 < kK ? K - t0 : kK);
        for (int e = threadIdx.x; e < kK * kTile; e += 256) {
            // A slab: 64 rows x 16 t, loaded row by row (16 contiguous doubles)
            const int rr = e / kK, kk = e % kK;
            const int64_t r = r0 + rr;
            As[kk][rr] = (r < n && kk < kmax) ? c[r * ldc + t0 + kk] : 0.0;
            const int kw = e / kTile, jj = e % kTile;
            Ws[kw][jj] = (kw < kmax && j0 + jj < ncol) ? w[(t0 + kw) * ldw + j0 + jj] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kmax; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[kk][ty * 4 + a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Ws[kk][tx * 4 + b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t r = r0 + ty * 4 + a;
        if (r >= n) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t j = j0 + tx * 4 + b;
            if (out_colmajor) {
                if (j < ncol) out[j * n + r] = scale != nullptr ? acc[a][b] * scale[j] : acc[a][b];
            } else if (j < ld_out) {
                out[r * ld_out + j] =
                    j < ncol ? (scale != nullptr ? acc[a][b] * scale[j] : acc[a][b]) : 0.0;
            }
        }
    }
}

__global__ void cm_to_rm_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                double* __restrict__ dst, int64_t ld) {
    const int64_t total = rows * ld;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / ld, j = e - (e / ld) * ld;
        dst[e] = j < cols ? src[j * rows + i] : 0.0;
    }
}

__global__ void rm_to_cm_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                int64_t ld, double* __restrict__ dst) {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / rows, i = e - (e / rows) * rows;
        dst[e] = src[i * ld + j];
    }
}

int grid_for(int64_t n) {
    const int64_t g = ceil_div(n, 256);
    return static_cast<int>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

void gaussian_rowmajor(double* out, int64_t rows, int64_t l, int64_t ld, uint64_t seed,
                       cudaStream_t stream, int64_t global_rows, int64_t row_offset) {
    if (rows * ld == 0) return;
    if (global_rows < 0) global_rows = rows;
    gaussian_kernel<<<grid_for(rows * ld), 256, 0, stream>>>(out, rows, l, ld, seed, global_rows,
                                                             row_offset);
    DSVD_LAUNCH_CHECK();
}

void shift_update(double* t, const double* q, int64_t count, const double* alpha,
                  const int32_t* gate, cudaStream_t stream) {
    if (count == 0) return;
    shift_kernel<<<grid_for(count), 256, 0, stream>>>(t, q, count, alpha, gate);
    DSVD_LAUNCH_CHECK();
}

namespace {
void gram_plan(int64_t n, int64_t l, int& ntiles, int& nchunk, int64_t& rows_per_chunk) {
    const int nt = static_cast<int>((l + kTile - 1) / kTile);
    ntiles = nt * (nt + 1) / 2;
    // ~4 blocks per SM in total, chunks of at least 64 rows
    int64_t target = (4 * kNumSMs + ntiles - 1) / ntiles;
    int64_t maxchunks = ceil_div(n, 64);
    nchunk = static_cast<int>(std::max<int64_t>(1, std::min(target, maxchunks)));
    rows_per_chunk = ceil_div(n, nchunk);
    rows_per_chunk = ceil_div(rows_per_chunk, kK) * kK;
    nchunk = static_cast<int>(std::max<int64_t>(1, ceil_div(n, rows_per_chunk)));
}
}  // namespace

size_t gram_workspace_bytes(int64_t n, int64_t l) {
    int ntiles, nchunk;
    int64_t rpc;
    gram_plan(n, l, ntiles, nchunk, rpc);
    return sizeof(double) * static_cast<size_t>(ntiles) * nchunk * kTile * kTile;
}

void gram(const double* c, int64_t n, int64_t l, int64_t ld, double* g, void* ws,
          size_t ws_bytes, const int32_t* gate, cudaStream_t stream) {
    int ntiles, nchunk;
    int64_t rpc;
    gram_plan(n, l, ntiles, nchunk, rpc);
    if (ws_bytes < gram_workspace_bytes(n, l)) fail(DSVD_OTHER, "gram: workspace too small");
    double* partial = static_cast<double*>(ws);
    gram_partial_kernel<<<dim3(ntiles, nchunk), 256, 0, stream>>>(c, n, l, ld, rpc, partial, gate);
    DSVD_LAUNCH_CHECK();
    gram_reduce_kernel<<<grid_for(static_cast<int64_t>(ntiles) * kTile * kTile), 256, 0, stream>>>(
        partial, nchunk, ntiles, l, g, gate);
    DSVD_LAUNCH_CHECK();
}

void rescale(const double* c, int64_t n, int64_t K, int64_t ldc, const double* w, int64_t ldw,
             const double* scale, int64_t ncol, double* out, int64_t ld_out, int out_colmajor,
             const int32_t* gate, cudaStream_t stream) {
    if (n == 0) return;
    const int64_t width = out_colmajor ? ncol : ld_out;
    dim3 grid(static_cast<unsigned>(ceil_div(n, kTile)), static_cast<unsigned>(ceil_div(width, kTile)));
    rescale_kernel<<<grid, 256, 0, stream>>>(c, n, K, ldc, w, ldw, scale, ncol, out, ld_out,
                                             out_colmajor, gate);
    DSVD_LAUNCH_CHECK();
}

void colmajor_to_rowmajor(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ld,
                          cudaStream_t stream) {
    if (rows * ld == 0) return;
    cm_to_rm_kernel<<<grid_for(rows * ld), 256, 0, stream>>>(src, rows, cols, dst, ld);
    DSVD_LAUNCH_CHECK();
}

void rowmajor_to_colmajor(const double* src, int64_t rows, int64_t cols, int64_t ld, double* dst,
                          cudaStream_t stream) {
    if (rows * cols == 0) return;
    rm_to_cm_kernel<<<grid_for(rows * cols), 256, 0, stream>>>(src, rows, cols, ld, dst);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
