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

// row_off (optional): the CSR offsets of the matrix whose rows these are; rows
// without nonzeros are never gathered (A^T Omega reads Omega at A's non-empty
// rows only), so they are written as 0.0 instead of drawn — the drawn rows are
// bit for bit the same.
__device__ __forceinline__ bool row_empty(const int64_t* __restrict__ row_off, int64_t i) {
    return row_off != nullptr && __ldg(row_off + i) == __ldg(row_off + i + 1);
}

__global__ void gaussian_kernel(double* __restrict__ out, int64_t rows, int64_t l, int64_t ld,
                                uint64_t seed, int64_t global_rows, int64_t row_offset, int w,
                                const int64_t* __restrict__ row_off) {
    if (w > 0) {  // slab-major (sparse.cuh slab_index): writes walk the output contiguously
        const int64_t total = (ld + w - 1) / w * w * rows;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
             e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t jj = e % w, rs = e / w, i = rs % rows, j = (rs / rows) * w + jj;
            out[e] = j < l && !row_empty(row_off, i)
                         ? normal_at(seed, static_cast<uint64_t>(j * global_rows + row_offset + i))
                         : 0.0;
        }
        return;
    }
    const int64_t total = rows * ld;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    // 32-bit index arithmetic (no emulated 64-bit division) only when no thread's
    // index can wrap past 2^32 while still below total: total + stride <= 2^32
    if (total + stride <= (int64_t(1) << 32)) {
        const uint32_t ld32 = static_cast<uint32_t>(ld);
        for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < static_cast<uint32_t>(total);
             e += gridDim.x * blockDim.x) {
            const uint32_t i = e / ld32, j = e - i * ld32;
            out[e] = j < l && !row_empty(row_off, i)
                         ? normal_at(seed, static_cast<uint64_t>(j) * global_rows + row_offset + i)
                         : 0.0;
        }
        return;
    }
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / ld;
        const int64_t j = e - i * ld;
        out[e] = j < l && !row_empty(row_off, i)
                     ? normal_at(seed, static_cast<uint64_t>(j * global_rows + row_offset + i))
                     : 0.0;
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


// ---- register-tiled kernels (8x8 accumulators per thread) -----------------------------
// Gram v2: one block per row chunk computes the whole upper triangle of its
// chunk's C^T C; thread t owns one 8x8 tile (ti <= tj) in registers, C rows
// are staged 8 at a time in shared memory (double buffered with cp.async),
// a (8 values, shared by most lanes of a warp -> broadcast) and b (8 values)
// give 64 DFMA per 16 loads. Chunk partials are reduced in a fixed order.
constexpr int kG2Rows = 8;        // rows per stage

__device__ __forceinline__ void cpa16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

__global__ void __launch_bounds__(256)
gram2_kernel(const double* __restrict__ c, int64_t n, int64_t ld, int lp8, int ntile,
             int64_t rows_per_block, double* __restrict__ partial, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ __align__(16) double g2s[];  // [2][kG2Rows][lp8]
    const int npair = ntile * (ntile + 1) / 2;
    // tile pair of this thread (row-major over ti <= tj)
    int ti = 0, rem = threadIdx.x;
    while (ti < ntile && rem >= ntile - ti) {
        rem -= ntile - ti;
        ++ti;
    }
    const int tj = ti + rem;
    const bool owner = threadIdx.x < npair;
    const int64_t r_beg = static_cast<int64_t>(blockIdx.x) * rows_per_block;
    const int64_t r_end = min(n, r_beg + rows_per_block);
    double acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    const int vec_per_row = static_cast<int>(ld / 2);  // 16-byte vectors per row
    auto stage = [&](int buf, int64_t r0) {
        double* dst = g2s + buf * kG2Rows * lp8;
        for (int e = threadIdx.x; e < kG2Rows * (lp8 / 2); e += blockDim.x) {
            const int rr = e / (lp8 / 2), v = e % (lp8 / 2);
            const int64_t r = r0 + rr;
            if (r < r_end && v < vec_per_row)
                cpa16(dst + rr * lp8 + 2 * v, c + r * ld + 2 * v);
            else
                *reinterpret_cast<double2*>(dst + rr * lp8 + 2 * v) = make_double2(0.0, 0.0);
        }
    };
    if (r_beg < r_end) stage(0, r_beg);
    cpa_commit();
    int buf = 0;
    for (int64_t r0 = r_beg; r0 < r_end; r0 += kG2Rows) {
        if (r0 + kG2Rows < r_end) stage(buf ^ 1, r0 + kG2Rows);
        cpa_commit();
        cpa_wait1();
        __syncthreads();
        if (owner) {
            const double* cs = g2s + buf * kG2Rows * lp8;
#pragma unroll
            for (int k = 0; k < kG2Rows; ++k) {
                double av[8], bv[8];
                const double2* ap = reinterpret_cast<const double2*>(cs + k * lp8 + 8 * ti);
                const double2* bp = reinterpret_cast<const double2*>(cs + k * lp8 + 8 * tj);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const double2 x = ap[h], y = bp[h];
                    av[2 * h] = x.x;
                    av[2 * h + 1] = x.y;
                    bv[2 * h] = y.x;
                    bv[2 * h + 1] = y.y;
                }
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
            }
        }
        __syncthreads();
        buf ^= 1;
    }
    cpa_wait0();
    if (owner) {
        double* out = partial + (static_cast<int64_t>(blockIdx.x) * npair + threadIdx.x) * 64;
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; b += 2)
                *reinterpret_cast<double2*>(out + a * 8 + b) = make_double2(acc[a][b], acc[a][b + 1]);
    }
}

// G(i, j) = G(j, i) = sum over blocks (fixed order) of the tile entry; one thread per upper entry.
__global__ void gram2_reduce_kernel(const double* __restrict__ partial, int nblk, int ntile,
                                    int64_t l, double* __restrict__ g, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    const int npair = ntile * (ntile + 1) / 2;
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= static_cast<int64_t>(npair) * 64) return;
    const int t = static_cast<int>(e / 64), w = static_cast<int>(e % 64);
    int ti = 0, rem = t;
    while (rem >= ntile - ti) {
        rem -= ntile - ti;
        ++ti;
    }
    const int tj = ti + rem;
    const int64_t i = 8 * ti + w / 8, j = 8 * tj + w % 8;
    if (i >= l || j >= l || i > j) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += partial[(static_cast<int64_t>(b) * npair + t) * 64 + w];
    g[i * l + j] = s;
    g[j * l + i] = s;
}

// Rescale v2: out(r, j) = (sum_t c(r,t) w(t,j)) * scale[j], t ascending from 0.0
// (bitwise the reference matmul order). Block = 64 rows x all ncol columns;
// thread owns an 8x8 output tile; C (transposed) and W are staged 8 t at a time.
constexpr int kR2Rows = 64;
// measured slower than rescale_kernel on C2 (0.89 vs 0.62 ms); kept for tuning
bool rescale_v2_enabled = false;
constexpr int kR2K = 8;

__global__ void __launch_bounds__(256)
rescale2_kernel(const double* __restrict__ c, int64_t n, int64_t K, int64_t ldc,
                const double* __restrict__ w, int64_t ldw, const double* __restrict__ scale,
                int64_t ncol, int np8, double* __restrict__ out, int64_t ld_out, int out_colmajor,
                const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    extern __shared__ __align__(16) double r2s[];
    double* As = r2s;                       // [kR2K][kR2Rows]   (transposed C tile)
    double* Ws = r2s + kR2K * kR2Rows;      // [kR2K][np8]
    const int ntc = np8 / 8;                // column tiles
    const int tr = threadIdx.x / ntc, tc = threadIdx.x % ntc;  // 8 row tiles x ntc col tiles
    const bool owner = tr < kR2Rows / 8;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kR2Rows;
    double acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    for (int64_t t0 = 0; t0 < K; t0 += kR2K) {
        const int kmax = static_cast<int>(K - t0 < kR2K ? K - t0 : kR2K);
        for (int e = threadIdx.x; e < kR2K * kR2Rows; e += blockDim.x) {
            const int rr = e / kR2K, kk = e % kR2K;
            const int64_t r = r0 + rr;
            As[kk * kR2Rows + rr] = (r < n && kk < kmax) ? c[r * ldc + t0 + kk] : 0.0;
        }
        for (int e = threadIdx.x; e < kR2K * np8; e += blockDim.x) {
            const int kk = e / np8, jj = e % np8;
            Ws[kk * np8 + jj] = (kk < kmax && jj < ncol) ? w[(t0 + kk) * ldw + jj] : 0.0;
        }
        __syncthreads();
        if (owner) {
            for (int kk = 0; kk < kmax; ++kk) {
                double av[8], bv[8];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const double2 x = reinterpret_cast<const double2*>(As + kk * kR2Rows + 8 * tr)[h];
                    const double2 y = reinterpret_cast<const double2*>(Ws + kk * np8 + 8 * tc)[h];
                    av[2 * h] = x.x;
                    av[2 * h + 1] = x.y;
                    bv[2 * h] = y.x;
                    bv[2 * h + 1] = y.y;
                }
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
            }
        }
        __syncthreads();
    }
    if (!owner) return;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int64_t r = r0 + 8 * tr + a;
        if (r >= n) continue;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int64_t j = 8 * tc + b;
            const double v = j < ncol ? (scale != nullptr ? acc[a][b] * scale[j] : acc[a][b]) : 0.0;
            if (out_colmajor) {
                if (j < ncol) out[j * n + r] = v;
            } else if (j < ld_out) {
                out[r * ld_out + j] = v;
            }
        }
    }
}

int grid_for(int64_t n) {
    const int64_t g = ceil_div(n, 256);
    return static_cast<int>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

void gaussian_rowmajor(double* out, int64_t rows, int64_t l, int64_t ld, uint64_t seed,
                       cudaStream_t stream, int64_t global_rows, int64_t row_offset, int slab_w,
                       const int64_t* row_off) {
    if (rows * ld == 0) return;
    if (global_rows < 0) global_rows = rows;
    gaussian_kernel<<<grid_for(rows * ld), 256, 0, stream>>>(out, rows, l, ld, seed, global_rows,
                                                             row_offset, slab_w, row_off);
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

namespace {
// v2 plan: lp8 = l rounded to 8, tile pairs must fit one block
struct Gram2Plan {
    int lp8, ntile, npair, nblk;
    int64_t rows_per_block;
    bool ok;
};
Gram2Plan gram2_plan(int64_t n, int64_t l, int64_t ld) {
    Gram2Plan p{};
    p.lp8 = static_cast<int>((l + 7) / 8 * 8);
    p.ntile = p.lp8 / 8;
    p.npair = p.ntile * (p.ntile + 1) / 2;
    // one thread per 8x8 block pair, ~190 registers each: at most 256 threads
    // per block (the kernel's launch bound; l <= 176)
    p.ok = p.npair <= 256 && ld % 2 == 0 && p.lp8 >= ld - 3;
    const int64_t target = 2 * kNumSMs;
    int64_t rpb = ceil_div(n, target);
    rpb = std::max<int64_t>(kG2Rows, ceil_div(rpb, kG2Rows) * kG2Rows);
    p.rows_per_block = rpb;
    p.nblk = static_cast<int>(std::max<int64_t>(1, ceil_div(n, rpb)));
    return p;
}
}  // namespace

size_t gram_workspace_bytes(int64_t n, int64_t l) {
    const Gram2Plan p2 = gram2_plan(n, l, padded_ld(l));
    const size_t v2 = sizeof(double) * static_cast<size_t>(p2.nblk) * p2.npair * 64;
    int ntiles, nchunk;
    int64_t rpc;
    gram_plan(n, l, ntiles, nchunk, rpc);
    return std::max(v2, sizeof(double) * static_cast<size_t>(ntiles) * nchunk * kTile * kTile);
}

void gram(const double* c, int64_t n, int64_t l, int64_t ld, double* g, void* ws,
          size_t ws_bytes, const int32_t* gate, cudaStream_t stream) {
    const Gram2Plan p2 = gram2_plan(n, l, ld);
    if (p2.ok && n > 0) {
        const size_t smem = sizeof(double) * 2 * kG2Rows * p2.lp8;
        const int threads = std::max(64, (p2.npair + 31) / 32 * 32);
        gram2_kernel<<<p2.nblk, threads, smem, stream>>>(c, n, ld, p2.lp8, p2.ntile, p2.rows_per_block,
                                                         static_cast<double*>(ws), gate);
        DSVD_LAUNCH_CHECK();
        const int64_t ne = static_cast<int64_t>(p2.npair) * 64;
        gram2_reduce_kernel<<<static_cast<unsigned>(ceil_div(ne, 256)), 256, 0, stream>>>(
            static_cast<const double*>(ws), p2.nblk, p2.ntile, l, g, gate);
        DSVD_LAUNCH_CHECK();
        return;
    }
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
    const int np8 = static_cast<int>((width + 7) / 8 * 8);
    const int threads = (kR2Rows / 8) * (np8 / 8);
    if (rescale_v2_enabled && threads <= 320 && np8 > 0) {
        const size_t smem = sizeof(double) * kR2K * (kR2Rows + np8);
        rescale2_kernel<<<static_cast<unsigned>(ceil_div(n, kR2Rows)), (threads + 31) / 32 * 32, smem, stream>>>(
            c, n, K, ldc, w, ldw, scale, ncol, np8, out, ld_out, out_colmajor, gate);
        DSVD_LAUNCH_CHECK();
        return;
    }
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
