// Sparse kernels of the dashSVD power loop on sm_100a.
//
//  - spmm: Y = A X (and the fused shifted update T = A^T Y - alpha Q) over
//    row-major l-column fp64 blocks. Each output element is ONE fused
//    multiply-add chain over its row's nonzeros in CSR order starting from
//    0.0 — the exact operation order of the reference kernel
//    (sparse_matrix.cpp:74-83, which GCC contracts to vfmadd) and of
//    add_scaled (dense_kernels.cpp:128-136) — so results are bitwise equal to
//    the reference. Work items are (row, 64-column slab) pairs, one warp each,
//    rows taken longest-first so hub rows of power-law matrices start first.
//  - build_transpose: CSR(A^T) as a stable sort of the nonzeros by column
//    (the counting sort of sparse_matrix.cpp:35-55 is stable in row order),
//    bitwise equal to the reference.
#include <cub/device/device_radix_sort.cuh>

#include "sparse.cuh"

namespace dsvd {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSlab = 64;  // doubles per warp work item: 32 lanes x double2

__device__ __forceinline__ double2 ld_x(const double* p) {
    return __ldg(reinterpret_cast<const double2*>(p));
}

// One warp = one (row, slab) item. Lanes own two adjacent columns each.
template <bool kShift>
__global__ void __launch_bounds__(256)
spmm_rowslab_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                    const double* __restrict__ val, const int32_t* __restrict__ order,
                    int64_t rows, int nslab, const double* __restrict__ x,
                    double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                    const double* __restrict__ alpha_p, const int32_t* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;
    const int lane = threadIdx.x & 31;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (item >= rows * nslab) return;
    const int64_t rpos = item / nslab;
    const int slab = static_cast<int>(item - rpos * nslab);
    const int64_t row = order != nullptr ? static_cast<int64_t>(order[rpos]) : rpos;
    const int64_t col = static_cast<int64_t>(slab) * kSlab + 2 * lane;
    const bool active = col < ld;  // ld is a multiple of 4, so col+1 < ld as well
    const int64_t beg = off[row], end = off[row + 1];
    const double* xc = x + (active ? col : 0);

    double a0 = 0.0, a1 = 0.0;
    for (int64_t p0 = beg; p0 < end; p0 += 32) {
        const int cnt = static_cast<int>(end - p0 < 32 ? end - p0 : 32);
        int c = 0;
        double v = 0.0;
        if (lane < cnt) {
            c = __ldg(idx + p0 + lane);
            v = __ldg(val + p0 + lane);
        }
        if (cnt == 32) {
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                const int cj = __shfl_sync(kFull, c, j);
                const double vj = __shfl_sync(kFull, v, j);
                if (active) {
                    const double2 xv = ld_x(xc + static_cast<int64_t>(cj) * ld);
                    a0 = fma(vj, xv.x, a0);
                    a1 = fma(vj, xv.y, a1);
                }
            }
        } else {
            for (int j = 0; j < cnt; ++j) {
                const int cj = __shfl_sync(kFull, c, j);
                const double vj = __shfl_sync(kFull, v, j);
                if (active) {
                    const double2 xv = ld_x(xc + static_cast<int64_t>(cj) * ld);
                    a0 = fma(vj, xv.x, a0);
                    a1 = fma(vj, xv.y, a1);
                }
            }
        }
    }
    if (!active) return;
    if (kShift) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) {  // solver.cpp:94 skips the update when alpha == 0
            const double2 qv = *reinterpret_cast<const double2*>(q + row * ld + col);
            a0 = fma(-alpha, qv.x, a0);
            a1 = fma(-alpha, qv.y, a1);
        }
    }
    *reinterpret_cast<double2*>(y + row * ld + col) = make_double2(a0, a1);
}

__global__ void narrow_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                              int64_t nnz, int64_t cols, int32_t* bad) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t c = src[p];
        if (c < 0 || c >= cols) {
            *bad = 1;
            c = 0;
        }
        dst[p] = static_cast<int32_t>(c);
    }
}

__global__ void widen_kernel(const int32_t* __restrict__ src, int64_t* __restrict__ dst,
                             int64_t nnz) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[p] = src[p];
}

__global__ void check_offsets_kernel(const int64_t* __restrict__ off, int64_t rows, int64_t nnz,
                                     int32_t* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (off[i] > off[i + 1] || off[i] < 0 || off[i + 1] > nnz) *bad = 1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[rows] != nnz)) *bad = 1;
}

// row_of[p] = i for p in [off[i], off[i+1]) — one warp per row.
__global__ void expand_rows_kernel(const int64_t* __restrict__ off, int64_t rows,
                                   int32_t* __restrict__ row_of) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
         i < rows; i += warps) {
        for (int64_t p = off[i] + lane; p < off[i + 1]; p += 32) row_of[p] = static_cast<int32_t>(i);
    }
}

__global__ void iota_kernel(int32_t* __restrict__ v, int64_t n) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[p] = static_cast<int32_t>(p);
}

__global__ void gather_transpose_kernel(const int32_t* __restrict__ perm,
                                        const int32_t* __restrict__ row_of,
                                        const double* __restrict__ val, int32_t* __restrict__ t_idx,
                                        double* __restrict__ t_val, int64_t nnz) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t p = perm[k];
        t_idx[k] = row_of[p];
        t_val[k] = val[p];
    }
}

// t_off[c] = first position whose (sorted) column key is >= c.
__global__ void offsets_from_keys_kernel(const int32_t* __restrict__ keys, int64_t nnz,
                                         int64_t cols, int64_t* __restrict__ t_off) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t key = keys[k];
        const int64_t prev = k > 0 ? static_cast<int64_t>(keys[k - 1]) : -1;
        for (int64_t c = prev + 1; c <= key; ++c) t_off[c] = k;
        if (k == nnz - 1)
            for (int64_t c = key + 1; c <= cols; ++c) t_off[c] = nnz;
    }
}

__global__ void fill_i64_kernel(int64_t* __restrict__ p, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void row_lengths_kernel(const int64_t* __restrict__ off, int64_t rows,
                                   int32_t* __restrict__ len, int32_t* __restrict__ ids) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t n = off[i + 1] - off[i];
        len[i] = static_cast<int32_t>(n > 0x7fffffff ? 0x7fffffff : n);
        ids[i] = static_cast<int32_t>(i);
    }
}

int grid_for(int64_t n, int threads = 256) {
    const int64_t g = ceil_div(n, threads);
    return static_cast<int>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

int key_bits(int64_t maxval) {
    int b = 1;
    while (b < 32 && (int64_t(1) << b) <= maxval) ++b;
    return b;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

void spmm(const SpmmArgs& s, cudaStream_t stream, int variant) {
    (void)variant;
    const DevCsr& a = *s.a;
    if (a.rows == 0) return;
    const int nslab = static_cast<int>(ceil_div(s.ld, kSlab));
    const int64_t items = a.rows * nslab;
    const int warps_per_block = 8;
    const int64_t blocks = ceil_div(items, warps_per_block);
    if (s.q != nullptr) {
        spmm_rowslab_kernel<true><<<static_cast<unsigned>(blocks), 32 * warps_per_block, 0, stream>>>(
            a.off, a.idx, a.val, a.order, a.rows, nslab, s.x, s.y, s.ld, s.q, s.alpha, s.gate);
    } else {
        spmm_rowslab_kernel<false><<<static_cast<unsigned>(blocks), 32 * warps_per_block, 0, stream>>>(
            a.off, a.idx, a.val, a.order, a.rows, nslab, s.x, s.y, s.ld, nullptr, nullptr, s.gate);
    }
    DSVD_LAUNCH_CHECK();
}

void narrow_indices(const int64_t* src, int32_t* dst, int64_t nnz, int64_t cols, int32_t* bad,
                    cudaStream_t stream) {
    if (nnz == 0) return;
    narrow_kernel<<<grid_for(nnz), 256, 0, stream>>>(src, dst, nnz, cols, bad);
    DSVD_LAUNCH_CHECK();
}

void widen_indices(const int32_t* src, int64_t* dst, int64_t nnz, cudaStream_t stream) {
    if (nnz == 0) return;
    widen_kernel<<<grid_for(nnz), 256, 0, stream>>>(src, dst, nnz);
    DSVD_LAUNCH_CHECK();
}

void check_offsets(const int64_t* off, int64_t rows, int64_t nnz, int32_t* bad,
                   cudaStream_t stream) {
    check_offsets_kernel<<<grid_for(rows), 256, 0, stream>>>(off, rows, nnz, bad);
    DSVD_LAUNCH_CHECK();
}

size_t csc_scratch_bytes(int64_t rows, int64_t cols, int64_t nnz) {
    (void)rows;
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), nnz > 0 ? nnz : 1, 0,
                                    key_bits(cols));
    return 4 * align_up(sizeof(int32_t) * (nnz > 0 ? nnz : 1)) + align_up(temp);
}

void build_transpose(const DevCsr& a, DevCsr& at, void* scratch, size_t scratch_bytes,
                     cudaStream_t stream) {
    at.rows = a.cols;
    at.cols = a.rows;
    at.nnz = a.nnz;
    const int64_t nnz = a.nnz;
    if (nnz == 0) {
        fill_i64_kernel<<<grid_for(at.rows + 1), 256, 0, stream>>>(at.off, at.rows + 1, 0);
        DSVD_LAUNCH_CHECK();
        return;
    }
    if (nnz > 0x7fffffffLL) fail(DSVD_UNSUPPORTED, "transpose: nnz >= 2^31 is not supported");
    char* p = static_cast<char*>(scratch);
    const size_t seg = align_up(sizeof(int32_t) * nnz);
    int32_t* row_of = reinterpret_cast<int32_t*>(p);
    int32_t* keys_out = reinterpret_cast<int32_t*>(p + seg);
    int32_t* perm_in = reinterpret_cast<int32_t*>(p + 2 * seg);
    int32_t* perm_out = reinterpret_cast<int32_t*>(p + 3 * seg);
    void* temp = p + 4 * seg;
    size_t temp_bytes = scratch_bytes - 4 * seg;

    expand_rows_kernel<<<grid_for(a.rows * 32), 256, 0, stream>>>(a.off, a.rows, row_of);
    DSVD_LAUNCH_CHECK();
    iota_kernel<<<grid_for(nnz), 256, 0, stream>>>(perm_in, nnz);
    DSVD_LAUNCH_CHECK();
    // LSD radix sort is stable: equal columns keep their CSR (row-major) order,
    // exactly the counting sort's placement.
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, a.idx, keys_out, perm_in,
                                                    perm_out, nnz, 0, key_bits(a.cols), stream));
    gather_transpose_kernel<<<grid_for(nnz), 256, 0, stream>>>(perm_out, row_of, a.val, at.idx,
                                                               at.val, nnz);
    DSVD_LAUNCH_CHECK();
    offsets_from_keys_kernel<<<grid_for(nnz), 256, 0, stream>>>(keys_out, nnz, at.rows, at.off);
    DSVD_LAUNCH_CHECK();
}

size_t order_scratch_bytes(int64_t rows) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairsDescending(
        nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
        static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
        rows > 0 ? rows : 1, 0, 32);
    return 3 * align_up(sizeof(int32_t) * (rows > 0 ? rows : 1)) + align_up(temp);
}

void build_row_order(DevCsr& m, void* scratch, size_t scratch_bytes, cudaStream_t stream) {
    if (m.rows == 0) return;
    char* p = static_cast<char*>(scratch);
    const size_t seg = align_up(sizeof(int32_t) * m.rows);
    int32_t* len = reinterpret_cast<int32_t*>(p);
    int32_t* len_sorted = reinterpret_cast<int32_t*>(p + seg);
    int32_t* ids = reinterpret_cast<int32_t*>(p + 2 * seg);
    void* temp = p + 3 * seg;
    size_t temp_bytes = scratch_bytes - 3 * seg;
    row_lengths_kernel<<<grid_for(m.rows), 256, 0, stream>>>(m.off, m.rows, len, ids);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, len, len_sorted,
                                                              ids, m.order, m.rows, 0, 32, stream));
}

}  // namespace dsvd
