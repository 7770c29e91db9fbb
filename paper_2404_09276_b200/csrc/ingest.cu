// Input side of the path on the device:
//  - csr_validate: SparseMatrix::validate (sparse_matrix.cpp:12-33) with the
//    reference's first-violation semantics (rows in order, within a row the
//    offsets check, then per nonzero: index range, strictly increasing
//    indices, finite value, non-zero value), one warp per row;
//  - coo_assemble: the Matrix Market canonicalisation assemble()
//    (matrix_market.cpp:90-115): sort by (row, col), sum duplicates in order,
//    drop exact zeros, build offsets. The sort is stable (radix), so
//    duplicates add in input order; the reference's std::sort leaves their
//    order unspecified, hence bit-exact whenever duplicate sums do not depend
//    on order (in particular with no duplicates).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ingest.cuh"
#include "rng.cuh"

namespace dsvd {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// first[0] = min over rows of (row << 3 | code): code 0 offsets decrease,
// 1 index out of range, 2 indices not increasing, 3 non-finite, 4 explicit zero
__global__ void csr_validate_kernel(const int64_t* __restrict__ off, const int64_t* __restrict__ idx,
                                    const double* __restrict__ val, int64_t rows, int64_t cols, int64_t nnz,
                                    unsigned long long* __restrict__ first) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (row >= rows) return;
    const int64_t b = off[row], e = off[row + 1];
    const unsigned long long base = static_cast<unsigned long long>(row) << 3;
    // b < 0 or e > nnz (with offsets spanning [0, nnz]) implies a decrease in a
    // later row; report it here rather than read out of bounds (the reference's
    // loop would).
    if (b > e || b < 0 || e > nnz) {
        if (lane == 0) atomicMin(first, base | 0ull);
        return;
    }
    for (int64_t p0 = b; p0 < e; p0 += 32) {
        const int64_t p = p0 + lane;
        int code = 7;
        if (p < e) {
            const int64_t c = idx[p];
            const double v = val[p];
            if (c < 0 || c >= cols) code = 1;
            else if (p > b && idx[p - 1] >= c) code = 2;
            else if (!isfinite(v)) code = 3;
            else if (v == 0.0) code = 4;
        }
        const unsigned bad = __ballot_sync(kFull, code != 7);
        if (bad) {
            const int l0 = __ffs(bad) - 1;
            const int c0 = __shfl_sync(kFull, code, l0);
            if (lane == 0) atomicMin(first, base | static_cast<unsigned long long>(c0));
            return;
        }
    }
}

__global__ void coo_keys_kernel(const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t n,
                                int64_t rows, int64_t cols, uint64_t* __restrict__ keys, int64_t* __restrict__ pos,
                                int32_t* __restrict__ bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t ri = r[i], ci = c[i];
        if (ri < 0 || ri >= rows || ci < 0 || ci >= cols) *bad = 1;
        keys[i] = static_cast<uint64_t>(ri) * static_cast<uint64_t>(cols) + static_cast<uint64_t>(ci);
        pos[i] = i;
    }
}

// head[i] = 1 where sorted key i starts a run of equal keys
__global__ void run_heads_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ head) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per run: value = sum in (stable) order; keep[run] = value != 0
__global__ void run_sum_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ pos,
                               const double* __restrict__ v, const int64_t* __restrict__ head_scan, int64_t n,
                               uint64_t* __restrict__ rkey, double* __restrict__ rval, int64_t* __restrict__ keep) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i != 0 && keys[i] == keys[i - 1]) continue;
        double s = v[pos[i]];
        for (int64_t j = i + 1; j < n && keys[j] == keys[i]; ++j) s += v[pos[j]];
        const int64_t run = head_scan[i];  // inclusive scan of heads - 1 (below)
        rkey[run] = keys[i];
        rval[run] = s;
        keep[run] = (s == 0.0) ? 0 : 1;
    }
}

__global__ void compact_kernel(const uint64_t* __restrict__ rkey, const double* __restrict__ rval,
                               const int64_t* __restrict__ keep, const int64_t* __restrict__ kscan, int64_t nr,
                               int64_t cols, int64_t* __restrict__ out_idx, double* __restrict__ out_val,
                               int64_t* __restrict__ row_count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nr;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!keep[i]) continue;
        const int64_t w = kscan[i];
        const int64_t row = static_cast<int64_t>(rkey[i] / static_cast<uint64_t>(cols));
        out_idx[w] = static_cast<int64_t>(rkey[i] - static_cast<uint64_t>(row) * static_cast<uint64_t>(cols));
        out_val[w] = rval[i];
        atomicAdd(reinterpret_cast<unsigned long long*>(row_count + row + 1), 1ull);
    }
}

__global__ void minus_one_kernel(int64_t* x, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] -= 1;
}

__global__ void rmat_keys_kernel(RmatParams P, uint64_t* __restrict__ keys, uint32_t* __restrict__ draw) {
    const int H = (P.scale + 3) / 4;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < P.draws;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t row = 0, col = 0, h = 0;
        for (int t = 0; t < P.scale; ++t) {
            if ((t & 3) == 0) h = splitmix64_at(P.edge_seed, static_cast<uint64_t>(e) * H + (t >> 2));
            const uint32_t q = static_cast<uint32_t>(h >> (16 * (t & 3))) & 0xffffu;
            const uint32_t quad = q < P.t_a ? 0u : (q < P.t_ab ? 1u : (q < P.t_abc ? 2u : 3u));
            row = (row << 1) | (quad >> 1);
            col = (col << 1) | (quad & 1u);
        }
        keys[e] = (row << P.scale) | col;
        draw[e] = static_cast<uint32_t>(e);
    }
}

__global__ void head_flags_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// first draw of each run of equal keys -> (column, value), row counts
__global__ void rmat_emit_kernel(RmatParams P, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ draw,
                                 const int64_t* __restrict__ incl, int64_t n, int64_t* __restrict__ out_idx,
                                 double* __restrict__ out_val, int64_t* __restrict__ row_count) {
    const uint64_t mask = (1ull << P.scale) - 1;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i != 0 && keys[i] == keys[i - 1]) continue;
        const int64_t w = incl[i] - 1;
        out_idx[w] = static_cast<int64_t>(keys[i] & mask);
        out_val[w] = P.value_mode == 0 ? 1.0
                                       : (static_cast<double>(splitmix64_at(P.val_seed, draw[i]) >> 11) + 1.0) *
                                             0x1p-53;
        atomicAdd(reinterpret_cast<unsigned long long*>(row_count + (keys[i] >> P.scale) + 1), 1ull);
    }
}

unsigned grid_n(int64_t n) {
    const int64_t g = ceil_div(n, 256);
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32)));
}

}  // namespace

void csr_validate(const int64_t* d_off, const int64_t* d_idx, const double* d_val, int64_t rows, int64_t cols,
                  int64_t nnz, unsigned long long* d_first, cudaStream_t stream) {
    // offsets.front() == 0 and offsets.back() == nnz are checked by the caller
    DSVD_CUDA_CHECK(cudaMemsetAsync(d_first, 0xff, sizeof(unsigned long long), stream));
    if (rows == 0) return;
    csr_validate_kernel<<<static_cast<unsigned>(ceil_div(rows * 32, 256)), 256, 0, stream>>>(d_off, d_idx, d_val,
                                                                                            rows, cols, nnz, d_first);
    DSVD_LAUNCH_CHECK();
}

size_t coo_scratch_bytes(int64_t n) {
    size_t sort_tmp = 0, scan_tmp = 0;
    const int nn = static_cast<int>(n > 0 ? n : 1);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, static_cast<const uint64_t*>(nullptr),
                                    static_cast<uint64_t*>(nullptr), static_cast<const int64_t*>(nullptr),
                                    static_cast<int64_t*>(nullptr), nn);
    cub::DeviceScan::InclusiveSum(nullptr, scan_tmp, static_cast<const int64_t*>(nullptr),
                                  static_cast<int64_t*>(nullptr), nn);
    const size_t a = (static_cast<size_t>(n > 0 ? n : 1) * 8 + 255) / 256 * 256;
    return 10 * a + std::max(sort_tmp, scan_tmp) + 256;
}

int64_t coo_assemble(const int64_t* d_r, const int64_t* d_c, const double* d_v, int64_t n, int64_t rows,
                     int64_t cols, void* scratch, int64_t* d_off, int64_t* d_idx_out, double* d_val_out,
                     int32_t* d_bad, cudaStream_t stream) {
    DSVD_CUDA_CHECK(cudaMemsetAsync(d_off, 0, sizeof(int64_t) * (rows + 1), stream));
    DSVD_CUDA_CHECK(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), stream));
    if (n == 0) return 0;
    const size_t a = (static_cast<size_t>(n) * 8 + 255) / 256 * 256;
    char* p = static_cast<char*>(scratch);
    uint64_t* keys = reinterpret_cast<uint64_t*>(p);
    uint64_t* keys_s = reinterpret_cast<uint64_t*>(p + a);
    int64_t* pos = reinterpret_cast<int64_t*>(p + 2 * a);
    int64_t* pos_s = reinterpret_cast<int64_t*>(p + 3 * a);
    int64_t* head = reinterpret_cast<int64_t*>(p + 4 * a);
    int64_t* hscan = reinterpret_cast<int64_t*>(p + 5 * a);
    uint64_t* rkey = reinterpret_cast<uint64_t*>(p + 6 * a);
    double* rval = reinterpret_cast<double*>(p + 7 * a);
    int64_t* keep = reinterpret_cast<int64_t*>(p + 8 * a);
    int64_t* kscan = reinterpret_cast<int64_t*>(p + 9 * a);
    void* tmp = p + 10 * a;
    size_t tmp_bytes = coo_scratch_bytes(n) - 10 * a;
    coo_keys_kernel<<<grid_n(n), 256, 0, stream>>>(d_r, d_c, n, rows, cols, keys, pos, d_bad);
    DSVD_LAUNCH_CHECK();
    int bits = 1;
    while (bits < 64 && (static_cast<uint64_t>(rows) * static_cast<uint64_t>(cols)) > (1ull << bits)) ++bits;
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_s, pos, pos_s, static_cast<int>(n), 0,
                                                    bits, stream));
    run_heads_kernel<<<grid_n(n), 256, 0, stream>>>(keys_s, n, head);
    DSVD_LAUNCH_CHECK();
    tmp_bytes = coo_scratch_bytes(n) - 10 * a;
    DSVD_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, head, hscan, static_cast<int>(n), stream));
    minus_one_kernel<<<grid_n(n), 256, 0, stream>>>(hscan, n);  // run index of each head
    DSVD_LAUNCH_CHECK();
    int64_t nr = 0;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&nr, hscan + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(stream));
    nr += 1;
    run_sum_kernel<<<grid_n(n), 256, 0, stream>>>(keys_s, pos_s, d_v, hscan, n, rkey, rval, keep);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, keep, kscan, static_cast<int>(nr), stream));
    int64_t last_scan = 0, last_keep = 0;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&last_scan, kscan + nr - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&last_keep, keep + nr - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    compact_kernel<<<grid_n(nr), 256, 0, stream>>>(rkey, rval, keep, kscan, nr, cols, d_idx_out, d_val_out, d_off);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, d_off + 1, d_off + 1, static_cast<int>(rows),
                                                  stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(stream));
    return last_scan + last_keep;
}

size_t rmat_scratch_bytes(int64_t draws) {
    size_t sort_tmp = 0, scan_tmp = 0;
    const int nn = static_cast<int>(draws > 0 ? draws : 1);
    cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, kb, vb, nn);
    cub::DeviceScan::InclusiveSum(nullptr, scan_tmp, static_cast<const int64_t*>(nullptr),
                                  static_cast<int64_t*>(nullptr), nn);
    const size_t n = static_cast<size_t>(draws > 0 ? draws : 1);
    const size_t a8 = (n * 8 + 255) / 256 * 256, a4 = (n * 4 + 255) / 256 * 256;
    return 2 * a8 + 2 * a4 + 2 * a8 + std::max(sort_tmp, scan_tmp) + 256;
}

int64_t rmat_generate(const RmatParams& P, void* scratch, int64_t* d_off, int64_t* d_idx, double* d_val,
                      cudaStream_t stream) {
    const int64_t rows = int64_t(1) << P.scale;
    DSVD_CUDA_CHECK(cudaMemsetAsync(d_off, 0, sizeof(int64_t) * (rows + 1), stream));
    const int64_t n = P.draws;
    if (n == 0) return 0;
    const size_t a8 = (static_cast<size_t>(n) * 8 + 255) / 256 * 256, a4 = (static_cast<size_t>(n) * 4 + 255) / 256 * 256;
    char* p = static_cast<char*>(scratch);
    uint64_t* k0 = reinterpret_cast<uint64_t*>(p);
    uint64_t* k1 = reinterpret_cast<uint64_t*>(p + a8);
    uint32_t* v0 = reinterpret_cast<uint32_t*>(p + 2 * a8);
    uint32_t* v1 = reinterpret_cast<uint32_t*>(p + 2 * a8 + a4);
    int64_t* flag = reinterpret_cast<int64_t*>(p + 2 * a8 + 2 * a4);
    int64_t* incl = reinterpret_cast<int64_t*>(p + 3 * a8 + 2 * a4);
    void* tmp = p + 4 * a8 + 2 * a4;
    size_t tmp_bytes = rmat_scratch_bytes(n) - (4 * a8 + 2 * a4);
    rmat_keys_kernel<<<grid_n(n), 256, 0, stream>>>(P, k0, v0);
    DSVD_LAUNCH_CHECK();
    cub::DoubleBuffer<uint64_t> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, static_cast<int>(n), 0, 2 * P.scale,
                                                    stream));
    const uint64_t* keys = kb.Current();
    const uint32_t* draw = vb.Current();
    head_flags_kernel<<<grid_n(n), 256, 0, stream>>>(keys, n, flag);
    DSVD_LAUNCH_CHECK();
    tmp_bytes = rmat_scratch_bytes(n) - (4 * a8 + 2 * a4);
    DSVD_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, flag, incl, static_cast<int>(n), stream));
    rmat_emit_kernel<<<grid_n(n), 256, 0, stream>>>(P, keys, draw, incl, n, d_idx, d_val, d_off);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, d_off + 1, d_off + 1, static_cast<int>(rows),
                                                  stream));
    int64_t nnz = 0;
    DSVD_CUDA_CHECK(cudaMemcpyAsync(&nnz, incl + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    DSVD_CUDA_CHECK(cudaStreamSynchronize(stream));
    return nnz;
}

}  // namespace dsvd
