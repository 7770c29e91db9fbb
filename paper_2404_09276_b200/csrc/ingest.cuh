// Device-side input handling: CSR validation and COO canonicalisation (ingest.cu).
#pragma once

#include "common.cuh"

namespace dsvd {

// d_first (device) <- min over violating rows of (row << 3 | code), or all ones.
void csr_validate(const int64_t* d_off, const int64_t* d_idx, const double* d_val, int64_t rows, int64_t cols,
                  int64_t nnz, unsigned long long* d_first, cudaStream_t stream);

size_t coo_scratch_bytes(int64_t n);
// Canonical CSR from n triplets (device arrays); outputs must hold n entries
// (d_off rows + 1). Returns nnz after summing duplicates and dropping zeros.
// *d_bad = 1 when an index is out of range.
int64_t coo_assemble(const int64_t* d_r, const int64_t* d_c, const double* d_v, int64_t n, int64_t rows,
                     int64_t cols, void* scratch, int64_t* d_off, int64_t* d_idx_out, double* d_val_out,
                     int32_t* d_bad, cudaStream_t stream);

// R-MAT edge generator (BASELINE.json configs 4/5), on the device.
// Draw e (0 <= e < draws) descends `scale` levels; level t takes 16 bits of
// splitmix64_at(edge_seed, e * H + t / 4), H = ceil(scale / 4), bits
// [16 (t % 4), 16 (t % 4) + 16), and picks quadrant 0/1/2/3 when they are
// below t_a / t_ab / t_abc / otherwise (row bit = quadrant >> 1, column bit =
// quadrant & 1, most significant first). Duplicate edges keep the first draw;
// its value is 1.0 (value_mode 0) or ((splitmix64_at(val_seed, e) >> 11) + 1)
// * 2^-53 in (0, 1] (value_mode 1). Output: canonical CSR (2^scale square).
struct RmatParams {
    int scale;
    int64_t draws;
    uint32_t t_a, t_ab, t_abc;
    int value_mode;
    uint64_t edge_seed, val_seed;
};
size_t rmat_scratch_bytes(int64_t draws);
// d_off (2^scale + 1), d_idx (int64), d_val sized for `draws`; returns nnz
int64_t rmat_generate(const RmatParams& P, void* scratch, int64_t* d_off, int64_t* d_idx, double* d_val,
                      cudaStream_t stream);

}  // namespace dsvd
