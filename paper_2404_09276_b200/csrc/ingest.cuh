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

}  // namespace dsvd
