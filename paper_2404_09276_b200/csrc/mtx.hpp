// Host-side Matrix Market reader / writer (mtx.cpp). Text parsing stays on the
// host; the triplets it yields are canonicalised on the device (ingest.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace dsvd {

struct MtxTriplets {
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> r, c;
    std::vector<double> v;
};

// Status of a parse: code is DSVD_OK, DSVD_PARSE (line = 1-based line number),
// DSVD_FORMAT (UnsupportedFormat) or DSVD_OTHER (I/O).
struct MtxStatus {
    int code = 0;
    int64_t line = 0;
    std::string what;
};

// load_matrix_market's reading half (matrix_market.cpp:117-165): header,
// size line, entries, symmetric / skew-symmetric expansion, zero filtering.
MtxStatus mtx_read(const char* path, MtxTriplets& out);

// write_matrix_market (matrix_market.cpp:167-177): "coordinate real general", %.17g values.
MtxStatus mtx_write(const char* path, int64_t rows, int64_t cols, const int64_t* offsets,
                    const int64_t* col_indices, const double* values);

struct DenseArray {
    int64_t rows = 0, cols = 0;
    std::vector<double> data;  // column-major
};

// load_dense_array (matrix_market.cpp:179-213): "array" header, size line,
// values in column-major order, any number per line.
MtxStatus dense_read(const char* path, DenseArray& out);
// write_dense_array (:215-223): "array real general", %.17g, column-major.
MtxStatus dense_write(const char* path, int64_t rows, int64_t cols, const double* colmajor);

// load_reference_spectrum / write_reference_spectrum (metrics.cpp:65-97): one
// non-negative, non-increasing value per line, blank lines and '#' comments skipped.
MtxStatus spectrum_read(const char* path, std::vector<double>& out);
MtxStatus spectrum_write(const char* path, const double* sigmas, int64_t n);

}  // namespace dsvd
