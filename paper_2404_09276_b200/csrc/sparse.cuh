// Device CSR storage and the sparse kernels of the power loop.
#pragma once

#include "common.cuh"

namespace dsvd {

// Canonical CSR on the device. Offsets stay int64 (nnz may exceed 2^31 at
// config 5); column indices are int32 (every dimension here is < 2^31), which
// cuts the per-nonzero stream from 16 to 12 bytes. `order` lists the rows by
// nonzero count, longest first, so SpMM starts hub rows first.
struct DevCsr {
    int64_t rows = 0, cols = 0, nnz = 0;
    int64_t* off = nullptr;
    int32_t* idx = nullptr;
    double* val = nullptr;
    int32_t* order = nullptr;
    // CSR range of row order[i] in order sequence (obeg[i] = off[order[i]],
    // olen[i] its length), so the column-slab kernel reads a row's range with one
    // load beside order[i] instead of a dependent off[] lookup; optional
    int64_t* obeg = nullptr;
    int32_t* olen = nullptr;
    int64_t max_row_nnz = 0;
    // every stored value has the bits of uval (e.g. an unweighted graph's 1.0):
    // the column-slab kernel then multiplies by uval instead of streaming the
    // values; fma(uval, x, acc) is the same operation on the same operands, so
    // the chains are bitwise unchanged (set at build time from a device scan)
    bool uniform = false;
    double uval = 0.0;
    // rows order[0 .. hub_rows) hold >= hub_threshold nonzeros and take the
    // deep-pipelined hub path of spmm (counted on the device at build time)
    int64_t hub_rows = 0;
    int64_t hub_threshold = 0;
    int32_t* d_hub_rows = nullptr;  // device copy written by build_row_order
    // rows with at least one nonzero: the prefix order[0 .. nonempty_rows) (-1:
    // unknown, every row is treated as non-empty); d_nonempty is the device count
    int64_t nonempty_rows = -1;
    int32_t* d_nonempty = nullptr;
    // rows with more than kShortRow nonzeros: the prefix order[0 .. long_rows);
    // the column-slab kernel runs the short rows after them in a leaner,
    // higher-occupancy launch (their time is the per-row latency chain)
    int64_t long_rows = -1;
    int32_t* d_long = nullptr;
    // rows with more than kMidRow nonzeros: the prefix order[0 .. mid_rows) (the
    // whole-row short-row kernel may take the rows after it; -1: unknown)
    int64_t mid_rows = -1;
    int32_t* d_mid = nullptr;
    // Split mode (split_chunk > 0): rows order[0 .. nsplit) hold more than
    // split_chunk nonzeros and are cut into nchunks CSR ranges of at most
    // split_chunk nonzeros; each chunk's FMA chain goes to a partial row and the
    // partials of a row are summed in chunk order (deterministic, not the
    // reference's single chain). split_chunk == 0 keeps every chain whole
    // (bit-exact, hub rows take the hub kernel).
    int64_t split_chunk = 0;
    int64_t nsplit = 0, nchunks = 0;
    int64_t* chunk_p0 = nullptr;     // nchunks: first nonzero of the chunk
    int64_t* chunk_p1 = nullptr;     // nchunks: one past the last nonzero
    int32_t* split_first = nullptr;  // nsplit+1: chunk range of split row i
    // chunk_slot[split_first[i] + t] = position in chunk_p0/p1 (and in the
    // partial rows) of split row i's t-th chunk; null = identity. The chunk
    // list itself is ordered by X-row panel (see build_chunks) so chunks
    // running together gather from an L2-resident slice of X.
    int32_t* chunk_slot = nullptr;
    int64_t max_row_chunks = 0;  // most chunks of one split row (picks the combine kernel)
};

constexpr int kShortRow = 8;
constexpr int kMidRow = 32;

// SpMM launch description. X and Y (and Q) are row-major with row stride ld.
struct SpmmArgs {
    const DevCsr* a;
    const double* x;      // a.cols x ld
    double* y;            // a.rows x ld
    int64_t ld;
    int64_t l;            // logical width (<= ld)
    const double* q;      // shift operand (a.rows x ld) or nullptr
    const double* alpha;  // device scalar: y = fma(-alpha, q, A x) unless alpha == 0
    const int32_t* gate;  // device flag: skip the launch's work when *gate != 0 (or nullptr)
    // Slab-major layouts (column-slab kernel only, slab width `slab`): element
    // (i, j) of an r-row block at (j / slab) * r * slab + i * slab + j % slab,
    // so one slab of X is contiguous (tools/micro/gather_tlb.cu: 256-byte
    // gathers from a contiguous 1 GB slab run at 16.7 TB/s, from the same
    // bytes spread over a 10 GB row-major block at 10.7 TB/s).
    int slab = 0;         // 0: every block row-major with stride ld
    bool x_slab = false;  // X is slab-major (a.cols rows)
    bool y_slab = false;  // write Y slab-major (a.rows rows); the shift operand q stays row-major
    // hot/cold-tagged copy of a.idx (tag_hot_indices) for the column-slab kernel's
    // L2 eviction priorities, or nullptr
    const int32_t* idx_tag = nullptr;
    // column-slab kernel: rows without nonzeros (the tail of a.order) are not
    // written at all (their Y rows are never read, e.g. the loop's A Q), instead
    // of being set to 0 (or -alpha q)
    bool skip_empty = false;
};

// idx_tag = m.idx with the sign bit set on every index outside the hot set, the
// k X rows listed first in order_x (the most referenced: the row order of the
// other matrix of the pair). hot is an m.cols-byte scratch.
void tag_hot_indices(const DevCsr& m, const int32_t* order_x, int64_t k, uint8_t* hot, int32_t* idx_tag,
                     cudaStream_t stream);

// Index of element (i, j) of an r-row block in the slab-major layout of width w.
inline int64_t slab_index(int64_t i, int64_t j, int64_t r, int w) { return (j / w) * r * w + i * w + j % w; }
// Doubles of an r-row, width-ld block in the slab-major layout of width w.
inline int64_t slab_block_size(int64_t r, int64_t ld, int w) { return ceil_div(ld, w) * w * r; }
// Row-major (stride ld) <-> slab-major (width w) copies of an r-row block.
void to_slab_major(const double* src, int64_t rows, int64_t ld, int w, double* dst, cudaStream_t stream);
void from_slab_major(const double* src, int64_t rows, int64_t ld, int w, double* dst, cudaStream_t stream);

// Launches the hub-row kernel on `side` (when the matrix has hub rows) and the
// kernel for all other rows on `stream`; `fork`/`join` order the two streams.
// bounds[r * (npanel + 1) + p] = first nonzero of split row r (the r-th row of
// m.order) whose index is >= p * panel_rows; p = npanel gives the row end.
// Requires sorted indices within each row (true for the transpose).
void panel_bounds(const DevCsr& m, int64_t nrows, int npanel, int64_t panel_rows, int64_t* bounds,
                  cudaStream_t stream);

void spmm(const SpmmArgs& args, cudaStream_t stream, int variant, cudaStream_t side = nullptr,
          cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr, double* partial = nullptr);

// Split-row chunk plan on the device (no host round trip but one scalar read):
// chunk_plan_count fills row_nch[rows] (chunks per row of m.order, 0 beyond the
// *m.d_hub_rows split rows), first[rows + 1] (their inclusive prefix, first[0] =
// 0 — the split_first array) and d_total_max = {total chunks, most chunks of one
// row}; chunk_plan_emit then writes the nc chunk ranges p0/p1 — in CSR order
// when npanel <= 1, else stably ordered by panel with slot[id] = list position.
size_t chunk_plan_scratch_bytes(int64_t rows, int64_t max_chunks);
void chunk_plan_count(const DevCsr& m, int npanel, int64_t panel_rows, int32_t* row_nch, int32_t* first,
                      int32_t* d_total_max, void* temp, size_t temp_bytes, cudaStream_t stream);
void chunk_plan_emit(const DevCsr& m, int64_t ns, int npanel, int64_t panel_rows, const int32_t* first, int64_t nc,
                     int64_t* p0, int64_t* p1, int32_t* slot, int64_t* tmp0, int64_t* tmp1, int32_t* keys,
                     int32_t* keys_sorted, int32_t* ids, int32_t* ids_sorted, void* temp, size_t temp_bytes,
                     cudaStream_t stream);

// Row bounds (offsets) of the first n rows of m.order, for the host-side
// construction of the split chunk list.
void prefix_row_bounds(const DevCsr& m, int64_t n, int64_t* d_beg, int64_t* d_end,
                       cudaStream_t stream);

// CSR(A^T) from CSR(A), bitwise equal to the reference transpose().
// Temporaries come from `scratch` (bytes given by csc_scratch_bytes).
size_t csc_scratch_bytes(int64_t rows, int64_t cols, int64_t nnz);
void build_transpose(const DevCsr& a, DevCsr& at, void* scratch, size_t scratch_bytes,
                     cudaStream_t stream, cudaEvent_t values_ready = nullptr);
// Row order by nonzero count (descending, ties by row index) into m.order,
// and the number of rows with >= m.hub_threshold nonzeros into *m.d_hub_rows.
size_t order_scratch_bytes(int64_t rows);
void build_row_order(DevCsr& m, void* scratch, size_t scratch_bytes, cudaStream_t stream);
// The short rows of the column-slab SpMM as whole rows: 0 off (per-slab items), 1 rows of
// at most kShortRow nonzeros, 2 rows of at most kMidRow nonzeros
void set_spmm_short_rows(int v);

// Compaction of a CSR's empty rows (engine.cu build_compact): newid[r] = the
// rank of row r among the non-empty rows (-1 if empty), oldid its inverse,
// off_c the offsets of the non-empty rows (positions unchanged) + nnz.
size_t compact_scratch_bytes(int64_t rows);
void compact_rows_map(const int64_t* off, int64_t rows, int32_t* newid, int32_t* oldid, int64_t* off_c,
                      void* scratch, size_t scratch_bytes, cudaStream_t stream);
// out[i] = map[in[i]] (column indices, row orders)
void remap_ids(const int32_t* in, int64_t n, const int32_t* map, int32_t* out, cudaStream_t stream);
// dst (rows x k, column-major, leading dim rows) = 0 except rows oldid[i] =
// src row i (src: rows_c x k column-major)
void scatter_rows_colmajor(const double* src, int64_t rows_c, int64_t k, const int32_t* oldid, double* dst,
                           int64_t rows, cudaStream_t stream);

// int64 -> int32 column indices with a bounds check; *bad is set to 1 when an
// index falls outside [0, cols) (the entry is clamped so no kernel faults).
void narrow_indices(const int64_t* src, int32_t* dst, int64_t nnz, int64_t cols, int32_t* bad,
                    cudaStream_t stream);
void widen_indices(const int32_t* src, int64_t* dst, int64_t nnz, cudaStream_t stream);
// *nonuniform = 1 unless all nnz values have the bits of val[0]; *first = val[0]
void check_uniform_values(const double* val, int64_t nnz, int32_t* nonuniform, double* first,
                          cudaStream_t stream);
// Offset checks: off[0] == 0, off[rows] == nnz, non-decreasing -> *bad = 1 otherwise.
void check_offsets(const int64_t* off, int64_t rows, int64_t nnz, int32_t* bad,
                   cudaStream_t stream);

}  // namespace dsvd
