/* dashsvd_b200.h — C ABI of the B200-native dashSVD hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or CUDA
 * types. Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core/include/dashsvd/ and
 * .../core/src/). include/dashsvd_b200.hpp wraps it in the reference's own
 * C++ API (dashsvd::solve & co.), and paper_2404_09276_b200/ binds it from
 * Python with ctypes.
 *
 * Conventions
 *  - Host dense matrices are column-major (dense_matrix.hpp:10-13).
 *  - Sparse input is canonical CSR with int64 offsets and int64 column
 *    indices and fp64 values (sparse_matrix.hpp:10-26); it is borrowed for the
 *    duration of the call only.
 *  - Every call returns a status (DSVD_OK or an error below). On error,
 *    dsvd_last_error() returns the message and dsvd_last_error_index() the
 *    RankDeficient index (errors.hpp:37-43), both thread-local.
 *  - A context owns one CUDA stream and its workspaces; it is NOT safe for
 *    concurrent solves from several threads (create one context per thread).
 *  - Results are deterministic run to run on a fixed GPU count: no float
 *    atomics, fixed reduction trees.
 */
#ifndef DASHSVD_B200_H
#define DASHSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DSVD_API __attribute__((visibility("default")))
#else
#define DSVD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped onto errors.hpp:10-59 by the wrappers) -------- */
enum {
    DSVD_OK = 0,
    DSVD_SHAPE = 1,         /* ShapeError                                   */
    DSVD_CONFIG = 2,        /* ConfigError                                  */
    DSVD_RANK_DEFICIENT = 3,/* RankDeficient{index}                         */
    DSVD_NUMERICAL = 4,     /* NumericalError (eig non-convergence, NaN)    */
    DSVD_CUDA = 5,          /* CUDA runtime failure (reference: Error)      */
    DSVD_OOM = 6,           /* device allocation failed (reference: Error)  */
    DSVD_NCCL = 7,          /* collective failure (reference: Error)        */
    DSVD_UNSUPPORTED = 8,   /* configuration outside the B200 path          */
    DSVD_OTHER = 9,
    DSVD_DEGENERATE = 10,   /* DegenerateReference (metrics)                */
    DSVD_FORMAT = 11,       /* UnsupportedFormat (cache / Matrix Market)    */
    DSVD_PARSE = 12         /* ParseError; dsvd_last_error_index() = line   */
};

/* Algorithm and StopReason keep the reference enum order (solver.hpp:13-18, :45). */
enum { DSVD_ALG_BASIC = 0, DSVD_ALG_SHIFTED = 1, DSVD_ALG_FIXED_SHIFT = 2, DSVD_ALG_DASH = 3 };
enum { DSVD_STOP_FIXED_P = 0, DSVD_STOP_TOL_MET = 1, DSVD_STOP_P_MAX_REACHED = 2 };

typedef struct dsvd_ctx dsvd_ctx;       /* device, stream, workspaces, optional NCCL comm */
typedef struct dsvd_matrix dsvd_matrix; /* device-resident CSR(A) + CSR(A^T)              */
typedef struct dsvd_loopback dsvd_loopback; /* in-process rank group (testing)            */

/* SolverConfig (solver.hpp:22-38). s < 0 means the default max(1, k/2).
 * flags: DSVD_FLAG_DIRECT runs the algorithm on `a` as given, like
 * shifted_rsvd / dash_svd (solver.cpp:190-212); without it the entry point
 * behaves like solve(), which factors the transpose of wide inputs and swaps
 * U and V (solver.cpp:217-220). DSVD_FLAG_ORTH_QR selects the QR
 * orthonormalizer of the basic algorithm (Orthonormalizer::qr, solver.hpp:20). */
enum { DSVD_FLAG_DIRECT = 1, DSVD_FLAG_ORTH_QR = 2 };
typedef struct {
    int64_t k;
    int64_t s;
    int64_t p;
    double tol;
    int64_t p_max;
    int32_t alg;
    int32_t flags;
    uint64_t seed;
} dsvd_config;

/* SolveResult (solver.hpp:51-61), caller-allocated.
 *   u[m*k], s[k], v[n*k] column-major; alphas[trace_cap], s_hat[trace_cap*l]
 *   (either trace pointer may be NULL). With outputs_on_device != 0 the
 *   u/s/v pointers are device pointers on the context's GPU (no D2H copy).
 *   iterations / stop_reason are written by the call. */
typedef struct {
    double* u;
    double* s;
    double* v;
    double* alphas;
    double* s_hat;
    int64_t trace_cap;
    int64_t iterations;
    int32_t stop_reason;
    int32_t outputs_on_device;
} dsvd_outputs;

/* IterationObserver (solver.hpp:63-74): called synchronously after each
 * power iteration's re-orthonormalisation, before the stop check. q_before /
 * q_after are HOST column-major n x l copies valid only during the callback. */
typedef void (*dsvd_observer_fn)(int64_t iteration, double alpha, const double* s_hat,
                                 int64_t l, const double* q_before, const double* q_after,
                                 int64_t n, void* user);

/* Per-context counters, filled when profiling is on (dsvd_ctx_set_profiling).
 * Times are device milliseconds measured with CUDA events on the context's
 * stream, summed over the last solve. */
typedef struct {
    double total_ms;        /* whole solve call                                  */
    double h2d_ms;          /* CSR upload (host-input entry points only)         */
    double csc_ms;          /* CSR -> CSR(A^T) construction                      */
    double omega_ms;        /* Gaussian sketch generation                        */
    double sketch_ms;       /* A^T Omega + first eigSVD                          */
    double loop_ms;         /* power iterations                                  */
    double finalize_ms;     /* B = A Q, eigSVD(B), U/V assembly                  */
    double d2h_ms;          /* result download (host-output entry points only)   */
    double spmm_ms;         /* all SpMM passes (A X and A^T Y - alpha Q)         */
    double gram_ms;         /* Gram partials + reduction                         */
    double eig_ms;          /* Jacobi eigensolver + rotation replay + finish     */
    double rescale_ms;      /* Q = T V diag(1/s) (and finalize U, V products)    */
    double allreduce_ms;    /* collectives of a row-sharded solve (multi-GPU)     */
    int64_t spmm_launches;
    int64_t kernel_launches;/* every kernel this library launched in the solve    */
    int64_t eig_sweeps;     /* Jacobi sweeps summed over all eigensolves          */
    int64_t spmm_bytes;     /* algorithmic SpMM bytes (SURVEY 8d B1/B2 formulas)  */
    double spmm_pass_ms[2]; /* pass 1 (A Q) and pass 2 (A^T Y - alpha Q), summed  */
    int64_t spmm_pass_bytes[2];
    int64_t spmm_pass_launches[2];
    int64_t pipelined;      /* loop schedule of the last solve: 1 pipelined, 0 serial */
} dsvd_stats;

/* ---- errors --------------------------------------------------------------- */
DSVD_API const char* dsvd_last_error(void);
DSVD_API long long dsvd_last_error_index(void);
DSVD_API const char* dsvd_version(void);

/* ---- context -------------------------------------------------------------- */
DSVD_API int dsvd_ctx_create(int device, dsvd_ctx** out);
DSVD_API int dsvd_ctx_destroy(dsvd_ctx* ctx);
DSVD_API int dsvd_ctx_set_profiling(dsvd_ctx* ctx, int on);
DSVD_API int dsvd_ctx_get_stats(const dsvd_ctx* ctx, dsvd_stats* out);
DSVD_API int dsvd_ctx_synchronize(dsvd_ctx* ctx);
/* Free the context's cached device workspaces (they are re-allocated on the
 * next call); matrix handles keep their own buffers. For very large inputs
 * that alternate between entry points. */
DSVD_API int dsvd_ctx_trim(dsvd_ctx* ctx);
/* Tuning knobs (testing/benchmarking); unknown names -> DSVD_CONFIG.
 * Loop schedule: "pipeline" -1 auto (default) / 0 serial /
 * 1 pipelined; "eig_priority" 1 (default) / 0; "gram_async" 0 (default) / 1;
 * "eig_overlap" -1 auto (default) / 2 tridiagonalisation beside the A T pass,
 * rest after it / 1 whole eig chain beside it / 0 none.
 * Row-sharded solves: "mgpu_mode" 2 (default: reduce-scatter + slab dense work
 * + all-gather) / 1 (all-reduce of the n x l partials, dense work redundant);
 * "mgpu_overlap" 1 (default: the A^T pass in G row panels, each panel's partial
 * reduced on a communication stream while the next panel computes) / 0 / 2 (v2:
 * each panel's rows stored by the SpMM straight into the owner's landing buffer
 * over peer memory — CUDA IPC under NCCL — then a barrier and the owner's sum).
 * Kernels: "spmm_variant", "split_chunk", "split_chunk_t", "split_panel_rows",
 * "hub_threshold", "eig_method", "dense_method"; column-slab SpMM: "spmm_slab"
 * (-1 auto / 0 / 32 / 64), "slab_layout", "spmm_slab_hint", "spmm_slab_depth",
 * "spmm_hot_mb", "uniform_values" (1 default: all-equal values are detected at
 * build time and not streamed; 0: always streamed).
 * Host buffers: "host_staging" 1 (default: PAGEABLE host inputs / outputs of a
 * solve — std::vector, numpy — move through a ring of 4 pinned slots, the copy
 * engine streaming one slot while host threads fill or drain another) / 0 (plain
 * cudaMemcpyAsync through the driver's bounce buffer); "host_stage_chunk" bytes
 * per slot (default 32 MB); "host_copy_threads" (0 default: min(16, cores)).
 * Pinned (dsvd_host_register / cudaHostAlloc) and device pointers are copied
 * directly either way. */
DSVD_API int dsvd_ctx_set_option(dsvd_ctx* ctx, const char* name, int64_t value);

/* Multi-GPU: one process per GPU. Rank 0 calls dsvd_comm_unique_id and
 * broadcasts the 128 bytes out of band (torch.distributed in the Python
 * layer); every rank then calls dsvd_ctx_attach_comm. A solve on an attached
 * context treats the matrix it gets as that rank's row shard. */
DSVD_API int dsvd_comm_unique_id(uint8_t out[128]);
DSVD_API int dsvd_ctx_attach_comm(dsvd_ctx* ctx, int nranks, int rank, const uint8_t id[128]);
/* In-process rank group (testing the row-sharded engine without a multi-GPU
 * node): nranks (<= 8) contexts of ONE process, each driven by its own host
 * thread, attach to the group; every collective synchronises the rank's
 * stream, meets the others at a host barrier and sums their device buffers in
 * fixed rank order. The contexts may share one GPU (no kernel waits on another
 * rank). Destroy the group after every attached context. */
DSVD_API int dsvd_loopback_create(int nranks, dsvd_loopback** out);
DSVD_API int dsvd_loopback_destroy(dsvd_loopback* group);
DSVD_API int dsvd_ctx_attach_loopback(dsvd_ctx* ctx, dsvd_loopback* group, int rank);
/* Row-shard placement used by dsvd_solve_csr / dsvd_solve_csr_device on an
 * attached context: the CSR passed is rows [row_offset, row_offset + rows) of
 * a global_rows x cols matrix. */
DSVD_API int dsvd_ctx_set_shard(dsvd_ctx* ctx, int64_t row_offset, int64_t global_rows);

/* ---- pinned host memory (for zero-copy-speed H2D/D2H of caller buffers) --- */
DSVD_API int dsvd_host_register(void* ptr, size_t bytes);
DSVD_API int dsvd_host_unregister(void* ptr);

/* ---- matrix handle: upload once, solve many -------------------------------
 * Replaces holding (a, transpose(a)) for the overloads taking a precomputed
 * transpose (solver.hpp:106-116). Builds CSR(A^T) on the device, bitwise
 * equal to transpose(a) (sparse_matrix.cpp:35-55). */
DSVD_API int dsvd_matrix_upload(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                       const int64_t* offsets, const int64_t* col_indices,
                       const double* values, dsvd_matrix** out);
/* Same, from DEVICE pointers on the context's GPU (inputs resident in HBM). */
DSVD_API int dsvd_matrix_from_device(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                            const int64_t* d_offsets, const int64_t* d_col_indices,
                            const double* d_values, dsvd_matrix** out);
DSVD_API int dsvd_matrix_destroy(dsvd_matrix* m);
/* Declare the handle a row shard: rows [row_offset, row_offset + rows) of a
 * global_rows x cols matrix (multi-GPU solves; see dsvd_ctx_attach_comm). */
DSVD_API int dsvd_matrix_set_shard(dsvd_matrix* m, int64_t row_offset, int64_t global_rows);
DSVD_API int dsvd_matrix_shape(const dsvd_matrix* m, int64_t* rows, int64_t* cols, int64_t* nnz);
/* Microbenchmark the SpMM of A (transpose = 0) or A^T (transpose = 1) on a
 * random l-column block: average milliseconds over `iters` launches.
 * variant: the spmm_variant bits (0 = the default kernels; +16 skips the bulk
 * rows, +32 the long rows; 4096 / 8192 the 32- / 64-column slab kernel). dsvd_matrix_hub_rows reports how many
 * rows of A / A^T take the hub path (option "hub_threshold"). */
DSVD_API int dsvd_matrix_bench_spmm(dsvd_matrix* m, int transpose, int64_t l, int variant,
                                    int iters, double* ms_out);
DSVD_API int dsvd_matrix_hub_rows(const dsvd_matrix* m, int64_t* hub_a, int64_t* hub_at);
/* Download CSR(A) as stored on the device (int64 offsets/indices, host buffers). */
DSVD_API int dsvd_matrix_download(const dsvd_matrix* m, int64_t* offsets, int64_t* col_indices, double* values);
/* Rows [r0, r1) of CSR(A) (offsets rebased to 0; r1 - r0 + 1 offsets), e.g. one
 * rank's row shard of a matrix generated on the device. */
DSVD_API int dsvd_matrix_download_rows(const dsvd_matrix* m, int64_t r0, int64_t r1, int64_t* offsets,
                                       int64_t* col_indices, double* values);
/* The rows + 1 offsets of CSR(A). */
DSVD_API int dsvd_matrix_row_offsets(const dsvd_matrix* m, int64_t* offsets);
/* Download the device-built transpose (int64 offsets/indices, host buffers). */
DSVD_API int dsvd_matrix_download_transpose(const dsvd_matrix* m, int64_t* t_offsets,
                                   int64_t* t_col_indices, double* t_values);

/* ---- solvers --------------------------------------------------------------
 * dsvd_solve             <- solve(a, at, cfg, observer)   solver.hpp:115-116 / solver.cpp:214-223
 * dsvd_solve_csr         <- solve(a, cfg)                 solver.hpp:104 / solver.cpp:225-227
 *                           (host CSR in, host U/S/V out; transpose built on device)
 * alg == DSVD_ALG_SHIFTED / FIXED_SHIFT / DASH run the shifted family
 * (shifted_rsvd :95 / dash_svd :99); alg == BASIC runs basic_core +
 * finalize_col_basis (solver.cpp:118-141, :166-176), with the QR
 * orthonormalizer when cfg->flags has DSVD_FLAG_ORTH_QR (l <= 160). */
DSVD_API int dsvd_solve(dsvd_ctx* ctx, const dsvd_matrix* a, const dsvd_config* cfg, dsvd_outputs* out,
               dsvd_observer_fn observer, void* user);
DSVD_API int dsvd_solve_csr(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                   const int64_t* offsets, const int64_t* col_indices, const double* values,
                   const dsvd_config* cfg, dsvd_outputs* out);
/* Same as dsvd_solve_csr with the CSR already in device memory (inputs
 * resident in HBM); the transpose is built inside the call, as solve(a, cfg)
 * does. Workspaces are cached in the context, so repeated calls allocate nothing. */
DSVD_API int dsvd_solve_csr_device(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                          const int64_t* d_offsets, const int64_t* d_col_indices,
                          const double* d_values, const dsvd_config* cfg, dsvd_outputs* out);

/* Device-side interval timer on the context's stream (CUDA events). */
DSVD_API int dsvd_ctx_timer_start(dsvd_ctx* ctx);
DSVD_API int dsvd_ctx_timer_stop(dsvd_ctx* ctx, double* elapsed_ms);

/* finalize_row_basis (solver.hpp:123, solver.cpp:159-164): host q (cols x l,
 * column-major) -> host u[rows*k], s[k], v[cols*k]. */
DSVD_API int dsvd_finalize_row_basis(dsvd_ctx* ctx, const dsvd_matrix* a, const double* q, int64_t l,
                            int64_t k, double* u, double* s, double* v);

/* ---- inputs -------------------------------------------
 * dsvd_csr_validate     <- SparseMatrix::validate()        sparse_matrix.cpp:12-33
 *   (on the device; same first violation and error type: ShapeError for
 *   offsets / index range / ordering, NumericalError for non-finite or
 *   explicit-zero values, message naming the row)
 * dsvd_save_cache       <- save_cache(path, a)             matrix_market.cpp:~241-255 (DSH1)
 * dsvd_matrix_load_cache<- load_cache(path) + validate()   matrix_market.cpp:257-275,
 *   read into pinned memory and uploaded; the device matrix handle is built
 *   directly (dims[3] receives rows, cols, nnz). DSVD_FORMAT: bad magic or
 *   truncated file.
 * dsvd_coo_assemble     <- assemble(rows, cols, triplets)  matrix_market.cpp:90-115
 *   (sort by (row, col), duplicates summed in input order, exact zeros
 *   dropped; *nnz receives the canonical count); dsvd_coo_fetch copies the
 *   resulting CSR to host arrays, dsvd_matrix_from_coo builds the device
 *   matrix handle from it without a host round trip.
 * dsvd_mtx_assemble     <- load_matrix_market(path)        matrix_market.cpp:117-165
 *   (text parsed on the host with the reference's errors: DSVD_PARSE with the
 *   1-based line in dsvd_last_error_index(), DSVD_FORMAT for unsupported
 *   headers, DSVD_OTHER when the file cannot be opened; the triplets are then
 *   assembled on the device as dsvd_coo_assemble; dims[3] = rows, cols, nnz)
 * dsvd_mtx_read / dsvd_mtx_fetch: the host parsing half alone (dims[3] = rows,
 *   cols, number of triplets after the symmetric expansion; fetch hands the
 *   0-based triplets out in file order and releases them)
 * dsvd_write_matrix_market <- write_matrix_market(path, a) matrix_market.cpp:167-177 */
DSVD_API int dsvd_csr_validate(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                               const int64_t* col_indices, const double* values);
DSVD_API int dsvd_save_cache(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
                             const int64_t* col_indices, const double* values);
DSVD_API int dsvd_matrix_load_cache(dsvd_ctx* ctx, const char* path, int validate, dsvd_matrix** out,
                                    int64_t* dims);
DSVD_API int dsvd_coo_assemble(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* r,
                               const int64_t* c, const double* v, int64_t* nnz);
DSVD_API int dsvd_coo_fetch(dsvd_ctx* ctx, int64_t* offsets, int64_t* col_indices, double* values);
DSVD_API int dsvd_matrix_from_coo(dsvd_ctx* ctx, dsvd_matrix** out);
DSVD_API int dsvd_mtx_assemble(dsvd_ctx* ctx, const char* path, int64_t* dims);
DSVD_API int dsvd_mtx_read(const char* path, int64_t* dims);
DSVD_API int dsvd_mtx_fetch(int64_t* r, int64_t* c, double* v);
DSVD_API int dsvd_write_matrix_market(const char* path, int64_t rows, int64_t cols, const int64_t* offsets,
                                      const int64_t* col_indices, const double* values);
/* Dense factor files and reference spectra (host text, used by the CLI):
 * dsvd_dense_read/_fetch   <- load_dense_array(path)          matrix_market.cpp:179-213
 *                             (dims[2] = rows, cols; fetch copies column-major)
 * dsvd_dense_write         <- write_dense_array(path, a)      :215-223
 * dsvd_spectrum_read/_fetch<- load_reference_spectrum(path)   metrics.cpp:71-90
 * dsvd_spectrum_write      <- write_reference_spectrum(path)  :92-97
 * Errors as the reference: DSVD_PARSE (line), DSVD_FORMAT, DSVD_OTHER (I/O). */
DSVD_API int dsvd_dense_read(const char* path, int64_t* dims);
DSVD_API int dsvd_dense_fetch(double* colmajor);
DSVD_API int dsvd_dense_write(const char* path, int64_t rows, int64_t cols, const double* colmajor);
DSVD_API int dsvd_spectrum_read(const char* path, int64_t* n);
DSVD_API int dsvd_spectrum_fetch(double* sigmas);
DSVD_API int dsvd_spectrum_write(const char* path, const double* sigmas, int64_t n);
/* R-MAT generator on the device (BASELINE.json configs 4/5; no reference
 * counterpart: the reference ships only sparse_random). Draws `draws` edges of
 * a 2^scale square graph with quadrant probabilities (a, b, c, 1-a-b-c) at
 * 16-bit resolution from counter-based SplitMix64 streams (ingest.cuh spells
 * out the rule), keeps the first draw of every duplicate edge, values 1.0
 * (value_mode 0) or uniform (0, 1] (value_mode 1), and builds the device pair
 * directly. *nnz receives the unique edge count; dsvd_matrix_download copies
 * the CSR to the host (e.g. for the CPU reference). */
DSVD_API int dsvd_synth_rmat(dsvd_ctx* ctx, int scale, int64_t draws, double a, double b, double c, int value_mode,
                             uint64_t seed, dsvd_matrix** out, int64_t* nnz);

/* ---- validation metrics (metrics.hpp / metrics.cpp:99-206) ----------------
 * Host factors (column-major u[rows*k], s[k], v[cols*k]) against the device
 * matrix; reference singular values sigmas[n_ref] descending. Reductions are
 * deterministic trees (values agree with the reference to rounding).
 * dsvd_eps_pve              <- eps_pve(a, u_hat, ref)           metrics.cpp:99-117
 * dsvd_eps_res              <- eps_res(a, approx, ref)          metrics.cpp:119-134
 * dsvd_eps_spec             <- eps_spec(a, approx, ref, it, seed) metrics.cpp:136-159
 * dsvd_max_triplet_residual <- max_triplet_residual(a, approx)  metrics.cpp:194-206
 * A reference that is too short or has a zero where one is divided by returns
 * DSVD_DEGENERATE (DegenerateReference). */
DSVD_API int dsvd_eps_pve(dsvd_ctx* ctx, const dsvd_matrix* a, const double* u, int64_t k, const double* sigmas,
                          int64_t n_ref, double* out);
DSVD_API int dsvd_eps_res(dsvd_ctx* ctx, const dsvd_matrix* a, const double* u, const double* s, const double* v,
                          int64_t k, const double* sigmas, int64_t n_ref, double* out);
DSVD_API int dsvd_eps_spec(dsvd_ctx* ctx, const dsvd_matrix* a, const double* u, const double* s, const double* v,
                           int64_t k, const double* sigmas, int64_t n_ref, int64_t power_iters, uint64_t seed,
                           double* out);
DSVD_API int dsvd_max_triplet_residual(dsvd_ctx* ctx, const dsvd_matrix* a, const double* u, const double* s,
                                       const double* v, int64_t k, double* out);

/* validate_config (solver.cpp:15-32), update_shift (:34-36), pve_stop_check
 * (:38-50): pure host functions with the reference's semantics; the device
 * loop evaluates the same expressions in the same order. */
DSVD_API int dsvd_validate_config(const dsvd_config* cfg, int64_t rows, int64_t cols);
DSVD_API double dsvd_update_shift(double alpha, double s_ll);
DSVD_API int dsvd_pve_stop_check(const double* s_hat_prev, int64_t n_prev, double alpha_prev,
                        const double* s_hat, int64_t n, double alpha, int64_t k, double tol,
                        int* stop);

/* ---- kernel-level entry points (host buffers in/out; for parity tests) ---
 * Each runs exactly the device kernel the solver uses. */
/* spmm (sparse_matrix.hpp:36 / .cpp:61-86): y = A x, x cols x l, y rows x l. */
DSVD_API int dsvd_spmm(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* offsets,
              const int64_t* col_indices, const double* values, const double* x, int64_t l,
              double* y);
/* spmm + add_scaled fused (solver.cpp:93-94, dense_kernels.cpp:128-136):
 * t = A y, then t += (-alpha) q unless alpha == 0. */
DSVD_API int dsvd_spmm_shift(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                    const int64_t* offsets, const int64_t* col_indices, const double* values,
                    const double* y, int64_t l, double alpha, const double* q, double* t);
/* transpose (sparse_matrix.hpp:30 / .cpp:35-55) */
DSVD_API int dsvd_transpose(dsvd_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                   const int64_t* offsets, const int64_t* col_indices, const double* values,
                   int64_t* t_offsets, int64_t* t_col_indices, double* t_values);
/* gram (dense_kernels.hpp:24 / .cpp:91-108): g = c^T c, exactly symmetric. */
DSVD_API int dsvd_gram(dsvd_ctx* ctx, int64_t rows, int64_t cols, const double* c, double* g);
/* sym_eig (sym_eig.hpp:20): ascending values, column-major vectors. */
DSVD_API int dsvd_sym_eig(dsvd_ctx* ctx, int64_t n, const double* g, double* values, double* vectors);
/* eig_svd (decompositions.hpp:28 / .cpp:45-75). */
DSVD_API int dsvd_eig_svd(dsvd_ctx* ctx, int64_t rows, int64_t cols, const double* c, double* u,
                 double* s, double* v);
/* matmul (dense_kernels.hpp:21 / .cpp:34-53): c = a b (m x kk times kk x n). */
DSVD_API int dsvd_matmul(dsvd_ctx* ctx, int64_t m, int64_t kk, int64_t n, const double* a,
                const double* b, double* c);
/* gaussian_matrix (random.hpp:20 / .cpp:29-36). */
DSVD_API int dsvd_gaussian_matrix(dsvd_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out);
/* Rows [row_offset, row_offset + rows) of gaussian_matrix(global_rows, cols, seed)
 * (a row shard's sketch Omega_g, random.cpp:29-36 with e = j*global_rows + i). */
DSVD_API int dsvd_gaussian_rows(dsvd_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, int64_t global_rows,
                                int64_t row_offset, double* out);
DSVD_API uint64_t dsvd_splitmix64_at(uint64_t seed, uint64_t i);

/* ---- synthetic inputs (host, deterministic, thread-count invariant) ------
 * Bench/test input preparation, not part of the solve path.
 * sparse_random (synthetic.hpp:37-38 / .cpp:72-120; config 1).
 * powerlaw: config 2 of BASELINE.json — row degrees round(lognormal(mu,
 * sigma)) clamped to [1, cols], columns Zipf(zipf_s) ranks mapped through a
 * seeded permutation, sampled without replacement per row, values N(0,1).
 * ratings: config 3 — like powerlaw with integer values 1..5.
 * Two-phase: the call returns nnz and keeps the arrays; *_fetch copies them out. */
DSVD_API int dsvd_synth_sparse_random(int64_t rows, int64_t cols, int64_t nnz_per_row, uint64_t seed,
                             int row_decay, int64_t* nnz);
DSVD_API int dsvd_synth_powerlaw(int64_t rows, int64_t cols, double mu, double sigma, double zipf_s,
                        int ratings, uint64_t seed, int64_t* nnz);
DSVD_API int dsvd_synth_fetch(int64_t* offsets, int64_t* col_indices, double* values);

#ifdef __cplusplus
}
#endif
#endif /* DASHSVD_B200_H */
