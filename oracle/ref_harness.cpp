// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// C-ABI wrapper around the *unmodified* reference library (dashsvd::core),
// compiled together with the reference sources where they lie under
// /root/reference/proj/core/src (see oracle/Makefile). The wrapper exists so
// that Python tests and bench.py's CPU-baseline leg can call the reference's
// own code path:
//   - dashsvd::solve / shifted_rsvd / dash_svd          solver.hpp:76-116
//   - dashsvd::transpose / spmm                          sparse_matrix.hpp:30-36
//   - dashsvd::gram / add_scaled / matmul                dense_kernels.hpp:24-33
//   - dashsvd::eig_svd / sym_eig                         decompositions.hpp:28, sym_eig.hpp:20
//   - dashsvd::gaussian_matrix / normal_at / splitmix64  random.hpp:11-20
//   - dashsvd::sparse_random                             synthetic.hpp:37-38
//   - dashsvd::finalize_row_basis                        solver.hpp:123
//   - SparseMatrix::validate                             sparse_matrix.hpp:22
//   - load_matrix_market / write_matrix_market / save_cache / load_cache
//                                                        matrix_market.hpp:14-34
// Dense matrices cross this boundary column-major (the reference's layout,
// dense_matrix.hpp:10-13). Output: oracle/_ref/libdashsvd_ref.so.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "dashsvd/decompositions.hpp"
#include "dashsvd/dense_kernels.hpp"
#include "dashsvd/errors.hpp"
#include "dashsvd/matrix_market.hpp"
#include "dashsvd/random.hpp"
#include "dashsvd/metrics.hpp"
#include "dashsvd/solver.hpp"
#include "dashsvd/sparse_matrix.hpp"
#include "dashsvd/sym_eig.hpp"
#include "dashsvd/synthetic.hpp"
#include "dashsvd/threads.hpp"

using namespace dashsvd;

namespace {

thread_local std::string g_err;
thread_local long long g_err_index = -1;

// Status codes shared with include/dashsvd_b200.h (DSVD_*).
enum { OK = 0, E_SHAPE = 1, E_CONFIG = 2, E_RANK = 3, E_NUMERICAL = 4, E_OTHER = 9, E_FORMAT = 11, E_PARSE = 12 };

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const RankDeficient& e) {
        g_err = e.what();
        g_err_index = e.index;
        return E_RANK;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return E_SHAPE;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return E_CONFIG;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return E_NUMERICAL;
    } catch (const ParseError& e) {
        g_err = e.what();
        g_err_index = e.line;
        return E_PARSE;
    } catch (const UnsupportedFormat& e) {
        g_err = e.what();
        return E_FORMAT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_OTHER;
    }
}

SparseMatrix make_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off,
                      const int64_t* idx, const double* val) {
    SparseMatrix a;
    a.rows = rows;
    a.cols = cols;
    a.offsets.assign(off, off + rows + 1);
    a.col_indices.assign(idx, idx + nnz);
    a.values.assign(val, val + nnz);
    return a;
}

DenseMatrix make_dense(int64_t rows, int64_t cols, const double* colmajor) {
    DenseMatrix d(rows, cols);
    std::memcpy(d.data(), colmajor, sizeof(double) * rows * cols);
    return d;
}

void put(const DenseMatrix& d, double* out) {
    if (out) std::memcpy(out, d.data(), sizeof(double) * d.size());
}

int g_orth_qr = 0;  // ref_set_orth: Orthonormalizer for the next make_cfg calls

SolverConfig make_cfg(int64_t k, int64_t s, int64_t p, double tol, int64_t p_max, int alg,
                      uint64_t seed) {
    SolverConfig c;
    c.orth = g_orth_qr ? Orthonormalizer::qr : Orthonormalizer::eigsvd;
    c.k = k;
    c.s = s;
    c.p = p;
    c.tol = tol;
    c.p_max = p_max;
    c.alg = static_cast<Algorithm>(alg);
    c.seed = seed;
    return c;
}

SparseMatrix g_rand;  // last sparse_random result, handed out by ref_sparse_random_fetch
SparseMatrix g_csr;   // last loaded matrix (ref_load_matrix_market / ref_load_cache)
DenseMatrix g_dense;  // last ref_load_dense_array result
std::vector<double> g_spec;  // last ref_load_spectrum result

void put_dims(const SparseMatrix& a, int64_t* dims) {
    dims[0] = a.rows;
    dims[1] = a.cols;
    dims[2] = a.nnz();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
long long ref_last_error_index() { return g_err_index; }
void ref_set_threads(int n) { set_thread_count(n); }
void ref_set_orth(int qr) { g_orth_qr = qr; }
int ref_thread_count() { return thread_count(); }

uint64_t ref_splitmix64_at(uint64_t seed, uint64_t i) { return splitmix64_at(seed, i); }
double ref_normal_at(uint64_t seed, uint64_t i) { return normal_at(seed, i); }

void ref_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    put(gaussian_matrix(rows, cols, seed), out);
}

int ref_sparse_random(int64_t rows, int64_t cols, int64_t npr, uint64_t seed, int decay,
                      int64_t* nnz_out) {
    return guarded([&] {
        g_rand = sparse_random(rows, cols, npr, seed, decay != 0);
        *nnz_out = g_rand.nnz();
    });
}

void ref_sparse_random_fetch(int64_t* off, int64_t* idx, double* val) {
    std::memcpy(off, g_rand.offsets.data(), sizeof(int64_t) * g_rand.offsets.size());
    std::memcpy(idx, g_rand.col_indices.data(), sizeof(int64_t) * g_rand.col_indices.size());
    std::memcpy(val, g_rand.values.data(), sizeof(double) * g_rand.values.size());
    g_rand = SparseMatrix();
}

int ref_transpose(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off, const int64_t* idx,
                  const double* val, int64_t* t_off, int64_t* t_idx, double* t_val) {
    return guarded([&] {
        SparseMatrix t = transpose(make_csr(rows, cols, nnz, off, idx, val));
        std::memcpy(t_off, t.offsets.data(), sizeof(int64_t) * (cols + 1));
        std::memcpy(t_idx, t.col_indices.data(), sizeof(int64_t) * nnz);
        std::memcpy(t_val, t.values.data(), sizeof(double) * nnz);
    });
}

int ref_spmm(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off, const int64_t* idx,
             const double* val, const double* x, int64_t l, double* y) {
    return guarded([&] {
        put(spmm(make_csr(rows, cols, nnz, off, idx, val), make_dense(cols, l, x)), y);
    });
}

int ref_add_scaled(int64_t rows, int64_t cols, double* y, double alpha, const double* x) {
    return guarded([&] {
        DenseMatrix yy = make_dense(rows, cols, y);
        add_scaled(yy, alpha, make_dense(rows, cols, x));
        put(yy, y);
    });
}

int ref_gram(int64_t rows, int64_t cols, const double* c, double* g) {
    return guarded([&] { put(gram(make_dense(rows, cols, c)), g); });
}

int ref_matmul(int64_t m, int64_t kk, int64_t n, const double* a, const double* b, double* c) {
    return guarded([&] { put(matmul(make_dense(m, kk, a), make_dense(kk, n, b)), c); });
}

int ref_sym_eig(int64_t n, const double* g, double* values, double* vectors) {
    return guarded([&] {
        EigenPair e = sym_eig(make_dense(n, n, g));
        std::memcpy(values, e.values.data(), sizeof(double) * n);
        put(e.vectors, vectors);
    });
}

int ref_eig_svd(int64_t rows, int64_t cols, const double* c, double* u, double* s, double* v) {
    return guarded([&] {
        TruncatedSvd f = eig_svd(make_dense(rows, cols, c));
        put(f.u, u);
        std::memcpy(s, f.s.data(), sizeof(double) * cols);
        put(f.v, v);
    });
}

int ref_finalize_row_basis(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off,
                           const int64_t* idx, const double* val, const double* q, int64_t l,
                           int64_t k, double* u, double* s, double* v) {
    return guarded([&] {
        TruncatedSvd f =
            finalize_row_basis(make_csr(rows, cols, nnz, off, idx, val), make_dense(cols, l, q), k);
        put(f.u, u);
        std::memcpy(s, f.s.data(), sizeof(double) * k);
        put(f.v, v);
    });
}

int ref_validate_config(int64_t rows, int64_t cols, int64_t k, int64_t s, int64_t p, double tol,
                        int64_t p_max, int alg) {
    return guarded([&] { validate_config(make_cfg(k, s, p, tol, p_max, alg, 0), rows, cols); });
}

double ref_update_shift(double alpha, double s_ll) { return update_shift(alpha, s_ll); }

int ref_pve_stop_check(const double* prev, int64_t n_prev, double alpha_prev, const double* cur,
                       int64_t n_cur, double alpha, int64_t k, double tol, int* stop) {
    return guarded([&] {
        *stop = pve_stop_check(std::span<const double>(prev, n_prev), alpha_prev,
                               std::span<const double>(cur, n_cur), alpha, k, tol)
                    ? 1
                    : 0;
    });
}

// Full solve through dashsvd::solve(a, at, cfg, observer) — the CLI's call
// (tools/dashsvd.cpp:169-170). Outputs are caller-allocated: u[m*k], s[k],
// v[n*k] column-major; alphas[cap], s_hat[cap*l]. times[0] = transpose
// seconds, times[1] = solve seconds, times[2..] = per-iteration observer
// timestamps relative to solve start (up to cap).
int ref_solve(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off, const int64_t* idx,
              const double* val, int64_t k, int64_t s, int64_t p, double tol, int64_t p_max,
              int alg, uint64_t seed, double* u, double* sv, double* v, double* alphas,
              double* s_hat, int64_t cap, int64_t* iterations, int* stop_reason, double* times) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        SparseMatrix a = make_csr(rows, cols, nnz, off, idx, val);
        const SolverConfig cfg = make_cfg(k, s, p, tol, p_max, alg, seed);
        const auto t0 = clk::now();
        SparseMatrix at = transpose(a);
        const auto t1 = clk::now();
        std::vector<double> stamps;
        IterationObserver obs = [&](const IterationState&) {
            stamps.push_back(std::chrono::duration<double>(clk::now() - t1).count());
        };
        SolveResult r = solve(a, at, cfg, times ? obs : IterationObserver{});
        const auto t2 = clk::now();
        put(r.svd.u, u);
        std::memcpy(sv, r.svd.s.data(), sizeof(double) * r.svd.s.size());
        put(r.svd.v, v);
        const int64_t l = cfg.sketch_width();
        for (int64_t c = 0; c < static_cast<int64_t>(r.trace.alphas.size()) && c < cap; ++c) {
            alphas[c] = r.trace.alphas[c];
            const auto& sh = r.trace.s_hat_history[c];  // empty for the qr orthonormalizer
            if (!sh.empty()) std::memcpy(s_hat + c * l, sh.data(), sizeof(double) * std::min<int64_t>(l, sh.size()));
        }
        *iterations = r.trace.iterations;
        *stop_reason = static_cast<int>(r.trace.stop_reason);
        if (times) {
            times[0] = std::chrono::duration<double>(t1 - t0).count();
            times[1] = std::chrono::duration<double>(t2 - t1).count();
            for (int64_t c = 0; c < static_cast<int64_t>(stamps.size()) && c < cap; ++c)
                times[2 + c] = stamps[c];
        }
    });
}

// metrics.cpp:99-206 on host factors (column-major): out = {eps_pve, eps_res,
// eps_spec, max_triplet_residual}
int ref_metrics(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off, const int64_t* idx, const double* val,
                const double* u, const double* s, const double* v, int64_t k, const double* sigmas, int64_t n_ref,
                int64_t power_iters, uint64_t seed, double* out) {
    return guarded([&] {
        SparseMatrix a = make_csr(rows, cols, nnz, off, idx, val);
        TruncatedSvd t;
        t.u = DenseMatrix(rows, k);
        t.v = DenseMatrix(cols, k);
        std::memcpy(t.u.data(), u, sizeof(double) * rows * k);
        std::memcpy(t.v.data(), v, sizeof(double) * cols * k);
        t.s.assign(s, s + k);
        ReferenceSpectrum ref;
        ref.sigmas.assign(sigmas, sigmas + n_ref);
        out[0] = eps_pve(a, t.u, ref);
        out[1] = eps_res(a, t, ref);
        out[2] = eps_spec(a, t, ref, power_iters, seed);
        out[3] = max_triplet_residual(a, t);
    });
}

// SparseMatrix::validate (sparse_matrix.cpp:12-33)
int ref_validate(int64_t rows, int64_t cols, int64_t nnz, const int64_t* off, const int64_t* idx, const double* val) {
    return guarded([&] { make_csr(rows, cols, nnz, off, idx, val).validate(); });
}

// matrix_market.cpp:117-275; the loaded matrix is handed out by ref_csr_fetch
int ref_load_matrix_market(const char* path, int64_t* dims) {
    return guarded([&] {
        g_csr = load_matrix_market(path);
        put_dims(g_csr, dims);
    });
}

int ref_load_cache(const char* path, int64_t* dims) {
    return guarded([&] {
        g_csr = load_cache(path);
        put_dims(g_csr, dims);
    });
}

void ref_csr_fetch(int64_t* off, int64_t* idx, double* val) {
    std::copy(g_csr.offsets.begin(), g_csr.offsets.end(), off);
    std::copy(g_csr.col_indices.begin(), g_csr.col_indices.end(), idx);
    std::copy(g_csr.values.begin(), g_csr.values.end(), val);
}

int ref_save_cache(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* off, const int64_t* idx,
                   const double* val) {
    return guarded([&] { save_cache(path, make_csr(rows, cols, nnz, off, idx, val)); });
}

int ref_write_matrix_market(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* off,
                            const int64_t* idx, const double* val) {
    return guarded([&] { write_matrix_market(path, make_csr(rows, cols, nnz, off, idx, val)); });
}

// load_dense_array / write_dense_array (matrix_market.cpp:179-223)
int ref_load_dense_array(const char* path, int64_t* dims) {
    return guarded([&] {
        g_dense = load_dense_array(path);
        dims[0] = g_dense.rows();
        dims[1] = g_dense.cols();
    });
}
void ref_dense_fetch(double* out) { put(g_dense, out); }
int ref_write_dense_array(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
    return guarded([&] { write_dense_array(path, make_dense(rows, cols, colmajor)); });
}

// load_reference_spectrum / write_reference_spectrum (metrics.cpp:71-97)
int ref_load_spectrum(const char* path, int64_t* n) {
    return guarded([&] {
        g_spec = load_reference_spectrum(path).sigmas;
        *n = static_cast<int64_t>(g_spec.size());
    });
}
void ref_spectrum_fetch(double* out) { std::copy(g_spec.begin(), g_spec.end(), out); }
int ref_write_spectrum(const char* path, const double* s, int64_t n) {
    return guarded([&] { write_reference_spectrum(path, std::vector<double>(s, s + n)); });
}

}  // extern "C"
