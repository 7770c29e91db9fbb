// dashsvd_b200.hpp — the reference's C++ API (namespace dashsvd, solver.hpp /
// sparse_matrix.hpp / dense_matrix.hpp / decompositions.hpp / errors.hpp of
// /root/reference/proj/core/include/dashsvd) re-expressed over the B200 C ABI.
//
// A caller of the reference library switches by including this header instead
// of <dashsvd/solver.hpp> and linking libdashsvd_b200.so: the types, function
// names, argument meanings and exception types are the reference's. Every
// computation runs on the GPU (sm_100a); there is no CPU fallback.
//
// Header-only; needs C++17.
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dashsvd_b200.h"

namespace dashsvd {

using index_t = std::int64_t;

// ---- errors.hpp:10-59 ---------------------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct RankDeficient : Error {
    RankDeficient(std::int64_t index_, const std::string& what_)
        : Error(what_ + " (index " + std::to_string(index_) + ")"), index(index_) {}
    std::int64_t index = 0;
};
struct NumericalError : Error {
    using Error::Error;
};

namespace b200 {
inline void check(int rc) {
    if (rc == DSVD_OK) return;
    const std::string msg = dsvd_last_error();
    switch (rc) {
        case DSVD_SHAPE: throw ShapeError(msg);
        case DSVD_CONFIG: throw ConfigError(msg);
        case DSVD_RANK_DEFICIENT: {
            const auto cut = msg.find(" (index");
            throw RankDeficient(dsvd_last_error_index(), msg.substr(0, cut));
        }
        case DSVD_NUMERICAL: throw NumericalError(msg);
        default: throw Error("[dashsvd_b200 status " + std::to_string(rc) + "] " + msg);
    }
}

// Process-wide device context (GPU 0 unless dsvd_default_device() is given
// another index first). One context per thread is the safe pattern for
// concurrent solves (see dashsvd_b200.h).
inline dsvd_ctx* context(int device = 0) {
    thread_local std::unique_ptr<dsvd_ctx, int (*)(dsvd_ctx*)> ctx{nullptr, dsvd_ctx_destroy};
    if (!ctx) {
        dsvd_ctx* c = nullptr;
        check(dsvd_ctx_create(device, &c));
        ctx.reset(c);
    }
    return ctx.get();
}
}  // namespace b200

// ---- dense_matrix.hpp:10-42 (column-major) ------------------------------------
class DenseMatrix {
  public:
    DenseMatrix() = default;
    DenseMatrix(index_t rows, index_t cols) : rows_(rows), cols_(cols) {
        if (rows < 0 || cols < 0) throw ShapeError("negative matrix dimension");
        data_.assign(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols), 0.0);
    }
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    index_t size() const { return rows_ * cols_; }
    double& operator()(index_t i, index_t j) { return data_[j * rows_ + i]; }
    double operator()(index_t i, index_t j) const { return data_[j * rows_ + i]; }
    double* col(index_t j) { return data_.data() + j * rows_; }
    const double* col(index_t j) const { return data_.data() + j * rows_; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }

  private:
    index_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// ---- sparse_matrix.hpp:14-36 ----------------------------------------------------
struct SparseMatrix {
    index_t rows = 0;
    index_t cols = 0;
    std::vector<index_t> offsets;
    std::vector<index_t> col_indices;
    std::vector<double> values;
    index_t nnz() const { return static_cast<index_t>(values.size()); }
};

// ---- decompositions.hpp:11-17, solver.hpp:13-74 ------------------------------------
struct TruncatedSvd {
    DenseMatrix u;
    std::vector<double> s;
    DenseMatrix v;
    index_t rank() const { return static_cast<index_t>(s.size()); }
};

enum class Algorithm { basic, shifted, fixed_shift, dash };
enum class Orthonormalizer { eigsvd, qr };
enum class StopReason { fixed_p, tol_met, p_max_reached };

struct SolverConfig {
    index_t k = 0;
    index_t s = -1;
    index_t p = -1;
    double tol = 1e-2;
    index_t p_max = 1000;
    Algorithm alg = Algorithm::dash;
    Orthonormalizer orth = Orthonormalizer::eigsvd;
    std::uint64_t seed = 0;
    bool deterministic = true;
    index_t effective_s(index_t k_) const { return s >= 0 ? s : (k_ / 2 > 0 ? k_ / 2 : 1); }
    index_t sketch_width() const { return k + effective_s(k); }
};

struct ShiftTrace {
    std::vector<double> alphas;
    std::vector<std::vector<double>> s_hat_history;
    index_t iterations = 0;
    StopReason stop_reason = StopReason::fixed_p;
};

struct SolveResult {
    TruncatedSvd svd;
    ShiftTrace trace;
};

struct IterationState {
    index_t iteration;
    double alpha;
    const std::vector<double>& s_hat;
    const DenseMatrix& q_before;
    const DenseMatrix& q_after;
};
using IterationObserver = std::function<void(const IterationState&)>;

namespace b200 {
inline dsvd_config to_c(const SolverConfig& c, bool direct) {
    dsvd_config r{};
    r.k = c.k;
    r.s = c.s;
    r.p = c.p;
    r.tol = c.tol;
    r.p_max = c.p_max;
    r.alg = static_cast<int32_t>(c.alg);
    r.flags = (direct ? DSVD_FLAG_DIRECT : 0) | (c.orth == Orthonormalizer::qr ? DSVD_FLAG_ORTH_QR : 0);
    r.seed = c.seed;
    return r;
}

struct ObserverBox {
    const IterationObserver* obs;
};

inline void observer_tramp(int64_t it, double alpha, const double* s_hat, int64_t l,
                           const double* qb, const double* qa, int64_t n, void* user) {
    auto* box = static_cast<ObserverBox*>(user);
    std::vector<double> sh(s_hat, s_hat + l);
    DenseMatrix before(n, l), after(n, l);
    std::memcpy(before.data(), qb, sizeof(double) * n * l);
    std::memcpy(after.data(), qa, sizeof(double) * n * l);
    (*box->obs)(IterationState{it, alpha, sh, before, after});
}

inline SolveResult run(const SparseMatrix& a, const SolverConfig& cfg,
                       const IterationObserver& observer, bool direct) {
    if (cfg.orth == Orthonormalizer::qr && cfg.alg != Algorithm::basic)
        throw ConfigError(
            "the qr orthonormalizer applies to the basic algorithm only; shifted iterations need "
            "the surrogate spectrum");
    dsvd_ctx* ctx = context();
    const dsvd_config c = to_c(cfg, direct);
    check(dsvd_validate_config(&c, a.rows, a.cols));
    const index_t l = cfg.sketch_width();
    const index_t cap = std::max<index_t>(1, cfg.alg == Algorithm::dash ? cfg.p_max : cfg.p);
    SolveResult r;
    r.svd.u = DenseMatrix(a.rows, cfg.k);
    r.svd.s.assign(cfg.k, 0.0);
    r.svd.v = DenseMatrix(a.cols, cfg.k);
    std::vector<double> alphas(cap), s_hat(static_cast<std::size_t>(cap * l));
    dsvd_outputs out{};
    out.u = r.svd.u.data();
    out.s = r.svd.s.data();
    out.v = r.svd.v.data();
    out.alphas = alphas.data();
    out.s_hat = s_hat.data();
    out.trace_cap = cap;
    if (!observer && !direct) {
        check(dsvd_solve_csr(ctx, a.rows, a.cols, a.nnz(), a.offsets.data(), a.col_indices.data(),
                             a.values.data(), &c, &out));
    } else {
        dsvd_matrix* m = nullptr;
        check(dsvd_matrix_upload(ctx, a.rows, a.cols, a.nnz(), a.offsets.data(),
                                 a.col_indices.data(), a.values.data(), &m));
        std::unique_ptr<dsvd_matrix, int (*)(dsvd_matrix*)> hold(m, dsvd_matrix_destroy);
        ObserverBox box{&observer};
        check(dsvd_solve(ctx, m, &c, &out, observer ? observer_tramp : nullptr, &box));
    }
    r.trace.iterations = out.iterations;
    r.trace.stop_reason = static_cast<StopReason>(out.stop_reason);
    const bool no_spectrum = cfg.alg == Algorithm::basic && cfg.orth == Orthonormalizer::qr;
    for (index_t j = 0; j < out.iterations && j < cap; ++j) {
        r.trace.alphas.push_back(alphas[j]);
        if (no_spectrum) r.trace.s_hat_history.emplace_back();  // qr: no surrogate spectrum
        else r.trace.s_hat_history.emplace_back(s_hat.begin() + j * l, s_hat.begin() + (j + 1) * l);
    }
    return r;
}
}  // namespace b200

// ---- solver.hpp:76-126 ------------------------------------------------------------
inline void validate_config(const SolverConfig& cfg, index_t rows, index_t cols) {
    const dsvd_config c = b200::to_c(cfg, false);
    b200::check(dsvd_validate_config(&c, rows, cols));
    if (cfg.orth == Orthonormalizer::qr && cfg.alg != Algorithm::basic)
        throw ConfigError("the qr orthonormalizer applies to the basic algorithm only; shifted "
                          "iterations need the surrogate spectrum");
}
inline double update_shift(double alpha, double s_ll) { return dsvd_update_shift(alpha, s_ll); }
inline bool pve_stop_check(const std::vector<double>& prev, double alpha_prev,
                           const std::vector<double>& cur, double alpha, index_t k, double tol) {
    int stop = 0;
    b200::check(dsvd_pve_stop_check(prev.data(), static_cast<int64_t>(prev.size()), alpha_prev,
                                    cur.data(), static_cast<int64_t>(cur.size()), alpha, k, tol,
                                    &stop));
    return stop != 0;
}

inline SolveResult solve(const SparseMatrix& a, const SolverConfig& cfg) {
    return b200::run(a, cfg, {}, false);
}
inline SolveResult solve(const SparseMatrix& a, const SparseMatrix& /*at*/,
                         const SolverConfig& cfg, const IterationObserver& observer = {}) {
    // the device builds its own transpose (bitwise equal to transpose(a))
    return b200::run(a, cfg, observer, false);
}
// basic_rsvd (solver.cpp:178-188): Alg. 1 on `a` as given
inline TruncatedSvd basic_rsvd(const SparseMatrix& a, const SolverConfig& cfg) {
    SolverConfig c = cfg;
    c.alg = Algorithm::basic;
    return b200::run(a, c, {}, true).svd;
}
inline TruncatedSvd basic_rsvd(const SparseMatrix& a, const SparseMatrix& /*at*/, const SolverConfig& cfg,
                               const IterationObserver& observer = {}) {
    SolverConfig c = cfg;
    c.alg = Algorithm::basic;
    return b200::run(a, c, observer, true).svd;
}
inline SolveResult shifted_rsvd(const SparseMatrix& a, const SolverConfig& cfg) {
    SolverConfig c = cfg;
    if (c.alg != Algorithm::fixed_shift) c.alg = Algorithm::shifted;
    return b200::run(a, c, {}, true);
}
inline SolveResult shifted_rsvd(const SparseMatrix& a, const SparseMatrix& /*at*/,
                                const SolverConfig& cfg, const IterationObserver& observer = {}) {
    SolverConfig c = cfg;
    if (c.alg != Algorithm::fixed_shift) c.alg = Algorithm::shifted;
    return b200::run(a, c, observer, true);
}
inline SolveResult dash_svd(const SparseMatrix& a, const SolverConfig& cfg) {
    SolverConfig c = cfg;
    c.alg = Algorithm::dash;
    return b200::run(a, c, {}, true);
}
inline SolveResult dash_svd(const SparseMatrix& a, const SparseMatrix& /*at*/,
                            const SolverConfig& cfg, const IterationObserver& observer = {}) {
    SolverConfig c = cfg;
    c.alg = Algorithm::dash;
    return b200::run(a, c, observer, true);
}

inline TruncatedSvd finalize_row_basis(const SparseMatrix& a, const DenseMatrix& q, index_t k) {
    if (q.rows() != a.cols) throw ShapeError("finalize_row_basis: basis does not match matrix");
    if (k < 1 || k > q.cols()) throw ShapeError("finalize_row_basis: k out of range");
    dsvd_ctx* ctx = b200::context();
    dsvd_matrix* m = nullptr;
    b200::check(dsvd_matrix_upload(ctx, a.rows, a.cols, a.nnz(), a.offsets.data(),
                                   a.col_indices.data(), a.values.data(), &m));
    std::unique_ptr<dsvd_matrix, int (*)(dsvd_matrix*)> hold(m, dsvd_matrix_destroy);
    TruncatedSvd f;
    f.u = DenseMatrix(a.rows, k);
    f.s.assign(k, 0.0);
    f.v = DenseMatrix(a.cols, k);
    b200::check(dsvd_finalize_row_basis(ctx, m, q.data(), q.cols(), k, f.u.data(), f.s.data(),
                                        f.v.data()));
    return f;
}

// ---- kernel seams used by the reference's tests -------------------------------------
inline SparseMatrix transpose(const SparseMatrix& a) {
    SparseMatrix t;
    t.rows = a.cols;
    t.cols = a.rows;
    t.offsets.resize(a.cols + 1);
    t.col_indices.resize(a.nnz());
    t.values.resize(a.nnz());
    b200::check(dsvd_transpose(b200::context(), a.rows, a.cols, a.nnz(), a.offsets.data(),
                               a.col_indices.data(), a.values.data(), t.offsets.data(),
                               t.col_indices.data(), t.values.data()));
    return t;
}
inline DenseMatrix spmm(const SparseMatrix& a, const DenseMatrix& x) {
    if (a.cols != x.rows()) throw ShapeError("spmm: inner dimensions differ");
    DenseMatrix y(a.rows, x.cols());
    b200::check(dsvd_spmm(b200::context(), a.rows, a.cols, a.nnz(), a.offsets.data(),
                          a.col_indices.data(), a.values.data(), x.data(), x.cols(), y.data()));
    return y;
}
inline DenseMatrix gram(const DenseMatrix& c) {
    DenseMatrix g(c.cols(), c.cols());
    b200::check(dsvd_gram(b200::context(), c.rows(), c.cols(), c.data(), g.data()));
    return g;
}
inline TruncatedSvd eig_svd(const DenseMatrix& c) {
    TruncatedSvd f;
    f.u = DenseMatrix(c.rows(), c.cols());
    f.s.assign(c.cols(), 0.0);
    f.v = DenseMatrix(c.cols(), c.cols());
    b200::check(dsvd_eig_svd(b200::context(), c.rows(), c.cols(), c.data(), f.u.data(),
                             f.s.data(), f.v.data()));
    return f;
}
inline DenseMatrix gaussian_matrix(index_t rows, index_t cols, std::uint64_t seed) {
    DenseMatrix g(rows, cols);
    b200::check(dsvd_gaussian_matrix(b200::context(), rows, cols, seed, g.data()));
    return g;
}
inline std::uint64_t splitmix64_at(std::uint64_t seed, std::uint64_t i) {
    return dsvd_splitmix64_at(seed, i);
}

}  // namespace dashsvd
