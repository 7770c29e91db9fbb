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

#include <algorithm>
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
struct ParseError : Error {
    ParseError(std::int64_t line_, const std::string& what_)
        : Error("parse error at line " + std::to_string(line_) + ": " + what_), line(line_) {}
    std::int64_t line = 0;
};
struct UnsupportedFormat : Error {
    using Error::Error;
};
struct DegenerateReference : Error {
    using Error::Error;
};
struct HypothesisError : Error {
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
        case DSVD_PARSE: throw ParseError(dsvd_last_error_index(), msg);
        case DSVD_FORMAT: throw UnsupportedFormat(msg);
        case DSVD_DEGENERATE: throw DegenerateReference(msg);
        case DSVD_OTHER: throw Error(msg);
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
    // dense_matrix.cpp:16-27
    static DenseMatrix from_data(index_t rows, index_t cols, std::vector<double> entries) {
        if (rows < 0 || cols < 0) throw ShapeError("negative matrix dimension");
        if (static_cast<index_t>(entries.size()) != rows * cols)
            throw ShapeError("entry count " + std::to_string(entries.size()) + " does not match " +
                             std::to_string(rows) + "x" + std::to_string(cols));
        for (double v : entries)
            if (!(v - v == 0.0)) throw NumericalError("non-finite entry in dense input");
        DenseMatrix m;
        m.rows_ = rows;
        m.cols_ = cols;
        m.data_ = std::move(entries);
        return m;
    }

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


// ---- matrix_market.hpp:14-34 (text parsing on the host, assembly / validation on the GPU)
inline SparseMatrix load_matrix_market(const std::string& path) {
    dsvd_ctx* ctx = b200::context();
    int64_t dims[3];
    b200::check(dsvd_mtx_assemble(ctx, path.c_str(), dims));
    SparseMatrix a;
    a.rows = dims[0];
    a.cols = dims[1];
    a.offsets.resize(a.rows + 1);
    a.col_indices.resize(dims[2]);
    a.values.resize(dims[2]);
    b200::check(dsvd_coo_fetch(ctx, a.offsets.data(), a.col_indices.data(), a.values.data()));
    return a;
}
inline void write_matrix_market(const std::string& path, const SparseMatrix& a) {
    b200::check(dsvd_write_matrix_market(path.c_str(), a.rows, a.cols, a.offsets.data(), a.col_indices.data(),
                                         a.values.data()));
}
inline void save_cache(const std::string& path, const SparseMatrix& a) {
    b200::check(dsvd_save_cache(path.c_str(), a.rows, a.cols, a.nnz(), a.offsets.data(), a.col_indices.data(),
                                a.values.data()));
}
inline DenseMatrix load_dense_array(const std::string& path) {
    int64_t dims[2];
    b200::check(dsvd_dense_read(path.c_str(), dims));
    DenseMatrix d(dims[0], dims[1]);
    b200::check(dsvd_dense_fetch(d.data()));
    return d;
}
inline void write_dense_array(const std::string& path, const DenseMatrix& a) {
    b200::check(dsvd_dense_write(path.c_str(), a.rows(), a.cols(), a.data()));
}

namespace b200 {
// A CSR(A) + CSR(A^T) pair resident on the GPU: load once, solve / measure many times.
class DeviceMatrix {
  public:
    DeviceMatrix() = default;
    explicit DeviceMatrix(const SparseMatrix& a) {
        dsvd_matrix* m = nullptr;
        check(dsvd_matrix_upload(context(), a.rows, a.cols, a.nnz(), a.offsets.data(), a.col_indices.data(),
                                 a.values.data(), &m));
        reset(m, a.rows, a.cols, a.nnz());
    }
    // ".dsh" -> load_cache (validated on the device), otherwise Matrix Market
    // assembled on the device (the CLI's load_input, dashsvd.cpp:78-82)
    static DeviceMatrix load(const std::string& path) {
        DeviceMatrix d;
        dsvd_matrix* m = nullptr;
        int64_t dims[3];
        if (path.size() > 4 && path.compare(path.size() - 4, 4, ".dsh") == 0) {
            check(dsvd_matrix_load_cache(context(), path.c_str(), 1, &m, dims));
        } else {
            check(dsvd_mtx_assemble(context(), path.c_str(), dims));
            check(dsvd_matrix_from_coo(context(), &m));
        }
        d.reset(m, dims[0], dims[1], dims[2]);
        return d;
    }
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    index_t nnz() const { return nnz_; }
    const dsvd_matrix* handle() const { return m_.get(); }
    SparseMatrix download() const {
        SparseMatrix a;
        a.rows = rows_;
        a.cols = cols_;
        a.offsets.resize(rows_ + 1);
        a.col_indices.resize(nnz_);
        a.values.resize(nnz_);
        check(dsvd_matrix_download(m_.get(), a.offsets.data(), a.col_indices.data(), a.values.data()));
        return a;
    }
    // solve(a, at, cfg) (solver.cpp:214-223) on the resident pair; `stats`
    // (optional) receives the device timing breakdown of the call
    SolveResult solve(const SolverConfig& cfg, dsvd_stats* stats = nullptr) const {
        if (cfg.orth == Orthonormalizer::qr && cfg.alg != Algorithm::basic)
            throw ConfigError(
                "the qr orthonormalizer applies to the basic algorithm only; shifted iterations need "
                "the surrogate spectrum");
        dsvd_ctx* ctx = context();
        const dsvd_config c = to_c(cfg, false);
        check(dsvd_validate_config(&c, rows_, cols_));
        const index_t l = cfg.sketch_width();
        const index_t cap = std::max<index_t>(1, cfg.alg == Algorithm::dash ? cfg.p_max : cfg.p);
        SolveResult r;
        r.svd.u = DenseMatrix(rows_, cfg.k);
        r.svd.s.assign(cfg.k, 0.0);
        r.svd.v = DenseMatrix(cols_, cfg.k);
        std::vector<double> alphas(cap), s_hat(static_cast<std::size_t>(cap * l));
        dsvd_outputs out{};
        out.u = r.svd.u.data();
        out.s = r.svd.s.data();
        out.v = r.svd.v.data();
        out.alphas = alphas.data();
        out.s_hat = s_hat.data();
        out.trace_cap = cap;
        if (stats) check(dsvd_ctx_set_profiling(ctx, 1));
        check(dsvd_solve(ctx, m_.get(), &c, &out, nullptr, nullptr));
        if (stats) check(dsvd_ctx_get_stats(ctx, stats));
        r.trace.iterations = out.iterations;
        r.trace.stop_reason = static_cast<StopReason>(out.stop_reason);
        const bool no_spectrum = cfg.alg == Algorithm::basic && cfg.orth == Orthonormalizer::qr;
        for (index_t j = 0; j < out.iterations && j < cap; ++j) {
            r.trace.alphas.push_back(alphas[j]);
            if (no_spectrum) r.trace.s_hat_history.emplace_back();
            else r.trace.s_hat_history.emplace_back(s_hat.begin() + j * l, s_hat.begin() + (j + 1) * l);
        }
        return r;
    }

  private:
    void reset(dsvd_matrix* m, index_t r, index_t c, index_t n) {
        m_.reset(m, [](dsvd_matrix* p) {
            if (p) dsvd_matrix_destroy(p);
        });
        rows_ = r;
        cols_ = c;
        nnz_ = n;
    }
    std::shared_ptr<dsvd_matrix> m_;
    index_t rows_ = 0, cols_ = 0, nnz_ = 0;
};
}  // namespace b200

inline SparseMatrix load_cache(const std::string& path) {
    if (!(path.size() > 4 && path.compare(path.size() - 4, 4, ".dsh") == 0)) {
        // load_cache does not look at the extension
        dsvd_matrix* m = nullptr;
        int64_t dims[3];
        b200::check(dsvd_matrix_load_cache(b200::context(), path.c_str(), 1, &m, dims));
        std::unique_ptr<dsvd_matrix, int (*)(dsvd_matrix*)> hold(m, dsvd_matrix_destroy);
        SparseMatrix a;
        a.rows = dims[0];
        a.cols = dims[1];
        a.offsets.resize(a.rows + 1);
        a.col_indices.resize(dims[2]);
        a.values.resize(dims[2]);
        b200::check(dsvd_matrix_download(m, a.offsets.data(), a.col_indices.data(), a.values.data()));
        return a;
    }
    return b200::DeviceMatrix::load(path).download();
}

// ---- metrics.hpp:13-69 ---------------------------------------------------------------
enum class ReferenceSource { oracle, file };
struct ReferenceSpectrum {
    std::vector<double> sigmas;
    ReferenceSource source = ReferenceSource::oracle;
};
inline ReferenceSpectrum load_reference_spectrum(const std::string& path) {
    int64_t n = 0;
    b200::check(dsvd_spectrum_read(path.c_str(), &n));
    ReferenceSpectrum r;
    r.sigmas.resize(n);
    r.source = ReferenceSource::file;
    b200::check(dsvd_spectrum_fetch(r.sigmas.data()));
    return r;
}
inline void write_reference_spectrum(const std::string& path, const std::vector<double>& sigmas) {
    b200::check(dsvd_spectrum_write(path.c_str(), sigmas.data(), static_cast<int64_t>(sigmas.size())));
}
inline double eps_pve(const b200::DeviceMatrix& a, const DenseMatrix& u_hat, const ReferenceSpectrum& ref) {
    double out = 0.0;
    b200::check(dsvd_eps_pve(b200::context(), a.handle(), u_hat.data(), u_hat.cols(), ref.sigmas.data(),
                             static_cast<int64_t>(ref.sigmas.size()), &out));
    return out;
}
inline double eps_res(const b200::DeviceMatrix& a, const TruncatedSvd& f, const ReferenceSpectrum& ref) {
    double out = 0.0;
    b200::check(dsvd_eps_res(b200::context(), a.handle(), f.u.data(), f.s.data(), f.v.data(), f.rank(),
                             ref.sigmas.data(), static_cast<int64_t>(ref.sigmas.size()), &out));
    return out;
}
inline double eps_spec(const b200::DeviceMatrix& a, const TruncatedSvd& f, const ReferenceSpectrum& ref,
                       index_t power_iters = 300, std::uint64_t seed = 0x5eed) {
    double out = 0.0;
    b200::check(dsvd_eps_spec(b200::context(), a.handle(), f.u.data(), f.s.data(), f.v.data(), f.rank(),
                              ref.sigmas.data(), static_cast<int64_t>(ref.sigmas.size()), power_iters, seed,
                              &out));
    return out;
}
inline double max_triplet_residual(const b200::DeviceMatrix& a, const TruncatedSvd& f) {
    double out = 0.0;
    b200::check(dsvd_max_triplet_residual(b200::context(), a.handle(), f.u.data(), f.s.data(), f.v.data(),
                                          f.rank(), &out));
    return out;
}
inline double eps_pve(const SparseMatrix& a, const DenseMatrix& u_hat, const ReferenceSpectrum& ref) {
    return eps_pve(b200::DeviceMatrix(a), u_hat, ref);
}
inline double eps_res(const SparseMatrix& a, const TruncatedSvd& f, const ReferenceSpectrum& ref) {
    return eps_res(b200::DeviceMatrix(a), f, ref);
}
inline double eps_spec(const SparseMatrix& a, const TruncatedSvd& f, const ReferenceSpectrum& ref,
                       index_t power_iters = 300, std::uint64_t seed = 0x5eed) {
    return eps_spec(b200::DeviceMatrix(a), f, ref, power_iters, seed);
}
inline double max_triplet_residual(const SparseMatrix& a, const TruncatedSvd& f) {
    return max_triplet_residual(b200::DeviceMatrix(a), f);
}
// metrics.cpp:160-170 (k values; host arithmetic)
inline double eps_sigma(const std::vector<double>& s_hat, const ReferenceSpectrum& ref) {
    const index_t k = static_cast<index_t>(s_hat.size());
    if (k < 1) throw ShapeError("eps_sigma: no singular values supplied");
    if (static_cast<index_t>(ref.sigmas.size()) < k)
        throw DegenerateReference("reference provides " + std::to_string(ref.sigmas.size()) +
                                  " singular values, need " + std::to_string(k));
    double worst = 0.0;
    for (index_t i = 0; i < k; ++i) {
        if (ref.sigmas[i] == 0.0) throw DegenerateReference("sigma_i is zero");
        const double e = (ref.sigmas[i] - s_hat[i] < 0 ? s_hat[i] - ref.sigmas[i] : ref.sigmas[i] - s_hat[i]) /
                         ref.sigmas[i];
        worst = e > worst ? e : worst;
    }
    return worst;
}

// synthetic.hpp:37-38 (sparse_random, generated on the host by the library)
inline SparseMatrix sparse_random(index_t rows, index_t cols, index_t nnz_per_row, std::uint64_t seed,
                                  bool row_decay = false) {
    int64_t nnz = 0;
    b200::check(dsvd_synth_sparse_random(rows, cols, nnz_per_row, seed, row_decay ? 1 : 0, &nnz));
    SparseMatrix a;
    a.rows = rows;
    a.cols = cols;
    a.offsets.resize(rows + 1);
    a.col_indices.resize(nnz);
    a.values.resize(nnz);
    b200::check(dsvd_synth_fetch(a.offsets.data(), a.col_indices.data(), a.values.data()));
    return a;
}

}  // namespace dashsvd
