/* TEST INFRASTRUCTURE ONLY (see dashsvd_oracle.h): a plain-C restatement of
 * the reference dashSVD hot path, written to reproduce the reference's
 * floating-point operation order exactly so it is bitwise comparable with
 * oracle/_ref. Every arithmetic statement that GCC contracts to an FMA in the
 * reference (-ffp-contract=fast) is written with the same shape here and
 * compiled with the same flags (oracle/Makefile).
 *
 * Citations are to /root/reference/proj/core/src/<file>:<line>.
 */
#include "dashsvd_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_msg[256];
static _Thread_local long long g_index = -1;

static int fail(int code, long long index, const char* msg) {
    snprintf(g_msg, sizeof g_msg, "%s", msg);
    g_index = index;
    return code;
}

const char* orc_last_error(void) { return g_msg; }
long long orc_last_error_index(void) { return g_index; }
void orc_free(void* p) { free(p); }

/* ---- RNG: random.cpp:8-36 ------------------------------------------------ */

uint64_t orc_splitmix64_at(uint64_t seed, uint64_t i) { /* random.cpp:8-13 */
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double unit_open(uint64_t x) { /* random.cpp:18-20: top 53 bits, centred */
    return ((double)(x >> 11) + 0.5) * 0x1p-53;
}

double orc_normal_at(uint64_t seed, uint64_t i) { /* random.cpp:23-27, Box-Muller */
    const double u1 = unit_open(orc_splitmix64_at(seed, 2 * i));
    const double u2 = unit_open(orc_splitmix64_at(seed, 2 * i + 1));
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

void orc_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    /* random.cpp:29-36: entry at column-major linear index e is draw e */
    const int64_t n = rows * cols;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) out[e] = orc_normal_at(seed, (uint64_t)e);
}

/* ---- synthetic.cpp:72-120 (config-1 generator) --------------------------- */

typedef struct {
    int64_t col;
    double val;
} entry;

static int entry_cmp(const void* pa, const void* pb) { /* std::pair lexicographic order */
    const entry* a = (const entry*)pa;
    const entry* b = (const entry*)pb;
    if (a->col != b->col) return a->col < b->col ? -1 : 1;
    if (a->val < b->val) return -1;
    if (a->val > b->val) return 1;
    return 0;
}

int orc_sparse_random(int64_t rows, int64_t cols, int64_t npr, uint64_t seed, int decay,
                      int64_t* nnz_out, int64_t** off_out, int64_t** idx_out, double** val_out) {
    if (rows < 1 || cols < 1 || npr < 1) return fail(ORC_SHAPE, -1, "sparse_random: empty shape");
    if (npr > cols) return fail(ORC_SHAPE, -1, "sparse_random: nnz_per_row exceeds cols");
    const uint64_t col_seed = orc_splitmix64_at(seed, 0);
    const uint64_t val_seed = orc_splitmix64_at(seed, 1);
    entry* buf = (entry*)malloc(sizeof(entry) * rows * npr);
    int64_t* len = (int64_t*)malloc(sizeof(int64_t) * rows);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        entry* row = buf + i * npr;
        const double scale = decay ? 1.0 / sqrt(1.0 + (double)i) : 1.0;
        for (int64_t t = 0; t < npr; ++t) {
            const uint64_t e = (uint64_t)i * (uint64_t)npr + (uint64_t)t;
            row[t].col = (int64_t)(orc_splitmix64_at(col_seed, e) % (uint64_t)cols);
            row[t].val = scale * orc_normal_at(val_seed, e);
        }
        qsort(row, (size_t)npr, sizeof(entry), entry_cmp);
        /* duplicate draws collapse by summation in sorted order; zero sums drop */
        int64_t w = 0;
        for (int64_t r = 0; r < npr;) {
            entry cur = row[r++];
            while (r < npr && row[r].col == cur.col) cur.val += row[r++].val;
            if (cur.val != 0.0) row[w++] = cur;
        }
        len[i] = w;
    }
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (rows + 1));
    off[0] = 0;
    for (int64_t i = 0; i < rows; ++i) off[i + 1] = off[i] + len[i];
    const int64_t nnz = off[rows];
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (nnz ? nnz : 1));
    double* val = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t t = 0; t < len[i]; ++t) {
            idx[off[i] + t] = buf[i * npr + t].col;
            val[off[i] + t] = buf[i * npr + t].val;
        }
    free(buf);
    free(len);
    *nnz_out = nnz;
    *off_out = off;
    *idx_out = idx;
    *val_out = val;
    return ORC_OK;
}

/* ---- sparse kernels: sparse_matrix.cpp:35-86 ------------------------------ */

int orc_transpose(const orc_csr* a, int64_t* t_off, int64_t* t_idx, double* t_val) {
    /* sparse_matrix.cpp:35-55: counting sort; scanning rows in order keeps each
     * transposed row sorted (stable). */
    memset(t_off, 0, sizeof(int64_t) * (a->cols + 1));
    for (int64_t p = 0; p < a->nnz; ++p) ++t_off[a->col_indices[p] + 1];
    for (int64_t j = 0; j < a->cols; ++j) t_off[j + 1] += t_off[j];
    int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (a->cols ? a->cols : 1));
    memcpy(cursor, t_off, sizeof(int64_t) * a->cols);
    for (int64_t i = 0; i < a->rows; ++i)
        for (int64_t p = a->offsets[i]; p < a->offsets[i + 1]; ++p) {
            const int64_t pos = cursor[a->col_indices[p]]++;
            t_idx[pos] = i;
            t_val[pos] = a->values[p];
        }
    free(cursor);
    return ORC_OK;
}

int orc_spmm(const orc_csr* a, const double* x, int64_t l, double* y) {
    /* sparse_matrix.cpp:61-86: y(i,t) is one FMA chain over row i's nonzeros in
     * CSR order, starting from 0.0 (the 48-column blocking there does not change
     * any chain, so it is not restated). x is a->cols x l, y a->rows x l. */
    const int64_t m = a->rows, n = a->cols;
    if (l == 0) return ORC_OK;
    double* xr = (double*)malloc(sizeof(double) * (n ? n : 1) * l); /* row-major repack */
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t t = 0; t < l; ++t) xr[j * l + t] = x[t * n + j];
#pragma omp parallel
    {
        double* acc = (double*)malloc(sizeof(double) * l);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            for (int64_t t = 0; t < l; ++t) acc[t] = 0.0;
            for (int64_t q = a->offsets[i]; q < a->offsets[i + 1]; ++q) {
                const double av = a->values[q];
                const double* row = xr + a->col_indices[q] * l;
                for (int64_t t = 0; t < l; ++t) acc[t] = fma(av, row[t], acc[t]);
            }
            for (int64_t t = 0; t < l; ++t) y[t * m + i] = acc[t];
        }
        free(acc);
    }
    free(xr);
    return ORC_OK;
}

/* ---- dense kernels: dense_kernels.cpp ------------------------------------- */

void orc_add_scaled(int64_t count, double* y, double alpha, const double* x) {
    /* dense_kernels.cpp:128-136: y += alpha*x, contracted to fma */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) y[i] = fma(alpha, x[i], y[i]);
}

void orc_gram(int64_t rows, int64_t cols, const double* c, double* g) {
    /* dense_kernels.cpp:91-108 + dot_tile :18-30: every upper entry is a single
     * FMA chain over all rows; the lower triangle mirrors it exactly. */
#pragma omp parallel for schedule(dynamic)
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i <= j; ++i) {
            const double* ci = c + i * rows;
            const double* cj = c + j * rows;
            double acc = 0.0;
            for (int64_t r = 0; r < rows; ++r) acc = fma(ci[r], cj[r], acc);
            g[j * cols + i] = acc;
            g[i * cols + j] = acc;
        }
}

void orc_matmul(int64_t m, int64_t kk, int64_t n, const double* a, const double* b, double* c) {
    /* dense_kernels.cpp:34-53: c(i,j) = FMA chain over t ascending from 0.0 */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t t = 0; t < kk; ++t) acc = fma(b[j * kk + t], a[t * m + i], acc);
            c[j * m + i] = acc;
        }
}

/* ---- symmetric eigensolver: sym_eig.cpp ----------------------------------- */

/* Householder reduction to tridiagonal form with the transform accumulated
 * (sym_eig.cpp:19-74). w is row-major n x n. The arithmetic statements keep
 * the reference's expression shapes so GCC contracts them identically. */
static void householder_tridiag(double* w, int64_t n, double* d, double* e) {
#define W(i, j) w[(i) * n + (j)]
    for (int64_t i = n - 1; i >= 1; --i) {
        const int64_t l = i - 1;
        double h = 0.0, scale = 0.0;
        if (l > 0) {
            for (int64_t k = 0; k <= l; ++k) scale += fabs(W(i, k));
            if (scale == 0.0) {
                e[i] = W(i, l);
            } else {
                for (int64_t k = 0; k <= l; ++k) {
                    W(i, k) /= scale;
                    h += W(i, k) * W(i, k);
                }
                double f = W(i, l);
                double g = f >= 0.0 ? -sqrt(h) : sqrt(h);
                e[i] = scale * g;
                h -= f * g;
                W(i, l) = f - g;
                f = 0.0;
                for (int64_t j = 0; j <= l; ++j) {
                    W(j, i) = W(i, j) / h;
                    g = 0.0;
                    for (int64_t k = 0; k <= j; ++k) g += W(j, k) * W(i, k);
                    for (int64_t k = j + 1; k <= l; ++k) g += W(k, j) * W(i, k);
                    e[j] = g / h;
                    f += e[j] * W(i, j);
                }
                const double hh = f / (h + h);
                for (int64_t j = 0; j <= l; ++j) {
                    f = W(i, j);
                    e[j] = g = e[j] - hh * f;
                    for (int64_t k = 0; k <= j; ++k) W(j, k) -= f * e[k] + g * W(i, k);
                }
            }
        } else {
            e[i] = W(i, l);
        }
        d[i] = h;
    }
    d[0] = 0.0;
    e[0] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (d[i] != 0.0) {
            for (int64_t j = 0; j < i; ++j) {
                double g = 0.0;
                for (int64_t k = 0; k < i; ++k) g += W(i, k) * W(k, j);
                for (int64_t k = 0; k < i; ++k) W(k, j) -= g * W(k, i);
            }
        }
        d[i] = W(i, i);
        W(i, i) = 1.0;
        for (int64_t j = 0; j < i; ++j) W(j, i) = W(i, j) = 0.0;
    }
#undef W
}

/* Implicit QL with Wilkinson shifts on (d, e); rotations accumulate into the
 * columns of w (sym_eig.cpp:78-130). Returns nonzero past 50 iterations. */
static int ql_implicit(double* w, int64_t n, double* d, double* e) {
#define Z(i, j) w[(i) * n + (j)]
    const double eps = DBL_EPSILON;
    for (int64_t i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    for (int64_t l = 0; l < n; ++l) {
        int iter = 0;
        int64_t m;
        do {
            for (m = l; m + 1 < n; ++m) {
                const double dd = fabs(d[m]) + fabs(d[m + 1]);
                if (fabs(e[m]) <= eps * dd) break;
            }
            if (m != l) {
                if (iter++ == 50) return 1;
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + copysign(r, g));
                double s = 1.0, c = 1.0, p = 0.0;
                int64_t i;
                for (i = m - 1; i >= l; --i) {
                    double f = s * e[i];
                    const double b = c * e[i];
                    e[i + 1] = r = hypot(f, g);
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    for (int64_t k = 0; k < n; ++k) {
                        f = Z(k, i + 1);
                        Z(k, i + 1) = s * Z(k, i) + c * f;
                        Z(k, i) = c * Z(k, i) - s * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
    return 0;
#undef Z
}

int orc_sym_eig(int64_t n, const double* g, double* values, double* vectors) {
    /* sym_eig.cpp:134-175 */
    if (n == 0) return ORC_OK;
    double scale = 0.0, asym = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
            scale = fmax(scale, fabs(g[j * n + i]));
            asym = fmax(asym, fabs(g[j * n + i] - g[i * n + j]));
        }
    if (asym > 1e-10 * fmax(scale, 1e-300))
        return fail(ORC_SHAPE, -1, "sym_eig: matrix is not symmetric");
    double* w = (double*)malloc(sizeof(double) * n * n);
    double* d = (double*)calloc((size_t)n, sizeof(double));
    double* e = (double*)calloc((size_t)n, sizeof(double));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) w[i * n + j] = g[j * n + i];
    int rc = ORC_OK;
    if (n == 1) {
        d[0] = w[0];
        w[0] = 1.0;
    } else {
        householder_tridiag(w, n, d, e);
        if (ql_implicit(w, n, d, e))
            rc = fail(ORC_NUMERICAL, -1, "symmetric QL iteration did not converge");
    }
    if (rc == ORC_OK) {
        /* stable ascending order (sym_eig.cpp:161-164): insertion sort is stable */
        int64_t* order = (int64_t*)malloc(sizeof(int64_t) * n);
        for (int64_t j = 0; j < n; ++j) {
            int64_t pos = j;
            while (pos > 0 && d[order[pos - 1]] > d[j]) {
                order[pos] = order[pos - 1];
                --pos;
            }
            order[pos] = j;
        }
        for (int64_t j = 0; j < n; ++j) {
            values[j] = d[order[j]];
            for (int64_t i = 0; i < n; ++i) vectors[j * n + i] = w[i * n + order[j]];
        }
        free(order);
    }
    free(w);
    free(d);
    free(e);
    return rc;
}

/* ---- eigSVD: decompositions.cpp:21-75 ------------------------------------- */

static void sign_convention(int64_t rows, int64_t cols, double* u, double* v) {
    /* decompositions.cpp:21-35: first nonzero of each V column made >= 0 */
    for (int64_t j = 0; j < cols; ++j) {
        double* vj = v + j * cols;
        double lead = 0.0;
        for (int64_t i = 0; i < cols; ++i)
            if (vj[i] != 0.0) {
                lead = vj[i];
                break;
            }
        if (lead >= 0.0) continue;
        for (int64_t i = 0; i < cols; ++i) vj[i] = -vj[i];
        double* uj = u + j * rows;
        for (int64_t i = 0; i < rows; ++i) uj[i] = -uj[i];
    }
}

int orc_eig_svd(int64_t rows, int64_t cols, const double* c, double* u, double* s, double* v) {
    const int64_t m = rows, n = cols;
    if (m < n) return fail(ORC_SHAPE, -1, "eig_svd: needs rows >= cols (factor the transpose instead)");
    if (n == 0) return ORC_OK;
    double* g = (double*)malloc(sizeof(double) * n * n);
    double* lam = (double*)malloc(sizeof(double) * n);
    double* vec = (double*)malloc(sizeof(double) * n * n);
    orc_gram(m, n, c, g);
    int rc = orc_sym_eig(n, g, lam, vec);
    if (rc == ORC_OK) {
        const double lambda_max = fmax(lam[n - 1], 0.0);
        const double rank_floor = (double)(m > n ? m : n) * DBL_EPSILON * sqrt(lambda_max);
        const double floor2 = rank_floor * rank_floor;
        for (int64_t r = 0; r < n && rc == ORC_OK; ++r) {
            const double lambda = lam[n - 1 - r];
            if (lambda <= floor2) {
                rc = fail(ORC_RANK, r, "eig_svd: singular value at or below the rank floor");
                break;
            }
            s[r] = sqrt(lambda);
            memcpy(v + r * n, vec + (n - 1 - r) * n, sizeof(double) * n);
        }
        if (rc == ORC_OK) {
            orc_matmul(m, n, n, c, v, u);
            for (int64_t r = 0; r < n; ++r) {
                const double inv = 1.0 / s[r];
                double* ur = u + r * m;
                for (int64_t i = 0; i < m; ++i) ur[i] *= inv;
            }
            sign_convention(m, n, u, v);
        }
    }
    free(g);
    free(lam);
    free(vec);
    return rc;
}

/* ---- solver: solver.cpp --------------------------------------------------- */

static int64_t eff_s(const orc_config* c) { /* solver.hpp:36 */
    return c->s >= 0 ? c->s : (c->k / 2 > 0 ? c->k / 2 : 1);
}

int orc_validate_config(const orc_config* cfg, int64_t rows, int64_t cols) {
    /* solver.cpp:15-32 */
    if (rows < 1 || cols < 1) return fail(ORC_SHAPE, -1, "solver needs a non-empty matrix");
    if (cfg->k < 1) return fail(ORC_CONFIG, -1, "k must be >= 1");
    const int64_t s = eff_s(cfg);
    const int64_t mn = rows < cols ? rows : cols;
    if (cfg->k + s > mn) return fail(ORC_CONFIG, -1, "k + s exceeds min(rows, cols)");
    if (cfg->alg == ORC_DASH) {
        if (s < 1) return fail(ORC_CONFIG, -1, "the accuracy-controlled mode needs oversampling s >= 1");
        if (!(cfg->tol > 0.0)) return fail(ORC_CONFIG, -1, "tol must be positive");
        if (cfg->p_max < 1) return fail(ORC_CONFIG, -1, "p_max must be >= 1");
    } else {
        if (cfg->p < 0) return fail(ORC_CONFIG, -1, "fixed-power algorithms need p >= 0");
    }
    if (cfg->orth_qr && cfg->alg != ORC_BASIC)
        return fail(ORC_CONFIG, -1, "the qr orthonormalizer applies to the basic algorithm only");
    return ORC_OK;
}

double orc_update_shift(double alpha, double s_ll) { /* solver.cpp:34-36 */
    return s_ll > alpha ? (s_ll + alpha) / 2.0 : alpha;
}

int orc_pve_stop_check(const double* prev, int64_t n_prev, double alpha_prev, const double* cur,
                       int64_t n_cur, double alpha, int64_t k, double tol, int* stop) {
    /* solver.cpp:38-50: operand order as written; NaN and x/0 never stop */
    if (k < 1) return fail(ORC_SHAPE, -1, "pve_stop_check: k must be >= 1");
    if (n_prev < k + 1 || n_cur < k + 1)
        return fail(ORC_SHAPE, -1, "pve_stop_check: surrogate arrays must hold at least k+1 values");
    const double denom = cur[k] + alpha;
    *stop = 1;
    for (int64_t i = 0; i < k; ++i) {
        const double change = fabs(prev[i] + alpha_prev - cur[i] - alpha);
        if (!(change / denom <= tol)) {
            *stop = 0;
            break;
        }
    }
    return ORC_OK;
}

/* Factor assembly for a row-space basis q (solver.cpp:159-164, truncate :60-66):
 * B = A q, eigSVD(B), keep k columns, V = q * V'[:, :k]. */
int orc_finalize_row_basis(const orc_csr* a, const double* q, int64_t l, int64_t k, double* u,
                           double* s, double* v) {
    if (k < 1 || k > l) return fail(ORC_SHAPE, -1, "finalize_row_basis: k out of range");
    const int64_t m = a->rows, n = a->cols;
    double* b = (double*)malloc(sizeof(double) * m * l);
    double* fu = (double*)malloc(sizeof(double) * m * l);
    double* fs = (double*)malloc(sizeof(double) * l);
    double* fv = (double*)malloc(sizeof(double) * l * l);
    orc_spmm(a, q, l, b);
    int rc = orc_eig_svd(m, l, b, fu, fs, fv);
    if (rc == ORC_OK) {
        memcpy(u, fu, sizeof(double) * m * k);
        memcpy(s, fs, sizeof(double) * k);
        orc_matmul(n, l, k, q, fv, v);
    }
    free(b);
    free(fu);
    free(fs);
    free(fv);
    return rc;
}

/* run_shifted_iterations (solver.cpp:76-116) + finalize, for a tall-or-square
 * a (solve_direct :143-155). */
static int shifted_direct(const orc_csr* a, const orc_csr* at, const orc_config* cfg, double* u,
                          double* s_out, double* v, double* alphas, double* s_hat, int64_t cap,
                          int64_t* iterations, int* stop_reason) {
    const int64_t m = a->rows, n = a->cols;
    const int64_t l = cfg->k + eff_s(cfg);
    const int dash = cfg->alg == ORC_DASH;
    const int64_t max_iters = dash ? cfg->p_max : cfg->p;
    double* omega = (double*)malloc(sizeof(double) * m * l);
    double* t = (double*)malloc(sizeof(double) * n * l);
    double* y = (double*)malloc(sizeof(double) * m * l);
    double* q = (double*)malloc(sizeof(double) * n * l);
    double* qn = (double*)malloc(sizeof(double) * n * l);
    double* fs = (double*)malloc(sizeof(double) * l);
    double* fv = (double*)malloc(sizeof(double) * l * l);
    double* s_stored = (double*)calloc((size_t)l, sizeof(double));
    int rc;

    orc_gaussian_matrix(m, l, cfg->seed, omega); /* Omega is rows x l (solver.cpp:83) */
    orc_spmm(at, omega, l, t);
    rc = orc_eig_svd(n, l, t, q, fs, fv);
    *stop_reason = dash ? ORC_STOP_P_MAX : ORC_STOP_FIXED_P;
    *iterations = 0;
    double alpha = 0.0, alpha_stored = 0.0;
    for (int64_t j = 1; rc == ORC_OK && j <= max_iters; ++j) {
        orc_spmm(a, q, l, y);
        orc_spmm(at, y, l, t);
        if (alpha != 0.0) orc_add_scaled(n * l, t, -alpha, q);
        rc = orc_eig_svd(n, l, t, qn, fs, fv);
        if (rc != ORC_OK) break;
        if (j - 1 < cap) {
            alphas[j - 1] = alpha;
            memcpy(s_hat + (j - 1) * l, fs, sizeof(double) * l);
        }
        *iterations = j;
        int stop = 0;
        if (dash) {
            rc = orc_pve_stop_check(s_stored, l, alpha_stored, fs, l, alpha, cfg->k, cfg->tol, &stop);
            if (rc != ORC_OK) break;
        }
        double* tmp = q;
        q = qn;
        qn = tmp;
        if (stop) {
            *stop_reason = ORC_STOP_TOL_MET;
            break;
        }
        if (cfg->alg != ORC_FIXED_SHIFT || j == 1) alpha = orc_update_shift(alpha, fs[l - 1]);
        memcpy(s_stored, fs, sizeof(double) * l);
        alpha_stored = alpha;
    }
    if (rc == ORC_OK) rc = orc_finalize_row_basis(a, q, l, cfg->k, u, s_out, v);
    free(omega);
    free(t);
    free(y);
    free(q);
    free(qn);
    free(fs);
    free(fv);
    free(s_stored);
    return rc;
}

/* qr_orth (decompositions.cpp:77-126): Householder QR of the column-major
 * m x n block c, the explicit m x n Q by backward accumulation; RankDeficient
 * when |R(k, k)| <= max(m, n) * eps * max |R(j, j)|. */
int orc_qr_orth(int64_t m, int64_t n, const double* c, double* q) {
    if (m < n) return fail(ORC_SHAPE, -1, "qr_orth: needs rows >= cols");
    if (n == 0) return ORC_OK;
    double* w = (double*)malloc(sizeof(double) * m * n);
    double* tau = (double*)calloc((size_t)n, sizeof(double));
    double* rdiag = (double*)calloc((size_t)n, sizeof(double));
    memcpy(w, c, sizeof(double) * m * n);
    for (int64_t k = 0; k < n; ++k) {
        double* wk = w + k * m;
        double norm2 = 0.0;
        for (int64_t i = k; i < m; ++i) norm2 += wk[i] * wk[i];
        const double alpha = wk[k];
        const double beta = alpha >= 0.0 ? -sqrt(norm2) : sqrt(norm2);
        rdiag[k] = beta;
        if (beta == 0.0) continue;
        tau[k] = (beta - alpha) / beta;
        const double scale = 1.0 / (alpha - beta);
        for (int64_t i = k + 1; i < m; ++i) wk[i] *= scale;
        wk[k] = 1.0;
        for (int64_t j = k + 1; j < n; ++j) {
            double* wj = w + j * m;
            double d = 0.0; /* dot(wk + k, wj + k, m - k) */
            for (int64_t i = k; i < m; ++i) d += wk[i] * wj[i];
            const double t = tau[k] * d;
            for (int64_t i = k; i < m; ++i) wj[i] -= t * wk[i];
        }
    }
    double max_diag = 0.0;
    for (int64_t k = 0; k < n; ++k) max_diag = fmax(max_diag, fabs(rdiag[k]));
    const double floor_ = (double)(m > n ? m : n) * DBL_EPSILON * max_diag;
    for (int64_t k = 0; k < n; ++k)
        if (fabs(rdiag[k]) <= floor_) {
            free(w);
            free(tau);
            free(rdiag);
            return fail(ORC_RANK, k, "qr_orth: diagonal of R at or below the rank floor");
        }
    memset(q, 0, sizeof(double) * m * n);
    for (int64_t j = 0; j < n; ++j) q[j * m + j] = 1.0;
    for (int64_t k = n - 1; k >= 0; --k) {
        if (tau[k] == 0.0) continue;
        const double* wk = w + k * m;
        for (int64_t j = k; j < n; ++j) {
            double* qj = q + j * m;
            double d = 0.0;
            for (int64_t i = k; i < m; ++i) d += wk[i] * qj[i];
            const double t = tau[k] * d;
            for (int64_t i = k; i < m; ++i) qj[i] -= t * wk[i];
        }
    }
    free(w);
    free(tau);
    free(rdiag);
    return ORC_OK;
}

/* basic_core + finalize_col_basis (solver.cpp:118-141, :166-176) on a as
 * given: q = orth(A Omega), Omega = gaussian_matrix(a.cols, l, seed); p times
 * q = orth(A (A^T q)); orth = eig_svd(.).u (its s is the trace's s_hat, alphas
 * 0) or qr_orth (empty s_hat: left untouched). Finalize: f = eig_svd(A^T q),
 * U = q f.v[:, :k], s = f.s[:k], V = f.u[:, :k]. */
static int basic_direct(const orc_csr* a, const orc_csr* at, const orc_config* cfg, int qr, double* u,
                        double* s_out, double* v, double* alphas, double* s_hat, int64_t cap,
                        int64_t* iterations, int* stop_reason) {
    const int64_t m = a->rows, n = a->cols;
    const int64_t l = cfg->k + eff_s(cfg), k = cfg->k;
    double* omega = (double*)malloc(sizeof(double) * n * l);
    double* t = (double*)malloc(sizeof(double) * n * l);
    double* y = (double*)malloc(sizeof(double) * m * l);
    double* q = (double*)malloc(sizeof(double) * m * l);
    double* fs = (double*)malloc(sizeof(double) * l);
    double* fv = (double*)malloc(sizeof(double) * l * l);
    double* fu = (double*)malloc(sizeof(double) * n * l);
    int rc;
    orc_gaussian_matrix(n, l, cfg->seed, omega);
    orc_spmm(a, omega, l, y);
    rc = qr ? orc_qr_orth(m, l, y, q) : orc_eig_svd(m, l, y, q, fs, fv);
    *iterations = 0;
    *stop_reason = ORC_STOP_FIXED_P;
    for (int64_t j = 1; rc == ORC_OK && j <= cfg->p; ++j) {
        orc_spmm(at, q, l, t);
        orc_spmm(a, t, l, y);
        rc = qr ? orc_qr_orth(m, l, y, q) : orc_eig_svd(m, l, y, q, fs, fv);
        if (rc != ORC_OK) break;
        if (j - 1 < cap) {
            alphas[j - 1] = 0.0;
            if (!qr) memcpy(s_hat + (j - 1) * l, fs, sizeof(double) * l);
        }
        *iterations = j;
    }
    if (rc == ORC_OK) {
        orc_spmm(at, q, l, t);
        rc = orc_eig_svd(n, l, t, fu, fs, fv);
        if (rc == ORC_OK) {
            orc_matmul(m, l, k, q, fv, u); /* head_cols(f.v, k) is the leading l x k block */
            memcpy(s_out, fs, sizeof(double) * k);
            memcpy(v, fu, sizeof(double) * n * k);
        }
    }
    free(omega);
    free(t);
    free(y);
    free(q);
    free(fs);
    free(fv);
    free(fu);
    return rc;
}

int orc_solve(const orc_csr* a, const orc_csr* at, const orc_config* cfg, double* u, double* s,
              double* v, double* alphas, double* s_hat, int64_t cap, int64_t* iterations,
              int* stop_reason) {
    /* solver.cpp:214-223: wide inputs run on the transpose and swap U/V */
    int rc = orc_validate_config(cfg, a->rows, a->cols);
    if (rc != ORC_OK) return rc;
    if (cfg->alg == ORC_BASIC) {
        const int qr = cfg->orth_qr != 0;
        if (a->rows < a->cols)
            return basic_direct(at, a, cfg, qr, v, s, u, alphas, s_hat, cap, iterations, stop_reason);
        return basic_direct(a, at, cfg, qr, u, s, v, alphas, s_hat, cap, iterations, stop_reason);
    }
    if (a->rows < a->cols)
        return shifted_direct(at, a, cfg, v, s, u, alphas, s_hat, cap, iterations, stop_reason);
    return shifted_direct(a, at, cfg, u, s, v, alphas, s_hat, cap, iterations, stop_reason);
}
