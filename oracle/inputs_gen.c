/* TEST / BASELINE INFRASTRUCTURE ONLY — host restatement of the synthetic
 * input generators of BASELINE.json configs 2-5, so that the CPU reference arm
 * of bench.py (and the parity tools) can build the exact input CSR without
 * loading the product library (paper_2404_09276_b200). Nothing in the product
 * path uses this file.
 *
 *  - gen_rmat: the R-MAT rule of dsvd_synth_rmat (ingest.cuh / ingest.cu
 *    rmat_keys_kernel + rmat_emit_kernel): draw e picks one quadrant per level
 *    from 16-bit slices of splitmix64_at(edge_seed, e*H + t/4), H = ceil(scale/4);
 *    duplicate (row, col) pairs keep their FIRST draw; value 1.0 or
 *    ((splitmix64_at(val_seed, first_draw) >> 11) + 1) * 2^-53. The reference
 *    ships no R-MAT generator (BASELINE.json configs 4/5 define the family).
 *    Rows are bucketed (counting sort by row), each bucket is sorted by
 *    (col, draw) and deduplicated — the same set as the device's radix sort.
 *  - gen_powerlaw: dsvd_synth_powerlaw (synth.cpp), statement for statement
 *    (compile with -ffp-contract=off and no -march, like synth.cpp, so the
 *    libm calls and roundings are identical).
 * splitmix64 / normal draws follow random.cpp:8-27.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t sm64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double unit(uint64_t x) { return ((double)(x >> 11) + 0.5) * 0x1p-53; }

static double normal(uint64_t seed, uint64_t i) {
    const double u1 = unit(sm64(seed, 2 * i));
    const double u2 = unit(sm64(seed, 2 * i + 1));
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

static int64_t g_rows, g_nnz;
static int64_t* g_off;
static int64_t* g_idx;
static double* g_val;

static void release(void) {
    free(g_off);
    free(g_idx);
    free(g_val);
    g_off = g_idx = NULL;
    g_val = NULL;
    g_rows = g_nnz = 0;
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Returns 0 on success, 1 on bad arguments, 2 on allocation failure. */
int gen_rmat(int scale, int64_t draws, double a, double b, double c, int uniform, uint64_t seed, int64_t* nnz_out) {
    release();
    if (scale < 1 || scale > 30 || draws < 0 || draws > 0xffffffffLL) return 1;
    const int64_t n = (int64_t)1 << scale;
    const uint32_t t_a = (uint32_t)llround(a * 65536.0);
    const uint32_t t_ab = (uint32_t)llround((a + b) * 65536.0);
    const uint32_t t_abc = (uint32_t)llround((a + b + c) * 65536.0);
    const uint64_t edge_seed = sm64(seed, 0), val_seed = sm64(seed, 1);
    const int H = (scale + 3) / 4;
    uint32_t* row = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(draws > 0 ? draws : 1));
    uint32_t* col = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(draws > 0 ? draws : 1));
    int64_t* start = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!row || !col || !start) {
        free(row);
        free(col);
        free(start);
        return 2;
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < draws; ++e) {
        uint64_t r = 0, cc = 0, h = 0;
        for (int t = 0; t < scale; ++t) {
            if ((t & 3) == 0) h = sm64(edge_seed, (uint64_t)e * (uint64_t)H + (uint64_t)(t >> 2));
            const uint32_t q = (uint32_t)(h >> (16 * (t & 3))) & 0xffffu;
            const uint32_t quad = q < t_a ? 0u : (q < t_ab ? 1u : (q < t_abc ? 2u : 3u));
            r = (r << 1) | (quad >> 1);
            cc = (cc << 1) | (quad & 1u);
        }
        row[e] = (uint32_t)r;
        col[e] = (uint32_t)cc;
#pragma omp atomic
        start[r + 1] += 1;
    }
    for (int64_t i = 0; i < n; ++i) start[i + 1] += start[i];
    /* bucket (col << 32 | draw) by row; order inside a bucket is fixed by the sort below */
    uint64_t* bucket = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(draws > 0 ? draws : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!bucket || !fill) {
        free(row);
        free(col);
        free(start);
        free(bucket);
        free(fill);
        return 2;
    }
    memcpy(fill, start, sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < draws; ++e) {
        int64_t pos;
#pragma omp atomic capture
        pos = fill[row[e]]++;
        bucket[pos] = ((uint64_t)col[e] << 32) | (uint64_t)e;
    }
    free(row);
    free(col);
    free(fill);
    /* sort each row, keep the first draw of each column */
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!cnt) {
        free(start);
        free(bucket);
        return 2;
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t* p = bucket + start[i];
        const int64_t len = start[i + 1] - start[i];
        if (len > 1) qsort(p, (size_t)len, sizeof(uint64_t), cmp_u64);
        int64_t u = 0;
        for (int64_t j = 0; j < len; ++j)
            if (j == 0 || (p[j] >> 32) != (p[j - 1] >> 32)) p[u++] = p[j];
        cnt[i + 1] = u;
    }
    g_off = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!g_off) {
        free(start);
        free(bucket);
        free(cnt);
        return 2;
    }
    g_off[0] = 0;
    for (int64_t i = 0; i < n; ++i) g_off[i + 1] = g_off[i] + cnt[i + 1];
    free(cnt);
    const int64_t nnz = g_off[n];
    g_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    g_val = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    if (!g_idx || !g_val) {
        free(start);
        free(bucket);
        release();
        return 2;
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t* p = bucket + start[i];
        for (int64_t j = 0, w = g_off[i]; w < g_off[i + 1]; ++j, ++w) {
            g_idx[w] = (int64_t)(p[j] >> 32);
            g_val[w] = uniform ? ((double)(sm64(val_seed, p[j] & 0xffffffffu) >> 11) + 1.0) * 0x1p-53 : 1.0;
        }
    }
    free(start);
    free(bucket);
    g_rows = n;
    g_nnz = nnz;
    *nnz_out = nnz;
    return 0;
}

/* ---- powerlaw (configs 2/3): dsvd_synth_powerlaw ------------------------- */

typedef struct {
    int64_t col;
    double val;
} Entry;

static int cmp_entry(const void* a, const void* b) {
    const Entry* x = (const Entry*)a;
    const Entry* y = (const Entry*)b;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return x->val < y->val ? -1 : (x->val > y->val ? 1 : 0);
}

/* first index r with cdf[r] >= u (std::lower_bound) */
static int64_t lower_bound(const double* cdf, int64_t n, double u) {
    int64_t lo = 0, len = n;
    while (len > 0) {
        const int64_t half = len / 2;
        if (cdf[lo + half] < u) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

int gen_powerlaw(int64_t rows, int64_t cols, double mu, double sigma, double zipf_s, int ratings, uint64_t seed,
                 int64_t* nnz_out) {
    release();
    if (rows < 1 || cols < 1) return 1;
    const uint64_t deg_seed = sm64(seed, 0), col_seed = sm64(seed, 1), val_seed = sm64(seed, 2),
                   perm_seed = sm64(seed, 3);
    double* cdf = (double*)malloc(sizeof(double) * (size_t)cols);
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)cols);
    int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)rows);
    g_off = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
    if (!cdf || !perm || !deg || !g_off) {
        free(cdf);
        free(perm);
        free(deg);
        release();
        return 2;
    }
    double acc = 0.0;
    for (int64_t r = 0; r < cols; ++r) {
        acc += pow((double)(r + 1), -zipf_s);
        cdf[r] = acc;
    }
    for (int64_t r = 0; r < cols; ++r) cdf[r] /= acc;
    cdf[cols - 1] = 1.0;
    for (int64_t i = 0; i < cols; ++i) perm[i] = i;
    for (int64_t i = cols - 1; i > 0; --i) {
        const int64_t j = (int64_t)(sm64(perm_seed, (uint64_t)i) % (uint64_t)(i + 1));
        const int64_t t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        const double d = (double)llround(exp(mu + sigma * normal(deg_seed, (uint64_t)i)));
        const double lo = d > 1.0 ? d : 1.0;
        deg[i] = (int64_t)(lo < (double)cols ? lo : (double)cols);
    }
    for (int64_t i = 0; i < rows; ++i) g_off[i + 1] = g_off[i] + deg[i];
    const int64_t total = g_off[rows];
    g_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    g_val = (double*)malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
    if (!g_idx || !g_val) {
        free(cdf);
        free(perm);
        free(deg);
        release();
        return 2;
    }
    const uint64_t kStride = (uint64_t)1 << 26;
    int overflow = 0;
#pragma omp parallel
    {
        /* open-addressing set of the row's columns (synth.cpp uses unordered_set) */
        size_t cap = 0;
        int64_t* set = NULL;
        Entry* row = NULL;
        size_t row_cap = 0;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < rows; ++i) {
            const int64_t d = deg[i];
            size_t need = 16;
            while (need < (size_t)d * 2) need <<= 1;
            if (need > cap) {
                free(set);
                cap = need;
                set = (int64_t*)malloc(sizeof(int64_t) * cap);
            }
            for (size_t t = 0; t < cap; ++t) set[t] = -1;
            if ((size_t)d > row_cap) {
                free(row);
                row_cap = (size_t)d;
                row = (Entry*)malloc(sizeof(Entry) * row_cap);
            }
            int64_t have = 0;
            uint64_t t = 0;
            while (have < d) {
                if (t >= kStride) {
#pragma omp atomic write
                    overflow = 1;
                    break;
                }
                const double u = unit(sm64(col_seed, (uint64_t)i * kStride + t++));
                int64_t rank = lower_bound(cdf, cols, u);
                const int64_t cidx = perm[rank < cols - 1 ? rank : cols - 1];
                size_t hsh = (size_t)(sm64(0, (uint64_t)cidx)) & (cap - 1);
                int dup = 0;
                while (set[hsh] != -1) {
                    if (set[hsh] == cidx) {
                        dup = 1;
                        break;
                    }
                    hsh = (hsh + 1) & (cap - 1);
                }
                if (dup) continue;
                set[hsh] = cidx;
                const uint64_t e = (uint64_t)i * kStride + (uint64_t)have;
                double v;
                if (ratings) {
                    const double r = unit(sm64(val_seed, e));
                    v = r < 0.05 ? 1.0 : r < 0.15 ? 2.0 : r < 0.40 ? 3.0 : r < 0.75 ? 4.0 : 5.0;
                } else {
                    v = normal(val_seed, e);
                    if (v == 0.0) v = 0x1p-60;
                }
                row[have].col = cidx;
                row[have].val = v;
                ++have;
            }
            qsort(row, (size_t)have, sizeof(Entry), cmp_entry);
            int64_t p = g_off[i];
            for (int64_t j = 0; j < have; ++j) {
                g_idx[p] = row[j].col;
                g_val[p++] = row[j].val;
            }
        }
        free(set);
        free(row);
    }
    free(cdf);
    free(perm);
    free(deg);
    if (overflow) {
        release();
        return 3;
    }
    g_rows = rows;
    g_nnz = total;
    *nnz_out = total;
    return 0;
}

void gen_fetch(int64_t* off, int64_t* idx, double* val) {
    memcpy(off, g_off, sizeof(int64_t) * (size_t)(g_rows + 1));
    memcpy(idx, g_idx, sizeof(int64_t) * (size_t)g_nnz);
    memcpy(val, g_val, sizeof(double) * (size_t)g_nnz);
    release();
}
