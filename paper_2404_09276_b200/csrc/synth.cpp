// Deterministic synthetic inputs for the BASELINE.json configurations (host
// side; input preparation, not part of the solve path). Every draw comes from
// a counter-based SplitMix64 stream indexed by (row, draw), so the matrices
// are identical for any thread count.
//
//  - sparse_random: the reference generator for config 1
//    (synthetic.cpp:72-120): per row, nnz_per_row uniform column draws,
//    N(0,1) values scaled by 1/sqrt(1+i) with row decay, duplicates summed in
//    sorted order, zero sums dropped.
//  - powerlaw: configs 2 and 3. Row degree round(exp(mu + sigma z)) clamped
//    to [1, cols]; column ranks ~ Zipf(s) by inverse-CDF search, mapped through
//    a seeded Fisher-Yates permutation; a row draws until it holds `degree`
//    DISTINCT columns (sampling without replacement); values N(0,1)
//    or integer ratings 1..5 with probabilities .05/.10/.25/.35/.25.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/dashsvd_b200.h"

namespace {

uint64_t sm64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double unit(uint64_t x) { return (static_cast<double>(x >> 11) + 0.5) * 0x1p-53; }

double normal(uint64_t seed, uint64_t i) {
    const double u1 = unit(sm64(seed, 2 * i));
    const double u2 = unit(sm64(seed, 2 * i + 1));
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

struct Result {
    std::vector<int64_t> off, idx;
    std::vector<double> val;
};
Result g_res;

thread_local std::string t_msg;

}  // namespace

extern "C" {

int dsvd_synth_sparse_random(int64_t rows, int64_t cols, int64_t npr, uint64_t seed, int decay,
                             int64_t* nnz) {
    if (rows < 1 || cols < 1 || npr < 1 || npr > cols) return DSVD_SHAPE;
    const uint64_t col_seed = sm64(seed, 0), val_seed = sm64(seed, 1);
    std::vector<std::vector<std::pair<int64_t, double>>> buf(rows);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        auto& row = buf[i];
        row.reserve(npr);
        const double scale = decay ? 1.0 / std::sqrt(1.0 + static_cast<double>(i)) : 1.0;
        for (int64_t t = 0; t < npr; ++t) {
            const uint64_t e = static_cast<uint64_t>(i) * npr + t;
            row.emplace_back(static_cast<int64_t>(sm64(col_seed, e) % static_cast<uint64_t>(cols)),
                             scale * normal(val_seed, e));
        }
        std::sort(row.begin(), row.end());
        size_t w = 0;
        for (size_t r = 0; r < row.size();) {
            auto cur = row[r++];
            while (r < row.size() && row[r].first == cur.first) cur.second += row[r++].second;
            if (cur.second != 0.0) row[w++] = cur;
        }
        row.resize(w);
    }
    Result& R = g_res;
    R.off.assign(rows + 1, 0);
    for (int64_t i = 0; i < rows; ++i) R.off[i + 1] = R.off[i] + static_cast<int64_t>(buf[i].size());
    R.idx.resize(R.off[rows]);
    R.val.resize(R.off[rows]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        int64_t p = R.off[i];
        for (const auto& e : buf[i]) {
            R.idx[p] = e.first;
            R.val[p++] = e.second;
        }
    }
    *nnz = R.off[rows];
    return DSVD_OK;
}

int dsvd_synth_powerlaw(int64_t rows, int64_t cols, double mu, double sigma, double zipf_s,
                        int ratings, uint64_t seed, int64_t* nnz) {
    if (rows < 1 || cols < 1) return DSVD_SHAPE;
    const uint64_t deg_seed = sm64(seed, 0), col_seed = sm64(seed, 1), val_seed = sm64(seed, 2),
                   perm_seed = sm64(seed, 3);
    // Zipf CDF over ranks 1..cols
    std::vector<double> cdf(cols);
    double acc = 0.0;
    for (int64_t r = 0; r < cols; ++r) {
        acc += std::pow(static_cast<double>(r + 1), -zipf_s);
        cdf[r] = acc;
    }
    for (auto& c : cdf) c /= acc;
    cdf[cols - 1] = 1.0;
    // seeded Fisher-Yates permutation rank -> column
    std::vector<int64_t> perm(cols);
    std::iota(perm.begin(), perm.end(), 0);
    for (int64_t i = cols - 1; i > 0; --i) {
        const int64_t j = static_cast<int64_t>(sm64(perm_seed, i) % static_cast<uint64_t>(i + 1));
        std::swap(perm[i], perm[j]);
    }
    Result& R = g_res;
    R.off.assign(rows + 1, 0);
    std::vector<int64_t> deg(rows);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        const double d = std::llround(std::exp(mu + sigma * normal(deg_seed, i)));
        deg[i] = static_cast<int64_t>(std::min<double>(std::max<double>(d, 1.0), static_cast<double>(cols)));
    }
    for (int64_t i = 0; i < rows; ++i) R.off[i + 1] = R.off[i] + deg[i];
    const int64_t total = R.off[rows];
    R.idx.resize(total);
    R.val.resize(total);
    const uint64_t kStride = uint64_t(1) << 26;  // draws reserved per row
    bool overflow = false;
#pragma omp parallel
    {
        std::unordered_set<int64_t> seen;
        std::vector<std::pair<int64_t, double>> row;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < rows; ++i) {
            const int64_t d = deg[i];
            seen.clear();
            seen.reserve(static_cast<size_t>(d) * 2);
            row.clear();
            uint64_t t = 0;
            while (static_cast<int64_t>(row.size()) < d) {
                if (t >= kStride) {
                    overflow = true;
                    break;
                }
                const double u = unit(sm64(col_seed, static_cast<uint64_t>(i) * kStride + t++));
                const int64_t rank = std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
                const int64_t c = perm[std::min<int64_t>(rank, cols - 1)];
                if (!seen.insert(c).second) continue;
                const uint64_t e = static_cast<uint64_t>(i) * kStride + row.size();
                double v;
                if (ratings) {
                    const double r = unit(sm64(val_seed, e));
                    v = r < 0.05 ? 1.0 : r < 0.15 ? 2.0 : r < 0.40 ? 3.0 : r < 0.75 ? 4.0 : 5.0;
                } else {
                    v = normal(val_seed, e);
                    if (v == 0.0) v = 0x1p-60;  // canonical form stores no explicit zeros
                }
                row.emplace_back(c, v);
            }
            std::sort(row.begin(), row.end());
            int64_t p = R.off[i];
            for (const auto& e : row) {
                R.idx[p] = e.first;
                R.val[p++] = e.second;
            }
        }
    }
    if (overflow) return DSVD_OTHER;
    *nnz = total;
    return DSVD_OK;
}

int dsvd_synth_fetch(int64_t* offsets, int64_t* col_indices, double* values) {
    Result& R = g_res;
    std::memcpy(offsets, R.off.data(), sizeof(int64_t) * R.off.size());
    std::memcpy(col_indices, R.idx.data(), sizeof(int64_t) * R.idx.size());
    std::memcpy(values, R.val.data(), sizeof(double) * R.val.size());
    g_res = Result();
    return DSVD_OK;
}

}  // extern "C"
