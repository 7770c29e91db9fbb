// Host cross-check of the table-driven correctly rounded log / cos of
// paper_2404_09276_b200/csrc/dd_math.cuh against the long-series evaluations
// they replace, on Box-Muller-shaped inputs plus edge cases. Built and run by
// tests/test_ddm.py; prints "mismatches <log> <cos> of <n>".
#define __host__
#define __device__
#define __forceinline__ inline
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <initializer_list>

#include "../paper_2404_09276_b200/csrc/dd_math.cuh"

static uint64_t sm64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double unit(uint64_t x) { return (static_cast<double>(x >> 11) + 0.5) * 0x1p-53; }
static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    long bad_log = 0, bad_cos = 0, total = 0, slow_log = 0, slow_cos = 0;
    auto check = [&](double u, double x) {
        ++total;
        // the fast paths (Ziv test + fallback), as rng.cuh uses them
        double fl, fc;
        if (!dsvd::ddm::log_fast(u, &fl)) {
            fl = dsvd::ddm::log_cr(u);
            ++slow_log;
        }
        if (!dsvd::ddm::cos_fast(x, &fc)) {
            fc = dsvd::ddm::cos_cr(x);
            ++slow_cos;
        }
        if (!same(fl, dsvd::ddm::log_cr_series(u))) {
            if (bad_log < 5) std::printf("fast log %a: %a vs %a\n", u, fl, dsvd::ddm::log_cr_series(u));
            ++bad_log;
        }
        if (!same(fc, dsvd::ddm::cos_cr_series(x))) {
            if (bad_cos < 5) std::printf("fast cos %a: %a vs %a\n", x, fc, dsvd::ddm::cos_cr_series(x));
            ++bad_cos;
        }
        if (!same(dsvd::ddm::log_cr(u), dsvd::ddm::log_cr_series(u))) {
            if (bad_log < 5) std::printf("log %a: %a vs %a\n", u, dsvd::ddm::log_cr(u), dsvd::ddm::log_cr_series(u));
            ++bad_log;
        }
        if (!same(dsvd::ddm::cos_cr(x), dsvd::ddm::cos_cr_series(x))) {
            if (bad_cos < 5) std::printf("cos %a: %a vs %a\n", x, dsvd::ddm::cos_cr(x), dsvd::ddm::cos_cr_series(x));
            ++bad_cos;
        }
    };
    for (long i = 0; i < n; ++i) {
        const double u1 = unit(sm64(7, 2 * i)), u2 = unit(sm64(7, 2 * i + 1));
        check(u1, 6.283185307179586 * u2);
    }
    // edges: extremes of the unit interval, table boundaries, quadrant boundaries
    check(0x1p-54, 0x1p-60);
    check(1.0 - 0x1p-53, 6.283185307179586 * (1.0 - 0x1p-53));
    for (int i = 45; i <= 91; ++i)
        for (double d : {-0x1p-20, -0x1p-40, 0.0, 0x1p-40, 0x1p-20}) {
            const double f = (i + 0.5) / 64.0 + d;
            check(f * 0.5, f);
        }
    for (int k = 0; k <= 4; ++k)
        for (int j = -26; j <= 26; ++j)
            for (double d : {-0x1p-30, 0.0, 0x1p-30}) {
                const double x = k * 1.5707963267948966 + (j + 0.5) / 32.0 + d;
                if (x > 0 && x < 6.3) check(0.5, x);
            }
    // near-midpoint log / cos arguments: the fast path must decline them
    for (long i = 0; i < n / 100; ++i) {
        const double u = unit(sm64(11, i));
        check(u, 6.283185307179586 * unit(sm64(13, i)));
        check(std::nextafter(u, 1.0), std::nextafter(6.283185307179586 * unit(sm64(13, i)), 7.0));
    }
    std::printf("fallbacks log %ld cos %ld of %ld\n", slow_log, slow_cos, total);
    std::printf("mismatches %ld %ld of %ld\n", bad_log, bad_cos, total);
    return 0;
}
