// Correctly rounded double log and cos, evaluated in double-double (~104-bit)
// arithmetic and rounded once, for the Box-Muller draws of the sketch
// (random.cpp:23-27). CUDA's libm log/cos are only <= 1 ulp; glibc's (used by
// the reference) are correctly rounded except within ~0.02 ulp of a rounding
// midpoint, where they misround (~0.08% of log and ~0.13% of cos evaluations
// on the config-1 sketch; each case confirmed against 60-digit decimal
// arithmetic). The correctly rounded result is the one the
// reference's formula defines mathematically.
//
// Everything is __host__ __device__ so the host tests can cross-check it.
#pragma once

#include <cmath>

#include "dd_consts.cuh"

namespace dsvd {
namespace ddm {

struct dd {
    double hi, lo;
};

__host__ __device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}

__host__ __device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}

__host__ __device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = a * b;
    return {p, fma(a, b, -p)};
}

__host__ __device__ __forceinline__ dd add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}

__host__ __device__ __forceinline__ dd mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}

__host__ __device__ __forceinline__ dd mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo += a.lo * b;
    return quick_two_sum(p.hi, p.lo);
}

__host__ __device__ __forceinline__ dd div(dd a, dd b) {
    const double q1 = a.hi / b.hi;
    dd r = add(a, mul_d(b, -q1));
    const double q2 = r.hi / b.hi;
    r = add(r, mul_d(b, -q2));
    const double q3 = r.hi / b.hi;
    dd q = quick_two_sum(q1, q2);
    return add(q, dd{q3, 0.0});
}

// Table entries (hi, lo) of dd_consts.cuh: device copies through the
// read-only cache, host copies in host code.
__host__ __device__ __forceinline__ dd tab_ld(const double* host, const double* dev, int i) {
#ifdef __CUDA_ARCH__
    const double2 v = __ldg(reinterpret_cast<const double2*>(dev) + i);
    return {v.x, v.y};
#else
    (void)dev;
    return {host[2 * i], host[2 * i + 1]};
#endif
}
#ifdef __CUDA_ARCH__
#define DSVD_TAB(name) nullptr, ddc::name##D
#else
#define DSVD_TAB(name) ddc::name##H, nullptr
#endif

// log(u) for finite u > 0, correctly rounded (ties to even) up to the
// ~2^-104 accuracy of the double-double evaluation. Table-driven: f = c (1+t)
// with c = i/64 the nearest table point, log c from a double-double table, and
// log(f/c) = 2 atanh(z), z = (f-c)/(f+c), |z| <= 2^-7.5, so the series needs
// three double-double Horner steps plus a plain-double tail (the w^4 .. w^7
// terms, below 2^-60 relative, whose rounding stays under 2^-113). Same value as
// log_cr_series (the 23-term reference evaluation) except with probability
// ~2^-50 per draw; tests/test_ddm.py checks both against each other.
__host__ __device__ inline double log_cr(double u) {
    int e;
    double f = frexp(u, &e);  // u = f * 2^e, f in [0.5, 1)
    if (f < 0.70710678118654752440) {
        f *= 2.0;
        e -= 1;
    }
    const int i = static_cast<int>(rint(f * 64.0));  // 45 .. 91
    const double c = i * 0.015625;
    const dd z = div(dd{f - c, 0.0}, two_sum(f, c));  // f - c exact (Sterbenz)
    const dd w = mul(z, z);
    const double wh = w.hi;
    const double tail = ddc::kAtanhHi(4) + wh * (ddc::kAtanhHi(5) + wh * (ddc::kAtanhHi(6) + wh * ddc::kAtanhHi(7)));
    dd p = add(dd{ddc::kAtanhHi(3), ddc::kAtanhLo(3)}, mul_d(w, tail));
    p = add(dd{ddc::kAtanhHi(2), ddc::kAtanhLo(2)}, mul(w, p));
    p = add(dd{ddc::kAtanhHi(1), ddc::kAtanhLo(1)}, mul(w, p));
    p = add(dd{1.0, 0.0}, mul(w, p));
    const dd lg = mul(mul_d(z, 2.0), p);
    const double ed = static_cast<double>(e);
    dd el = add(dd{ed * ddc::kLn2Hi, 0.0}, two_prod(ed, ddc::kLn2Mid));
    el = add(el, dd{ed * ddc::kLn2Lo, 0.0});
    const dd lc = tab_ld(DSVD_TAB(kLogCTab), i - ddc::kLogCFirst);
    const dd r = add(add(el, lc), lg);
    return r.hi + r.lo;
}

// cos(x) for 0 <= x <= 8, correctly rounded (same caveat as log_cr).
// Table-driven: x = k pi/2 + r, r = a + s with a = j/32, |s| <= 1/64, and
// cos/sin(a + s) from double-double cos a, sin a and short cos s, sin s series
// (three double-double Horner steps each, plain-double tails).
__host__ __device__ inline double cos_cr(double x) {
    const double kq = rint(x * ddc::kTwoOverPi);
    const int k = static_cast<int>(kq);
    dd r = two_sum(x, -kq * ddc::kPio2_1);
    r = add(r, dd{-kq * ddc::kPio2_2, 0.0});
    r = add(r, dd{-kq * ddc::kPio2_3, 0.0});
    r = add(r, two_prod(-kq, ddc::kPio2_4));
    const int j = static_cast<int>(rint(r.hi * 32.0));  // -25 .. 25
    const int ja = j < 0 ? -j : j;
    const dd s = two_sum(r.hi - j * 0.03125, r.lo);     // r.hi - j/32 exact (Sterbenz)
    const dd w = mul(s, s);
    const double wh = w.hi;
    // cos s = 1 + w (c1 + w (c2 + w (c3 + w tail_c)))
    const double tc = ddc::kCosHi(4) + wh * (ddc::kCosHi(5) + wh * ddc::kCosHi(6));
    dd pc = add(dd{ddc::kCosHi(3), ddc::kCosLo(3)}, mul_d(w, tc));
    pc = add(dd{ddc::kCosHi(2), ddc::kCosLo(2)}, mul(w, pc));
    pc = add(dd{ddc::kCosHi(1), ddc::kCosLo(1)}, mul(w, pc));
    const dd cs = add(dd{1.0, 0.0}, mul(w, pc));
    // sin s = s (1 + w (d1 + w (d2 + w (d3 + w tail_s))))
    const double ts = ddc::kSinHi(4) + wh * (ddc::kSinHi(5) + wh * ddc::kSinHi(6));
    dd ps = add(dd{ddc::kSinHi(3), ddc::kSinLo(3)}, mul_d(w, ts));
    ps = add(dd{ddc::kSinHi(2), ddc::kSinLo(2)}, mul(w, ps));
    ps = add(dd{ddc::kSinHi(1), ddc::kSinLo(1)}, mul(w, ps));
    const dd sn = mul(s, add(dd{1.0, 0.0}, mul(w, ps)));
    dd res;
    if (ja == 0) {
        res = (k & 1) == 0 ? cs : sn;
    } else {
        const dd ca = tab_ld(DSVD_TAB(kCosTab), ja);
        dd sa = tab_ld(DSVD_TAB(kSinTab), ja);
        if (j < 0) sa = dd{-sa.hi, -sa.lo};
        if ((k & 1) == 0) {
            res = add(mul(ca, cs), mul(dd{-sa.hi, -sa.lo}, sn));  // cos(a+s)
        } else {
            res = add(mul(sa, cs), mul(ca, sn));  // sin(a+s)
        }
    }
    const int q = k & 3;
    const double v = res.hi + res.lo;
    return (q == 1 || q == 2) ? -v : v;
}

// ---- fast paths (Ziv's strategy) ------------------------------------------------
// Mostly-double evaluations returning a double-double estimate R = Rh + Rl with a
// proven absolute error bound err; the correctly rounded value is Rh whenever the
// whole interval [R - err, R + err] rounds to Rh, which the test below decides
// (Rh = fl(Rh + Rl) after the final renormalisation, so only the side of Rl can
// cross a rounding boundary; err is doubled to cover the rounding of Rl + err).
// Otherwise the caller evaluates log_cr / cos_cr above. ~5x fewer FP64
// operations than the double-double evaluations; tests/ddm_check.cpp checks
// fast-or-fallback against the series versions bit for bit.
__host__ __device__ __forceinline__ bool ziv_rounds(dd r, double err) {
    const double t = r.lo + copysign(2.0 * err, r.lo);
    return r.hi + t == r.hi;
}

__host__ __device__ __forceinline__ double tab1(const double* host, const double* dev, int i) {
#ifdef __CUDA_ARCH__
    (void)host;
    return __ldg(dev + i);
#else
    (void)dev;
    return host[i];
#endif
}

// log(u), u > 0 finite: u = f 2^e with f in [sqrt(1/2), sqrt(2)); r = 8-bit
// reciprocal of the 1/256-cell of f, so z = f r - 1 is exact (one FMA) with
// |z| < 2^-7; log u = e ln2 - log r + log1p(z), log1p(z) = z - z^2/2 + z^3 P(z)
// with z^2 exact (two_prod) and P to z^8 (truncation < 2^-87). Error: the z^3 P
// term's roundings (< 2^-53 |z|^3) plus the double-double sums (< 2^-100 of the
// parts' magnitudes); err below carries a 4x and 16x margin on those.
__host__ __device__ inline bool log_fast(double u, double* out) {
    int e;
    double f = frexp(u, &e);
    if (f < 0.70710678118654752440) {
        f *= 2.0;
        e -= 1;
    }
    const int i = static_cast<int>(rint(f * 256.0)) - ddc::kRcpFirst;  // 0 .. 181
    const double r = tab1(DSVD_TAB(kRcpLogTab), 3 * i);
    const dd lr{tab1(DSVD_TAB(kRcpLogTab), 3 * i + 1), tab1(DSVD_TAB(kRcpLogTab), 3 * i + 2)};
    const double z = fma(f, r, -1.0);  // exact
    const dd z2 = two_prod(z, z);
    const double p = 0x1.5555555555555p-2 + z * (-0.25 + z * (0.2 + z * (-0x1.5555555555555p-3 +
                     z * (0x1.2492492492492p-3 + z * (-0.125 + z * (0x1.c71c71c71c71cp-4 +
                     z * (-0.1 + z * 0x1.745d1745d1746p-4)))))));
    const double z3p = z2.hi * z * p;
    dd y = two_sum(z, -0.5 * z2.hi);
    const double ed = static_cast<double>(e);
    y.lo += fma(ed, ddc::kLn2Lo, -0.5 * z2.lo) + z3p;
    y = quick_two_sum(y.hi, y.lo);
    const dd el{ed * ddc::kLn2Hi, ed * ddc::kLn2Mid};  // both exact (42-bit pieces, |e| <= 1075)
    const dd res = add(add(el, lr), y);
    const double err = 0x1p-51 * fabs(z2.hi * z) + 0x1p-96 * (fabs(el.hi) + fabs(lr.hi) + fabs(y.hi));
    *out = res.hi;
    return ziv_rounds(res, err);
}

// cos(x), 0 <= x <= 8: x = k pi/2 + r (three exact Cody-Waite steps, the fourth
// piece and the third's product added to the low word: |error of r| < 2^-104),
// r = j/32 + s with |s| <= 1/64, cos/sin(j/32) from the double-double tables,
// cos s - 1 = -s^2/2 (exact) + s^4 (..), sin s = s + s^3 (..), combined in
// double-double. Error < 2^-72 absolute (the s^3 terms' roundings) + the
// reduction's 2^-104; for k odd and j = 0 the result is sin s itself and the
// polynomial error is relative to s.
__host__ __device__ inline bool cos_fast(double x, double* out) {
    const double kq = rint(x * ddc::kTwoOverPi);
    const int k = static_cast<int>(kq);
    const double r1 = fma(-kq, ddc::kPio2_1, x);  // exact (Sterbenz; kq * P1 exact)
    dd r = two_sum(r1, -kq * ddc::kPio2_2);         // kq * P2 exact
    r.lo = fma(-kq, ddc::kPio2_4, fma(-kq, ddc::kPio2_3, r.lo));
    r = two_sum(r.hi, r.lo);
    const int j = static_cast<int>(rint(r.hi * 32.0));  // -25 .. 25
    const dd s = two_sum(r.hi - j * 0.03125, r.lo);     // r.hi - j/32 exact (Sterbenz)
    const dd p = two_prod(s.hi, s.hi);
    const double s2 = p.hi;
    // cos s - 1 = cm.hi + cm.lo
    const dd cm{-0.5 * p.hi, fma(-s.hi, s.lo, -0.5 * p.lo) +
                                 s2 * s2 * (0x1.5555555555555p-5 + s2 * (-0x1.6c16c16c16c17p-10 +
                                                                         s2 * 0x1.a01a01a01a01ap-16))};
    // sin s = s.hi + sn_lo
    const double sn_lo = s.lo + s.hi * s2 * (-0x1.5555555555555p-3 + s2 * (0x1.1111111111111p-7 +
                                             s2 * (-0x1.a01a01a01a01ap-13 + s2 * 0x1.71de3a556c734p-19)));
    dd res;
    double err;
    if (j == 0) {
        if ((k & 1) == 0) {
            res = quick_two_sum(1.0, cm.hi);
            res = quick_two_sum(res.hi, res.lo + cm.lo);
            err = 0x1p-78;
        } else {  // sin s: the s^3 term's roundings, relative to s^3
            res = quick_two_sum(s.hi, sn_lo);
            err = 0x1p-50 * fabs(s.hi) * s2;
        }
    } else {
        const int ja = j < 0 ? -j : j;
        const dd ca = tab_ld(DSVD_TAB(kCosTab), ja);
        dd sa = tab_ld(DSVD_TAB(kSinTab), ja);
        if (j < 0) sa = dd{-sa.hi, -sa.lo};
        // cos s = 1 + cm, sin s = s.hi + sn_lo
        if ((k & 1) == 0) {  // cos(a + s) = ca + ca cm - sa sin s
            dd t2 = two_prod(ca.hi, cm.hi);
            t2.lo += ca.hi * cm.lo + ca.lo * cm.hi;
            dd t3 = two_prod(-sa.hi, s.hi);
            t3.lo += -sa.hi * sn_lo - sa.lo * s.hi;
            res = add(add(ca, t2), t3);
        } else {  // sin(a + s) = sa + sa cm + ca sin s
            dd t2 = two_prod(sa.hi, cm.hi);
            t2.lo += sa.hi * cm.lo + sa.lo * cm.hi;
            dd t3 = two_prod(ca.hi, s.hi);
            t3.lo += ca.hi * sn_lo + ca.lo * s.hi;
            res = add(add(sa, t2), t3);
        }
        err = 0x1p-68;  // the s^3 term of sin s: < 2^-70.4
    }
    const int q = k & 3;
    const bool neg = q == 1 || q == 2;
    *out = neg ? -res.hi : res.hi;
    return ziv_rounds(res, err + 0x1p-102);
}

// The series evaluations the table-driven versions above replace (kept as the
// cross-check of tests/test_ddm.py).
__host__ __device__ inline double log_cr_series(double u) {
    int e;
    double f = frexp(u, &e);  // u = f * 2^e, f in [0.5, 1)
    if (f < 0.70710678118654752440) {
        f *= 2.0;
        e -= 1;
    }
    // log(f) = 2 atanh(z), z = (f - 1) / (f + 1); f - 1 is exact (Sterbenz)
    const dd z = div(dd{f - 1.0, 0.0}, two_sum(f, 1.0));
    const dd w = mul(z, z);
    constexpr int K = 23;  // |z| <= 0.1716: w^23/47 < 2^-118
    dd p{ddc::kAtanhHi(K - 1), ddc::kAtanhLo(K - 1)};
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int k = K - 2; k >= 0; --k) p = add(mul(p, w), dd{ddc::kAtanhHi(k), ddc::kAtanhLo(k)});
    dd lg = mul(mul_d(z, 2.0), p);
    const double ed = static_cast<double>(e);
    // e*ln2: hi part exact (42-bit ln2_hi), mid part as an exact product
    dd el = add(dd{ed * ddc::kLn2Hi, 0.0}, two_prod(ed, ddc::kLn2Mid));
    el = add(el, dd{ed * ddc::kLn2Lo, 0.0});
    const dd r = add(el, lg);
    return r.hi + r.lo;
}

__host__ __device__ inline double cos_cr_series(double x) {
    const double kq = rint(x * ddc::kTwoOverPi);
    const int k = static_cast<int>(kq);
    // r = x - kq*pi/2 with pi/2 in four pieces (kq*piece_i exact for the first three)
    dd r = two_sum(x, -kq * ddc::kPio2_1);
    r = add(r, dd{-kq * ddc::kPio2_2, 0.0});
    r = add(r, dd{-kq * ddc::kPio2_3, 0.0});
    r = add(r, two_prod(-kq, ddc::kPio2_4));
    const dd w = mul(r, r);
    constexpr int J = 16;  // |r| <= pi/4: w^15/30! < 2^-118
    dd res;
    if ((k & 1) == 0) {
        dd c{ddc::kCosHi(J - 1), ddc::kCosLo(J - 1)};
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
        for (int j = J - 2; j >= 0; --j) c = add(mul(c, w), dd{ddc::kCosHi(j), ddc::kCosLo(j)});
        res = c;
    } else {
        dd s{ddc::kSinHi(J - 1), ddc::kSinLo(J - 1)};
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
        for (int j = J - 2; j >= 0; --j) s = add(mul(s, w), dd{ddc::kSinHi(j), ddc::kSinLo(j)});
        res = mul(s, r);
    }
    const int q = k & 3;
    const double v = res.hi + res.lo;
    return (q == 1 || q == 2) ? -v : v;
}

}  // namespace ddm
}  // namespace dsvd
