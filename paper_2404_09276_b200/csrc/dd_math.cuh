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

// log(u) for finite u > 0, correctly rounded (ties to even) up to the
// ~2^-104 accuracy of the double-double evaluation.
__host__ __device__ inline double log_cr(double u) {
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
#pragma unroll
    for (int k = K - 2; k >= 0; --k) p = add(mul(p, w), dd{ddc::kAtanhHi(k), ddc::kAtanhLo(k)});
    dd lg = mul(mul_d(z, 2.0), p);
    const double ed = static_cast<double>(e);
    // e*ln2: hi part exact (42-bit ln2_hi), mid part as an exact product
    dd el = add(dd{ed * ddc::kLn2Hi, 0.0}, two_prod(ed, ddc::kLn2Mid));
    el = add(el, dd{ed * ddc::kLn2Lo, 0.0});
    const dd r = add(el, lg);
    return r.hi + r.lo;
}

// cos(x) for 0 <= x <= 8, correctly rounded (same caveat as log_cr).
__host__ __device__ inline double cos_cr(double x) {
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
#pragma unroll
        for (int j = J - 2; j >= 0; --j) c = add(mul(c, w), dd{ddc::kCosHi(j), ddc::kCosLo(j)});
        res = c;
    } else {
        dd s{ddc::kSinHi(J - 1), ddc::kSinLo(J - 1)};
#pragma unroll
        for (int j = J - 2; j >= 0; --j) s = add(mul(s, w), dd{ddc::kSinHi(j), ddc::kSinLo(j)});
        res = mul(s, r);
    }
    const int q = k & 3;
    const double v = res.hi + res.lo;
    return (q == 1 || q == 2) ? -v : v;
}

}  // namespace ddm
}  // namespace dsvd
