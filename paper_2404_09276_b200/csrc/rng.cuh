// Counter-based SplitMix64 stream and Box-Muller normals, the generator the
// reference seeds Omega with (random.cpp:8-27). The integer part is exact;
// log and cos are correctly rounded (dd_math.cuh). glibc's log/cos misround in
// ~0.1% of draws (verified against 60-digit decimal arithmetic), so
// those draws differ from the reference by one ulp; callers that need the
// reference's exact bits can pass their own sketch.
#pragma once

#include <cstdint>

#include "dd_math.cuh"

namespace dsvd {

__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ double unit_open(uint64_t x) {
    return (static_cast<double>(x >> 11) + 0.5) * 0x1p-53;
}

// the double-double evaluations, out of line: taken by ~1 lane in 3,000
static __device__ __noinline__ double log_slow(double u) { return ddm::log_cr(u); }
static __device__ __noinline__ double cos_slow(double x) { return ddm::cos_cr(x); }

__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t i) {
    const double u1 = unit_open(splitmix64_at(seed, 2 * i));
    const double u2 = unit_open(splitmix64_at(seed, 2 * i + 1));
    // 2*pi rounded to double, times u2: the same two roundings as
    // `2.0 * std::numbers::pi * u2` (constant-folded) in the reference.
    const double x = 6.283185307179586 * u2;
    double lg, cs;
    // fast evaluations; the double-double ones only where they cannot decide the rounding
    if (!ddm::log_fast(u1, &lg)) lg = log_slow(u1);
    if (!ddm::cos_fast(x, &cs)) cs = cos_slow(x);
    return sqrt(-2.0 * lg) * cs;
}

}  // namespace dsvd
