// Host side of the staged host<->device copies (engine.cu `stage_d2h` /
// `stage_h2d`): a byte copy between a pinned staging slot and the caller's
// pageable buffer, split over host threads. The caller's buffer is often
// freshly allocated (std::vector / numpy outputs of the reference-shaped API),
// so this copy also takes its first-touch page faults — in parallel.
#include <cstdint>
#include <cstring>

#include <immintrin.h>
#include <omp.h>

namespace dsvd {
namespace {

// memcpy with non-temporal 32-byte stores: the destination (the caller's
// output array, or a pinned slot the copy engine reads next) is not read back
// by this thread, so the stores skip the read-for-ownership and the caches
__attribute__((target("avx2"))) void copy_stream_avx2(char* dst, const char* src, size_t n) {
    const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
    if (n < head + 256) {
        std::memcpy(dst, src, n);
        return;
    }
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
    }
    _mm_sfence();
    if (i < n) std::memcpy(dst + i, src + i, n - i);
}

void copy_slice(char* dst, const char* src, size_t n) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2) copy_stream_avx2(dst, src, n);
    else std::memcpy(dst, src, n);
}

}  // namespace

void host_parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
    constexpr size_t kMinPerThread = size_t(1) << 20;
    int t = threads < 1 ? 1 : threads;
    if (bytes / kMinPerThread < static_cast<size_t>(t)) t = static_cast<int>(bytes / kMinPerThread);
    if (t <= 1) {
        copy_slice(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
        return;
    }
    // 4 KB-aligned slices (whole pages per thread)
    const size_t per = ((bytes + t - 1) / t + 4095) & ~size_t(4095);
#pragma omp parallel num_threads(t)
    {
        const size_t b = static_cast<size_t>(omp_get_thread_num()) * per;
        if (b < bytes) {
            const size_t n = bytes - b < per ? bytes - b : per;
            copy_slice(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, n);
        }
    }
}

// Writes one zero byte per 4 KB page of [p, p + bytes): the pages of a fresh
// output array are faulted in (and zeroed by the kernel) here, on a host thread
// while the solve runs on the device, instead of inside the staged copies at
// the end of the solve.
void host_prefault(void* p, size_t bytes, int threads) {
    volatile char* c = static_cast<volatile char*>(p);
    const int64_t pages = static_cast<int64_t>((bytes + 4095) / 4096);
#pragma omp parallel for num_threads(threads < 1 ? 1 : threads) schedule(static)
    for (int64_t i = 0; i < pages; ++i) c[i * 4096] = 0;
}

}  // namespace dsvd
