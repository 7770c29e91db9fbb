// Host side of the staged host<->device copies (engine.cu `stage_d2h` /
// `stage_h2d`): a byte copy between a pinned staging slot and the caller's
// pageable buffer, split over host threads. The caller's buffer is often
// freshly allocated (std::vector / numpy outputs of the reference-shaped API),
// so this copy also takes its first-touch page faults — in parallel.
#include <cstdint>
#include <cstring>

#include <omp.h>

namespace dsvd {

void host_parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
    constexpr size_t kMinPerThread = size_t(1) << 20;
    int t = threads < 1 ? 1 : threads;
    if (bytes / kMinPerThread < static_cast<size_t>(t)) t = static_cast<int>(bytes / kMinPerThread);
    if (t <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    // 4 KB-aligned slices (whole pages per thread)
    const size_t per = ((bytes + t - 1) / t + 4095) & ~size_t(4095);
#pragma omp parallel num_threads(t)
    {
        const size_t b = static_cast<size_t>(omp_get_thread_num()) * per;
        if (b < bytes) {
            const size_t n = bytes - b < per ? bytes - b : per;
            std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, n);
        }
    }
}

}  // namespace dsvd
