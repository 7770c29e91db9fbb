// Host copy rates behind the staged pageable transfers (engine.cu copy_d2h /
// copy_h2d): 32 MB slices from a pinned-like source into (a) warm and (b) fresh
// (first-touch) destination pages, glibc memcpy vs host_io.cpp's streaming copy.
//   g++-13 -O2 -fopenmp -std=c++17 paper_2404_09276_b200/csrc/host_io.cpp tools/micro/host_copy.cpp
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>

#include <omp.h>

namespace dsvd {
void host_parallel_memcpy(void*, const void*, size_t, int);
}

static void glibc_parallel(void* dst, const void* src, size_t bytes, int t) {
    const size_t per = ((bytes + t - 1) / t + 4095) & ~size_t(4095);
#pragma omp parallel num_threads(t)
    {
        const size_t b = size_t(omp_get_thread_num()) * per;
        if (b < bytes) std::memcpy((char*)dst + b, (const char*)src + b, bytes - b < per ? bytes - b : per);
    }
}

int main() {
    const size_t N = size_t(4) << 30, chunk = size_t(32) << 20;
    char* src = (char*)aligned_alloc(4096, N);
    std::memset(src, 1, N);
    for (int fresh = 0; fresh < 2; ++fresh)
        for (int kind = 0; kind < 2; ++kind)
            for (int t : {4, 8, 16}) {
                char* dst = (char*)mmap(nullptr, N, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
                madvise(dst, N, MADV_HUGEPAGE);
                if (!fresh) std::memset(dst, 0, N);
                auto t0 = std::chrono::steady_clock::now();
                for (size_t c = 0; c < N; c += chunk) {
                    if (kind) dsvd::host_parallel_memcpy(dst + c, src + c, chunk, t);
                    else glibc_parallel(dst + c, src + c, chunk, t);
                }
                const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                printf("%s dst, %s, %2d threads: %.1f GB/s\n", fresh ? "fresh" : "warm ", kind ? "stream" : "glibc ", t,
                       N / s / 1e9);
                munmap(dst, N);
            }
}
