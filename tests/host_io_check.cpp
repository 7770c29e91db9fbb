// CPU check of the host side of the staged copies (csrc/host_io.cpp): the
// threaded streaming copy against memcmp over odd alignments, sizes and thread
// counts (bytes around the destination untouched), and the page-in helper.
#include <cstdio>
#include <cstring>
#include <vector>

namespace dsvd {
void host_parallel_memcpy(void*, const void*, size_t, int);
void host_prefault(void*, size_t, int);
}

int main() {
    std::vector<char> a((40 << 20) + 64), b((40 << 20) + 8192);
    for (size_t i = 0; i < a.size(); ++i) a[i] = static_cast<char>(i * 131 + 7);
    long bad = 0, cases = 0;
    const size_t offs[] = {0, 1, 7, 31, 33, 4095};
    const size_t sizes[] = {0, 5, 255, 300, 4096 + 17, (size_t(3) << 20) + 13, (size_t(33) << 20) + 5};
    const int threads[] = {1, 3, 16};
    for (size_t off : offs)
        for (size_t n : sizes)
            for (int t : threads) {
                std::memset(b.data(), 0, b.size());
                dsvd::host_parallel_memcpy(b.data() + off, a.data() + 3, n, t);
                ++cases;
                if (std::memcmp(b.data() + off, a.data() + 3, n) != 0) ++bad;
                for (size_t i = 0; i < off; ++i) bad += b[i] != 0;
                bad += b[off + n] != 0;
            }
    std::vector<char> p(size_t(5) << 20, 1);
    dsvd::host_prefault(p.data() + 3, p.size() - 3, 4);
    for (size_t i = 3; i < p.size(); ++i)
        if (p[i] != ((i - 3) % 4096 == 0 ? 0 : 1)) ++bad;
    std::printf("cases %ld bad %ld\n", cases, bad);
    return bad != 0;
}
