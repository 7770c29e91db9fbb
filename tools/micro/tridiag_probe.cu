// Per-step phase clocks of tbi_tridiag_kernel on one 150 x 150 Gram matrix:
//   nvcc ... -DDSVD_TRID_PROBE tridiag_probe.cu  (includes the kernel source)
#define DSVD_TRID_PROBE
#include "../../paper_2404_09276_b200/csrc/eig_tbi.cu"

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 150, rows = 4 * n;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> b(static_cast<size_t>(rows) * n), g(static_cast<size_t>(n) * n, 0.0);
    for (auto& x : b) x = nd(rng);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int r = 0; r < rows; ++r) s += b[r * n + i] * b[r * n + j] * (1.0 + 10.0 * (i == j) * i);
            g[i * n + j] = s;
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) g[i * n + j] = g[j * n + i];
    double *dg, *d, *e, *hv, *tau;
    cudaMalloc(&dg, sizeof(double) * n * n);
    cudaMalloc(&d, sizeof(double) * n);
    cudaMalloc(&e, sizeof(double) * n);
    cudaMalloc(&hv, sizeof(double) * n * n);
    cudaMalloc(&tau, sizeof(double) * n);
    cudaMemcpy(dg, g.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    const size_t s1 = dsvd::tridiag_smem_bytes(n);
    cudaFuncSetAttribute(dsvd::tbi_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s1));
    cudaEvent_t a0, a1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a0);
        dsvd::tbi_tridiag_kernel<<<1, dsvd::kTridThreads, s1>>>(dg, n, d, e, hv, tau, nullptr, nullptr);
        cudaEventRecord(a1);
        cudaEventSynchronize(a1);
        cudaEventElapsedTime(&ms, a0, a1);
    }
    printf("n %d: %.1f us (%s)\n", n, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    long long pr[192][4];
    cudaMemcpyFromSymbol(pr, dsvd::g_trid_probe, sizeof(pr));
    long long sb = 0, sc1 = 0, sc2 = 0, sw = 0;
    for (int k = 0; k + 2 < n; ++k) {
        const long long b_ = pr[k][1] - pr[k][0], c1 = pr[k][2] - pr[k][1];
        const long long next = (k + 3 < n) ? pr[k + 1][0] : pr[k][2];
        const long long c2 = next - pr[k][2], w0 = pr[k][3] - pr[k][0];
        sb += b_;
        sc1 += c1;
        sc2 += c2;
        sw += w0;
        if (k % 16 == 0 || k + 3 == n)
            printf("step %3d (m=%3d): B (reflector | matvec) %6lld  C1 %6lld  C2 update %6lld  (reflector %6lld) cycles\n",
                   k, n - k - 1, b_, c1, c2, w0);
    }
    printf("sum: B %lld  C1 %lld  C2 %lld  reflector %lld cycles\n", sb, sc1, sc2, sw);
    return 0;
}
