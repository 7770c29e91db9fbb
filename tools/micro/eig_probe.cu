// Per-eigenvalue phase clocks of tbi_eig_kernel (multisection, cluster check,
// LU, inverse-iteration solves) on a 150 x 150 Gram-like matrix.
#define DSVD_EIG_PROBE
#include "../../paper_2404_09276_b200/csrc/eig_tbi.cu"

#include <cstdio>
#include <random>
#include <vector>
#include <algorithm>

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 150, rows = 4 * n;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> b(static_cast<size_t>(rows) * n), g(static_cast<size_t>(n) * n, 0.0);
    for (auto& x : b) x = nd(rng);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int r = 0; r < rows; ++r) s += b[r * n + i] * b[r * n + j];
            g[i * n + j] = g[j * n + i] = s * (1.0 + 1e3 * (i == j) * i * i);
        }
    double *dg, *ws, *lam, *vecs;
    int32_t* flag;
    cudaMalloc(&dg, sizeof(double) * n * n);
    cudaMalloc(&ws, dsvd::tbi_workspace_bytes(n));
    cudaMalloc(&lam, sizeof(double) * n);
    cudaMalloc(&vecs, sizeof(double) * n * n);
    cudaMalloc(&flag, 4);
    cudaMemcpy(dg, g.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    dsvd::EigWorkspace w;
    w.l = n;
    w.lp = n;
    w.lam = lam;
    w.vecs = vecs;
    for (int rep = 0; rep < 3; ++rep) dsvd::tbi_eig(dg, w, ws, flag, nullptr, 0);
    cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    long long pr[256][6];
    cudaMemcpyFromSymbol(pr, dsvd::g_eig_probe, sizeof(pr));
    double s[2] = {0, 0};
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < 2; ++k) s[k] += pr[j][k + 1] - pr[j][k];
    printf("avg cycles per eigenvalue: multisection %.0f  twisted-factorization vector %.0f\n", s[0] / n, s[1] / n);
    return 0;
}
