// Drop-in use of the B200 path from C++: the reference's API (namespace
// dashsvd, solver.hpp) through include/dashsvd_b200.hpp. Solves BASELINE.json
// configs[0] (sparse_random(10000, 5000, 25, seed 0, row decay), shifted, k=50,
// s=25, p=10) and prints the leading singular values.
//   g++ -std=c++17 -O2 -I include examples/cpp_solve.cpp
//       -L paper_2404_09276_b200/_lib -ldashsvd_b200 -Wl,-rpath,$PWD/paper_2404_09276_b200/_lib
#include <cstdio>

#include "dashsvd_b200.hpp"

int main() {
    dashsvd::SparseMatrix a;
    a.rows = 10000;
    a.cols = 5000;
    int64_t nnz = 0;
    dashsvd::b200::check(dsvd_synth_sparse_random(a.rows, a.cols, 25, 0, 1, &nnz));
    a.offsets.resize(a.rows + 1);
    a.col_indices.resize(nnz);
    a.values.resize(nnz);
    dsvd_synth_fetch(a.offsets.data(), a.col_indices.data(), a.values.data());

    dashsvd::SolverConfig cfg;
    cfg.k = 50;
    cfg.s = 25;
    cfg.p = 10;
    cfg.alg = dashsvd::Algorithm::shifted;
    try {
        dashsvd::SolveResult r = dashsvd::solve(a, cfg);
        std::printf("nnz=%lld iterations=%lld sigma_1=%.17g sigma_50=%.17g alpha_10=%.17g\n",
                    static_cast<long long>(nnz), static_cast<long long>(r.trace.iterations),
                    r.svd.s[0], r.svd.s[49], r.trace.alphas[9]);
    } catch (const dashsvd::Error& e) {
        std::fprintf(stderr, "dashsvd error: %s\n", e.what());
        return 2;
    }
    return 0;
}
