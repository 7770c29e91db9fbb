// l x l symmetric eigensolver (parallel cyclic Jacobi) and the eigSVD
// assembly that turns its output into (s, V, 1/s), plus the device-side
// shift update / PVE stop rule of the power loop.
#pragma once

#include "common.cuh"

namespace dsvd {

struct EigWorkspace {
    int l = 0, lp = 0;        // logical and padded (even) order
    int max_sweeps = 0;
    double* gbuf = nullptr;   // lp*lp, used when G does not fit in shared memory
    double2* rot_log = nullptr;  // max_sweeps * (lp-1) * lp/2 rotations
    double* lam = nullptr;    // lp eigenvalues (diagonal after convergence)
    double* vecs = nullptr;   // lp*lp eigenvectors, row-major: vecs[t*lp + j]
};
size_t eig_workspace_bytes(int l, int max_sweeps);
void eig_workspace_bind(EigWorkspace& w, int l, int max_sweeps, void* mem);

// Jacobi on the l x l matrix g (device, row-major == column-major) -> w.lam,
// w.vecs (unsorted). Sweep count goes to ctrl->eig_sweeps (and is added to
// ctrl->total_sweeps); non-convergence sets ctrl->status = DSVD_NUMERICAL.
// `need` (optional): the kernels only run when *need != 0 (the tridiagonal
// path's fallback flag).
void jacobi_eig(const double* g, EigWorkspace& w, Control* ctrl, const int32_t* gate,
                cudaStream_t stream, const int32_t* need = nullptr);

// Tridiagonal path (eig_tbi.cu): Householder + multisection + inverse
// iteration. Sets *clustered when eigenvalues are too close for inverse
// iteration; callers then run jacobi_eig with need = clustered.
bool tbi_supported(int l);
size_t tbi_workspace_bytes(int l);
// phase 0: the whole path; 1: the tridiagonalisation only (the one long,
// single-CTA kernel); 2: the rest (multisection .. back-transform)
void tbi_eig(const double* g, EigWorkspace& w, void* tbi_ws, int32_t* clustered, const int32_t* gate,
             cudaStream_t stream, int phase = 0);

// Loop-mode parameters of eig_svd_finish (solver.cpp:97-112).
struct LoopStep {
    int64_t k = 0;
    double tol = 0;
    int alg = 0;
    double* alphas = nullptr;   // trace, cap entries
    double* s_hat = nullptr;    // trace, cap x l
    int64_t cap = 0;
    double* s_stored = nullptr; // l
};

// eigSVD assembly (decompositions.cpp:52-73) from the Jacobi output:
// descending order, rank floor (rows = row count of the factored matrix),
// s = sqrt(lambda), W = V with the sign convention applied (l x ldw row-major),
// inv_s = 1/s. With `loop` non-null also records the trace, evaluates the PVE
// stop rule and updates the shift (solver.cpp:97-112) in ctrl.
void eig_svd_finish(const EigWorkspace& w, int64_t rows, double* W, int64_t ldw, double* s,
                    double* inv_s, Control* ctrl, const LoopStep* loop, const int32_t* gate,
                    cudaStream_t stream);

// sym_eig output convention (sym_eig.cpp:161-172): ascending stable order,
// column-major vectors.
void sym_eig_finish(const EigWorkspace& w, double* values, double* vectors_colmajor,
                    cudaStream_t stream);

// Basic-algorithm iteration without a spectrum (qr orthonormalizer): alphas[j-1]
// = 0 and ctrl->iteration = j.
void trace_basic_iteration(Control* ctrl, double* alphas, int64_t cap, cudaStream_t stream);

// ctrl->stopped = ctrl->stop_pending (first kernel of each loop iteration).
void loop_begin(Control* ctrl, cudaStream_t stream);
void control_init(Control* ctrl, double* s_stored, int l, cudaStream_t stream);

}  // namespace dsvd
