// Shared helpers for the sm_100a dashSVD kernels and the engine.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/dashsvd_b200.h"

namespace dsvd {

// Error carried from the engine to the C ABI boundary, where it becomes a
// status code (dsvd_* functions never throw).
struct Failure : std::runtime_error {
    int code;
    long long index;
    Failure(int c, const std::string& msg, long long idx = -1)
        : std::runtime_error(msg), code(c), index(idx) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg, long long idx = -1) {
    throw Failure(code, msg, idx);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        const int code = (e == cudaErrorMemoryAllocation) ? DSVD_OOM : DSVD_CUDA;
        fail(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                       std::to_string(line) + ")");
    }
}

#define DSVD_CUDA_CHECK(x) ::dsvd::cuda_check((x), #x, __FILE__, __LINE__)
#define DSVD_LAUNCH_CHECK() ::dsvd::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

constexpr int kNumSMs = 148;

// Host-side NVTX range (nsys / ncu --nvtx timelines) around a phase of the solve.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Row stride of every tall-skinny device block (Omega, Q, Y, T): l rounded up
// to 4 doubles so each row starts on a 32-byte sector boundary and lanes can
// use 128-bit loads.
inline int64_t padded_ld(int64_t l) { return (l + 3) & ~int64_t(3); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Device-side control block of one solve (lives in device memory).
struct Control {
    double alpha;          // shift used by the next product (solver.cpp:88)
    double alpha_stored;   // alpha' of the stop rule (post-update alpha, :111-112)
    int64_t iteration;     // completed power iterations
    int64_t status_index;  // RankDeficient index
    int64_t total_sweeps;  // Jacobi sweeps summed over the solve
    int32_t stopped;       // loop kernels are skipped once set
    int32_t stop_pending;  // set by the stop rule; becomes `stopped` at the next iteration
    int32_t status;        // DSVD_OK or an error raised on the device
    int32_t eig_sweeps;    // sweeps of the last eigensolve
    int32_t status_src;    // 1: the status was raised by the QR orthonormalizer
};

#ifdef __CUDACC__
// Device-side bounds assertions of the checked build (-DDSVD_CHECKED; `make
// checked`): a violated invariant prints where and traps, failing the call with
// a CUDA error. Compiled out of the product build.
#ifdef DSVD_CHECKED
#define DSVD_DCHECK(cond)                                                                            \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("DSVD_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                     \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define DSVD_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

// Gate words (Control::stopped / stop_pending) can be set by a kernel on
// another stream while the reading kernel runs: read them at L2, not through
// the non-coherent read-only path, so late blocks see a stop and skip.
__device__ __forceinline__ bool gate_closed(const int32_t* gate) {
    if (gate == nullptr) return false;
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(gate));
    return v != 0;
}
#endif

}  // namespace dsvd
