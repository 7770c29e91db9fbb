// Engine internals shared by the C ABI translation units (engine.cu,
// abi_inputs.cu, abi_metrics.cu).
#pragma once

#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "sparse.cuh"

namespace dsvd {

void set_device(dsvd_ctx* ctx);
void count_launch(int n = 1);
// host <-> device copies that stage pageable host buffers through pinned slots
// (engine.cu); pinned / registered / device pointers take one cudaMemcpyAsync
bool host_is_pageable(const void* p);
void copy_d2h(dsvd_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t producer,
              cudaEvent_t ready = nullptr);
void copy_h2d(dsvd_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);
// page-in of pageable host outputs on a host thread during the solve (joined by
// copy_d2h and, on every exit path, by PrefaultScope)
void prefault_outputs(dsvd_ctx* ctx, const dsvd_outputs* out, int64_t rows, int64_t cols, int64_t k);
void prefault_join(dsvd_ctx* ctx) noexcept;
struct PrefaultScope {
    dsvd_ctx* ctx;
    ~PrefaultScope() { prefault_join(ctx); }
};

struct CsrAlloc {
    // allocate through the context arena (prefix) or as owned buffers
    dsvd_ctx* ctx;
    std::string prefix;
    std::vector<void*>* owned;
    void* get(const std::string& name, size_t bytes) {
        if (owned) {
            void* p = nullptr;
            DSVD_CUDA_CHECK(cudaMalloc(&p, bytes > 0 ? bytes : 1));
            owned->push_back(p);
            return p;
        }
        return ctx->buf(prefix + name, bytes);
    }
};

// CSR(A) and its transpose on the device from device arrays (int64 offsets and
// indices, fp64 values); copy_inputs makes owned copies of off/val.
void build_pair(dsvd_ctx* ctx, CsrAlloc& al, int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_off,
                const int64_t* d_idx64, const double* d_val, DevCsr& a, DevCsr& at, bool copy_inputs,
                cudaEvent_t values_ready = nullptr);
// The same from host arrays (values copied on ctx->copy beside the CSC build).
// omega_cfg: also start the solve's sketch on the side stream once the offsets
// are on the device (pregenerate_omega).
void upload_pair(dsvd_ctx* ctx, CsrAlloc& al, int64_t rows, int64_t cols, int64_t nnz, const int64_t* off,
                 const int64_t* idx, const double* val, DevCsr& a, DevCsr& at,
                 const dsvd_config* omega_cfg = nullptr);
// Starts the sketch Omega of a solve of an rows x cols matrix on the side stream
// (the next solve_tall with the same shape / seed waits on it instead).
void pregenerate_omega(dsvd_ctx* ctx, int64_t rows, int64_t cols, const dsvd_config& cfg,
                       const int64_t* d_off = nullptr);

// Partial rows of the split chunks (spmm's `partial` argument) in the context arena.
inline double* partial_for(dsvd_ctx* ctx, const DevCsr& a, int64_t ld) {
    if (a.nchunks == 0) return nullptr;
    return ctx->tbuf<double>("spmm.partial", a.nchunks * ld);
}

// Run `f` with the boundary contract: Failure -> status code + message.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return DSVD_OK;
    } catch (const Failure& e) {
        set_error(e.what(), e.index);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed", -1);
        return DSVD_OOM;
    } catch (const std::exception& e) {
        set_error(e.what(), -1);
        return DSVD_OTHER;
    }
}

}  // namespace dsvd
