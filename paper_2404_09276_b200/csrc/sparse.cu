// Sparse kernels of the dashSVD power loop on sm_100a.
//
//  - spmm: Y = A X (and the fused shifted update T = A^T Y - alpha Q) over
//    row-major l-column fp64 blocks. Each output element is ONE fused
//    multiply-add chain over its row's nonzeros in CSR order starting from
//    0.0 — the exact operation order of the reference kernel
//    (sparse_matrix.cpp:74-83, which GCC contracts to vfmadd) and of
//    add_scaled (dense_kernels.cpp:128-136) — so results are bitwise equal to
//    the reference. Work items are (row, 64-column slab) pairs, one warp each,
//    rows taken longest-first so hub rows of power-law matrices start first.
//  - build_transpose: CSR(A^T) as a stable sort of the nonzeros by column
//    (the counting sort of sparse_matrix.cpp:35-55 is stable in row order),
//    bitwise equal to the reference.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <string>

#include "sparse.cuh"

namespace dsvd {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSlab = 64;  // doubles per warp work item: 32 lanes x double2

__device__ __forceinline__ double2 ld_x(const double* p) {
    return __ldg(reinterpret_cast<const double2*>(p));
}

// One warp = one (row, slab) item. Lanes own two adjacent columns each; the
// next batch's (index, value) pairs are fetched while the current batch's
// gathers run. Bulk throughput is bound by random 512-byte gathers
// (tools/micro/gather_bw.cu), hence the slab-major order below.
// kChunk: the item is a CSR range [chunk_p0, chunk_p1) of a split row and the
// result goes to row `rpos` of `partial` (no shift; added in the combine).
template <bool kShift, bool kChunk>
__global__ void __launch_bounds__(256)
spmm_bulk_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                 const double* __restrict__ val, const int32_t* __restrict__ order,
                 int64_t row_start, int64_t rows, int nslab, const double* __restrict__ x,
                 double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                 const double* __restrict__ alpha_p, const int32_t* __restrict__ gate,
                 const int64_t* __restrict__ chunk_p0, const int64_t* __restrict__ chunk_p1) {
    if (gate_closed(gate)) return;
    const int lane = threadIdx.x & 31;
    // slab-major order: all rows' first 64 columns, then the next 64, ... so
    // the X columns being gathered (rows x 512 B) stay resident in L2
    const int64_t nrows = rows - row_start;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (item >= nrows * nslab) return;
    const int slab = static_cast<int>(item / nrows);
    const int64_t rpos = row_start + item % nrows;
    int64_t row, beg, end;
    if (kChunk) {
        row = rpos;
        beg = chunk_p0[rpos];
        end = chunk_p1[rpos];
    } else {
        row = static_cast<int64_t>(order[rpos]);
        beg = off[row];
        end = off[row + 1];
    }
    const int64_t col = static_cast<int64_t>(slab) * kSlab + 2 * lane;
    const bool active = col < ld;  // ld is a multiple of 4, so col+1 < ld as well
    const double* xc = x + (active ? col : 0);

    double a0 = 0.0, a1 = 0.0;
    int c = 0;
    double v = 0.0;
    if (beg + lane < end) {
        c = __ldg(idx + beg + lane);
        v = __ldg(val + beg + lane);
    }
    for (int64_t p0 = beg; p0 < end; p0 += 32) {
        const int cnt = static_cast<int>(end - p0 < 32 ? end - p0 : 32);
        int cn = 0;
        double vn = 0.0;
        if (p0 + 32 + lane < end) {  // next batch's pairs, in flight during this one
            cn = __ldg(idx + p0 + 32 + lane);
            vn = __ldg(val + p0 + 32 + lane);
        }
        if (cnt == 32) {
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                const int cj = __shfl_sync(kFull, c, j);
                const double vj = __shfl_sync(kFull, v, j);
                if (active) {
                    const double2 xv = ld_x(xc + static_cast<int64_t>(cj) * ld);
                    a0 = fma(vj, xv.x, a0);
                    a1 = fma(vj, xv.y, a1);
                }
            }
        } else {
            for (int j = 0; j < cnt; ++j) {
                const int cj = __shfl_sync(kFull, c, j);
                const double vj = __shfl_sync(kFull, v, j);
                if (active) {
                    const double2 xv = ld_x(xc + static_cast<int64_t>(cj) * ld);
                    a0 = fma(vj, xv.x, a0);
                    a1 = fma(vj, xv.y, a1);
                }
            }
        }
        c = cn;
        v = vn;
    }
    if (!active) return;
    if (kChunk) {
        *reinterpret_cast<double2*>(y + rpos * ld + col) = make_double2(a0, a1);
        return;
    }
    if (kShift) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) {  // solver.cpp:94 skips the update when alpha == 0
            const double2 qv = *reinterpret_cast<const double2*>(q + row * ld + col);
            a0 = fma(-alpha, qv.x, a0);
            a1 = fma(-alpha, qv.y, a1);
        }
    }
    *reinterpret_cast<double2*>(y + row * ld + col) = make_double2(a0, a1);
}

// Whole-row variant of spmm_bulk_kernel for ld <= 192: one warp = one row
// (or chunk) and all its columns. Lane L owns columns [4L, 4L+4) (one
// 256-bit load per nonzero) and [128+2L, 128+2L+2) (a 128-bit load, lanes
// with 128+2L < ld). The batch's (value, index) pairs are staged in shared
// memory and read back with one broadcast LDS.128 per nonzero; gathers are
// issued U nonzeros ahead of their FMAs, which stay in CSR order (bitwise
// the same chains as the slab kernel). Per nonzero a warp issues ~10
// instructions for 8*ld bytes instead of ~8 per 512-byte slab. The kernel is
// bound by gathers in flight per SM: U = 2 at 64 registers (32 warps per SM;
// ptxas spills ~40 bytes outside the inner loop) measured fastest on C2
// (pass 1 bulk rows 1.11 ms; 24 warps: 1.17 ms; slab kernel: 1.56 ms).
constexpr int kRowWarps = 8;

__device__ __forceinline__ void ld256(const double* p, double (&r)[4]) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

template <bool kShift, bool kChunk, int U>
__global__ void __launch_bounds__(32 * kRowWarps, U == 2 ? 4 : (U == 4 ? 2 : 1))
spmm_row_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, const double* __restrict__ val,
                const int32_t* __restrict__ order, int64_t row_start, int64_t rows, const double* __restrict__ x,
                double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                const double* __restrict__ alpha_p, const int32_t* __restrict__ gate,
                const int64_t* __restrict__ chunk_p0, const int64_t* __restrict__ chunk_p1) {
    if (gate_closed(gate)) return;
    __shared__ __align__(16) double2 cv[kRowWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rpos = row_start + static_cast<int64_t>(blockIdx.x) * kRowWarps + warp;
    if (rpos >= rows) return;
    int64_t row, beg, end;
    if (kChunk) {
        row = rpos;
        beg = chunk_p0[rpos];
        end = chunk_p1[rpos];
    } else {
        row = static_cast<int64_t>(order[rpos]);
        beg = off[row];
        end = off[row + 1];
    }
    const bool act4 = 4 * lane < ld, act2 = 128 + 2 * lane < ld;
    const double* x4 = x + (act4 ? 4 * lane : 0);
    const double* x2 = x + (act2 ? 128 + 2 * lane : 0);
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int c = 0;
    double v = 0.0;
    if (beg + lane < end) {
        c = __ldg(idx + beg + lane);
        v = __ldg(val + beg + lane);
    }
    double2* slot = cv[warp];
    for (int64_t p0 = beg; p0 < end; p0 += 32) {
        const int cnt = static_cast<int>(end - p0 < 32 ? end - p0 : 32);
        __syncwarp();
        slot[lane] = make_double2(v, __longlong_as_double(static_cast<long long>(c)));
        __syncwarp();
        if (p0 + 32 + lane < end) {  // next batch, in flight during this one
            c = __ldg(idx + p0 + 32 + lane);
            v = __ldg(val + p0 + 32 + lane);
        }
        for (int j0 = 0; j0 < cnt; j0 += U) {
            double xa[U][4], xb[U][2], vj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u;
                vj[u] = 0.0;
                if (j < cnt) {
                    const double2 e = slot[j];
                    vj[u] = e.x;
                    const int64_t cj = __double_as_longlong(e.y);
                    if (act4) ld256(x4 + cj * ld, xa[u]);
                    if (act2) {
                        const double2 t = __ldg(reinterpret_cast<const double2*>(x2 + cj * ld));
                        xb[u][0] = t.x;
                        xb[u][1] = t.y;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (j0 + u < cnt) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) acc[t] = fma(vj[u], xa[u][t], acc[t]);
                    acc[4] = fma(vj[u], xb[u][0], acc[4]);
                    acc[5] = fma(vj[u], xb[u][1], acc[5]);
                }
            }
        }
    }
    double* yr = y + (kChunk ? rpos : row) * ld;
    if (kShift && !kChunk) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) {  // solver.cpp:94 skips the update when alpha == 0
            const double* qr = q + row * ld;
            if (act4) {
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[t] = fma(-alpha, qr[4 * lane + t], acc[t]);
            }
            if (act2) {
                acc[4] = fma(-alpha, qr[128 + 2 * lane], acc[4]);
                acc[5] = fma(-alpha, qr[128 + 2 * lane + 1], acc[5]);
            }
        }
    }
    if (act4) {
        *reinterpret_cast<double2*>(yr + 4 * lane) = make_double2(acc[0], acc[1]);
        *reinterpret_cast<double2*>(yr + 4 * lane + 2) = make_double2(acc[2], acc[3]);
    }
    if (act2) *reinterpret_cast<double2*>(yr + 128 + 2 * lane) = make_double2(acc[4], acc[5]);
}

// Whole-row kernel for 192 < ld <= 320 (C4's l = 300): lane L owns columns
// [8L, 8L+8) (two 256-bit loads per nonzero) and [256+2L, 256+2L+2) (a
// 128-bit load, lanes with 256+2L < ld). Same staging, lookahead (2) and
// CSR-order FMA chains as spmm_row_kernel, so the results are bitwise those of
// the slab kernel; one warp gathers the whole 2.4 KB row per nonzero instead
// of five 512-byte slabs, and A is read once instead of once per slab.
template <bool kShift, bool kChunk>
__global__ void __launch_bounds__(32 * kRowWarps, 2)
spmm_row_wide_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, const double* __restrict__ val,
                     const int32_t* __restrict__ order, int64_t row_start, int64_t rows, const double* __restrict__ x,
                     double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                     const double* __restrict__ alpha_p, const int32_t* __restrict__ gate,
                     const int64_t* __restrict__ chunk_p0, const int64_t* __restrict__ chunk_p1) {
    constexpr int U = 4;
    if (gate_closed(gate)) return;
    __shared__ __align__(16) double2 cv[kRowWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rpos = row_start + static_cast<int64_t>(blockIdx.x) * kRowWarps + warp;
    if (rpos >= rows) return;
    int64_t row, beg, end;
    if (kChunk) {
        row = rpos;
        beg = chunk_p0[rpos];
        end = chunk_p1[rpos];
    } else {
        row = static_cast<int64_t>(order[rpos]);
        beg = off[row];
        end = off[row + 1];
    }
    const bool act0 = 8 * lane < ld, act1 = 8 * lane + 4 < ld, act2 = 256 + 2 * lane < ld;
    const double* x0 = x + (act0 ? 8 * lane : 0);
    const double* x1 = x + (act1 ? 8 * lane + 4 : 0);
    const double* x2 = x + (act2 ? 256 + 2 * lane : 0);
    double acc[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int c = 0;
    double v = 0.0;
    if (beg + lane < end) {
        c = __ldg(idx + beg + lane);
        v = __ldg(val + beg + lane);
    }
    double2* slot = cv[warp];
    for (int64_t p0 = beg; p0 < end; p0 += 32) {
        const int cnt = static_cast<int>(end - p0 < 32 ? end - p0 : 32);
        __syncwarp();
        slot[lane] = make_double2(v, __longlong_as_double(static_cast<long long>(c)));
        __syncwarp();
        if (p0 + 32 + lane < end) {
            c = __ldg(idx + p0 + 32 + lane);
            v = __ldg(val + p0 + 32 + lane);
        }
        for (int j0 = 0; j0 < cnt; j0 += U) {
            double xa[U][4], xc[U][4], xb[U][2], vj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u;
                vj[u] = 0.0;
                if (j < cnt) {
                    const double2 e = slot[j];
                    vj[u] = e.x;
                    const int64_t cj = __double_as_longlong(e.y);
                    if (act0) ld256(x0 + cj * ld, xa[u]);
                    if (act1) ld256(x1 + cj * ld, xc[u]);
                    if (act2) {
                        const double2 t = __ldg(reinterpret_cast<const double2*>(x2 + cj * ld));
                        xb[u][0] = t.x;
                        xb[u][1] = t.y;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (j0 + u < cnt) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) acc[t] = fma(vj[u], xa[u][t], acc[t]);
#pragma unroll
                    for (int t = 0; t < 4; ++t) acc[4 + t] = fma(vj[u], xc[u][t], acc[4 + t]);
                    acc[8] = fma(vj[u], xb[u][0], acc[8]);
                    acc[9] = fma(vj[u], xb[u][1], acc[9]);
                }
            }
        }
    }
    double* yr = y + (kChunk ? rpos : row) * ld;
    if (kShift && !kChunk) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) {
            const double* qr = q + row * ld;
            if (act0) {
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[t] = fma(-alpha, qr[8 * lane + t], acc[t]);
            }
            if (act1) {
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[4 + t] = fma(-alpha, qr[8 * lane + 4 + t], acc[4 + t]);
            }
            if (act2) {
                acc[8] = fma(-alpha, qr[256 + 2 * lane], acc[8]);
                acc[9] = fma(-alpha, qr[256 + 2 * lane + 1], acc[9]);
            }
        }
    }
    if (act0) {
        *reinterpret_cast<double2*>(yr + 8 * lane) = make_double2(acc[0], acc[1]);
        *reinterpret_cast<double2*>(yr + 8 * lane + 2) = make_double2(acc[2], acc[3]);
    }
    if (act1) {
        *reinterpret_cast<double2*>(yr + 8 * lane + 4) = make_double2(acc[4], acc[5]);
        *reinterpret_cast<double2*>(yr + 8 * lane + 6) = make_double2(acc[6], acc[7]);
    }
    if (act2) *reinterpret_cast<double2*>(yr + 256 + 2 * lane) = make_double2(acc[8], acc[9]);
}

// Column-slab kernel (slab-major over the whole launch). The work item is a
// (W-column slab, row) pair; the grid walks every row of slab 0, then every
// row of slab 1, ... so at any moment the SMs gather from ONE W-column slab of
// X — 8 W bytes per X row — and the slab's hot rows stay in L2 (C4: a 32-column
// slab of the 10 GB X is 1.07 GB, and its ~500k hottest rows, ~88% of the R-MAT
// gathers, fit in the 126 MB L2; a whole 2.4 KB row per gather keeps only ~45%).
// The price is re-reading the (index, value) stream once per slab (12 B per
// nonzero per slab), which is why it is a per-ld choice.
// A warp holds R = 128 / W rows (ordered longest first, so neighbours have
// similar lengths); each group of G = W / 4 lanes owns one row and gathers the
// row's slab with one 256-bit load per lane and nonzero, U nonzeros ahead of the
// FMAs. The chains are the reference's CSR-order FMA chains from 0.0, so the
// result is bitwise that of the whole-row kernels. The split rows' chunks are
// items of the same launch (first, in list order), written to `partial`.
// kHint: the (index, value) stream and the output rows are marked L2
// evict_first, so the streaming bytes do not evict the slab's hot X rows.
template <int W>
struct SlabCfg {
    static constexpr int G = W / 4;   // lanes per row
    static constexpr int R = 32 / G;  // rows per warp
};
constexpr int kSlabWarps = 8;

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <bool kHint>
__device__ __forceinline__ int32_t ld_idx(const int32_t* p, uint64_t pol) {
    if (!kHint) return __ldg(p);
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

template <bool kHint>
__device__ __forceinline__ double ld_val(const double* p, uint64_t pol) {
    if (!kHint) return __ldg(p);
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

template <bool kHint>
__device__ __forceinline__ void st4(double* p, const double (&a)[4], uint64_t pol) {
    if (!kHint) {
        *reinterpret_cast<double2*>(p) = make_double2(a[0], a[1]);
        *reinterpret_cast<double2*>(p + 2) = make_double2(a[2], a[3]);
        return;
    }
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(a[0]),
                 "d"(a[1]), "d"(a[2]), "d"(a[3]), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 256-bit gather with an L2 eviction-priority policy, not allocated in L1
__device__ __forceinline__ void ld256_pol(const double* p, double (&r)[4], uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
        : "l"(p), "l"(pol));
}

// kTag: `idx` is the hot/cold-tagged copy of the column indices (sign bit set
// on the X rows outside the hot set, DevCsr-independent, built per solve by
// the engine): hot gathers carry L2 evict_last, cold ones evict_first, so the
// L2 keeps the most-referenced slab rows (an LFU-like policy) instead of LRU's
// mix (C4: ~84% of the 64-column slab gathers go to the 246k hottest rows, which
// fit in the L2, but LRU kept only 51-60% hits; profiles/README.md)
template <bool kShift, int W, int U, bool kHint, int MB, bool kTag>
__global__ void __launch_bounds__(32 * kSlabWarps, MB)
spmm_slab_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ idx, const double* __restrict__ val,
                 const int32_t* __restrict__ order, int64_t nsplit, int64_t nchunks,
                 const int64_t* __restrict__ chunk_p0, const int64_t* __restrict__ chunk_p1, int64_t rows,
                 int64_t blocks_per_slab, const double* __restrict__ x, double* __restrict__ y,
                 double* __restrict__ partial, int64_t ld, const double* __restrict__ q,
                 const double* __restrict__ alpha_p, const int32_t* __restrict__ gate, int64_t x_rows, bool x_slab,
                 bool y_slab, int64_t active, const int64_t* __restrict__ obeg, const int32_t* __restrict__ olen,
                 bool uni, double uval) {
    constexpr int G = SlabCfg<W>::G, R = SlabCfg<W>::R;
    if (gate_closed(gate)) return;
    __shared__ __align__(16) double2 cv[kSlabWarps][R][2 * (G + 1)];  // two batches; +1: groups on distinct banks
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / G, t = lane % G;
    const int slab = static_cast<int>(blockIdx.x / blocks_per_slab);
    const int64_t rb = blockIdx.x - static_cast<int64_t>(slab) * blocks_per_slab;
    const int64_t items = nchunks + (active - nsplit);
    const int64_t it = (rb * kSlabWarps + warp) * R + g;
    const bool valid = it < items;
    const int64_t col = static_cast<int64_t>(slab) * W + 4 * t;
    int64_t beg = 0, end = 0;
    double* out = nullptr;  // this lane's four outputs
    const double* qrow = nullptr;
    if (valid) {
        if (it < nchunks) {
            beg = chunk_p0[it];
            end = chunk_p1[it];
            DSVD_DCHECK(beg <= end);
            out = partial + it * ld + col;
        } else {
            const int64_t pos = nsplit + (it - nchunks);
            const int64_t row = order[pos];
            DSVD_DCHECK(row >= 0 && row < rows);
            if (obeg != nullptr) {  // independent of the order[] load
                beg = obeg[pos];
                end = beg + olen[pos];
            } else {
                beg = off[row];
                end = off[row + 1];
            }
            out = y_slab ? y + (static_cast<int64_t>(slab) * rows + row) * W + 4 * t : y + row * ld + col;
            if (kShift) qrow = q + row * ld;
        }
    }
    const bool act = valid && col < ld;  // ld is a multiple of 4: all four columns exist
    // X row c's slab: x + c * ld + col (row-major) or x + (slab * x_rows + c) * W + 4t (slab-major)
    const double* xc = x_slab ? x + static_cast<int64_t>(slab) * x_rows * W + 4 * t : x + (act ? col : 0);
    const int64_t xstride = x_slab ? W : ld;
    const int len = static_cast<int>(end - beg);  // <= split_chunk (or a whole short row)
    int maxlen = len;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(kFull, maxlen, o));
    const uint64_t pol = kHint ? evict_first_policy() : 0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // Rolling gather pipeline, D = U loads in flight per lane at all times:
    // nonzero q is consumed (its FMAs, in CSR order) just before the load of
    // nonzero q + U is issued into the same registers. The (index, value) pairs
    // sit in a two-batch shared-memory ring per row (batch = G nonzeros, staged
    // one batch ahead) fed from registers loaded two batches ahead, so neither
    // the index loads nor the gathers expose their latency at batch boundaries.
    double2* ring = cv[warp][g];  // [2][G], padded per group
    const uint64_t pol_hot = kTag ? evict_last_policy() : 0, pol_cold = kTag ? evict_first_policy() : 0;
    // gather of tagged index e: strip the tag, pick the policy
    auto gather = [&](long long e, double (&r)[4]) {
        if (kTag) {
            const int32_t ci = static_cast<int32_t>(e);
            DSVD_DCHECK((ci & 0x7fffffff) < x_rows);
            ld256_pol(xc + static_cast<int64_t>(ci & 0x7fffffff) * xstride, r, ci < 0 ? pol_cold : pol_hot);
        } else {
            DSVD_DCHECK(e >= 0 && e < x_rows);
            ld256(xc + e * xstride, r);
        }
    };
    int cb = 0;
    double vb = 0.0;
    // (uni: every value is uval, the value stream is not read)
    if (t < len) {
        cb = ld_idx<kHint>(idx + beg + t, pol);
        vb = uni ? uval : ld_val<kHint>(val + beg + t, pol);
    }
    ring[t] = make_double2(vb, __longlong_as_double(static_cast<long long>(cb)));  // batch 0
    cb = 0;
    vb = 0.0;
    if (G + t < len) {  // batch 1, staged when batch 0 starts
        cb = ld_idx<kHint>(idx + beg + G + t, pol);
        vb = uni ? uval : ld_val<kHint>(val + beg + G + t, pol);
    }
    __syncwarp();
    double xa[U][4], va[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // the first U gathers
        va[u] = 0.0;
        if (u < len && act) {
            const double2 e = ring[u];
            va[u] = e.x;
            gather(__double_as_longlong(e.y), xa[u]);
        }
    }
    for (int p = 0; p < maxlen; p += U) {
        if (p % G == 0) {  // entering batch p / G: stage batch p / G + 1, fetch batch p / G + 2
            const int b = p / G;
            __syncwarp();
            ring[((b + 1) & 1) * (G + 1) + t] = make_double2(vb, __longlong_as_double(static_cast<long long>(cb)));
            __syncwarp();
            cb = 0;
            vb = 0.0;
            if ((b + 2) * G + t < len) {
                cb = ld_idx<kHint>(idx + beg + (b + 2) * G + t, pol);
                vb = uni ? uval : ld_val<kHint>(val + beg + (b + 2) * G + t, pol);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = p + u;
            if (q < len) {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[k] = fma(va[u], xa[u][k], acc[k]);
            }
            const int qn = q + U;
            if (qn < len && act) {
                const double2 e = ring[((qn / G) & 1) * (G + 1) + qn % G];
                va[u] = e.x;
                gather(__double_as_longlong(e.y), xa[u]);
            }
        }
    }
    if (!act) return;
    if (kShift && qrow != nullptr) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) {  // solver.cpp:94 skips the update when alpha == 0
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = fma(-alpha, qrow[col + k], acc[k]);
        }
    }
    if (it < nchunks) st4<false>(out, acc, pol);  // read back by the combine: keep in L2
    else st4<kHint>(out, acc, pol);
}

// y(row_i, :) = sum over the row's chunks, in chunk order, of partial(chunk, :),
// then the shift epilogue.
// y(row_i, :) = sum of the row's chunk partials (chunk_slot maps its chunks, in
// CSR order, to partial rows), then the shift epilogue. One block per (split
// row, 64-column group): warp w sums a contiguous eighth of the chunks in
// order, the eight warp sums are added in warp order (a fixed tree:
// deterministic), so a hub row with hundreds of chunks is not one thread's
// serial chain.
template <bool kShift>
__global__ void __launch_bounds__(256)
split_combine_tree_kernel(const double* __restrict__ partial, const int32_t* __restrict__ split_first,
                     const int32_t* __restrict__ slot, const int32_t* __restrict__ order, int64_t nsplit,
                     double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                     const double* __restrict__ alpha_p, const int32_t* __restrict__ gate, int y_slab_w = 0,
                     int64_t y_rows = 0) {
    if (gate_closed(gate)) return;
    __shared__ double2 red[8][32];
    const int64_t i = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t col = static_cast<int64_t>(blockIdx.y) * 64 + 2 * lane;
    const bool act = col < ld;  // ld is a multiple of 4
    const int32_t c0 = split_first[i], c1 = split_first[i + 1];
    const int32_t per = (c1 - c0 + 7) / 8;
    const int32_t a = c0 + warp * per, b = min(c1, a + per);
    double2 acc = make_double2(0.0, 0.0);
    if (act) {
        auto at = [&](int32_t c) {
            const int64_t r = slot != nullptr ? slot[c] : c;
            DSVD_DCHECK(r >= 0 && c >= c0 && c < c1);
            return *reinterpret_cast<const double2*>(partial + r * ld + col);
        };
        int32_t c = a;
        for (; c + 4 <= b; c += 4) {
            const double2 v0 = at(c), v1 = at(c + 1), v2 = at(c + 2), v3 = at(c + 3);
            acc.x += v0.x; acc.y += v0.y;
            acc.x += v1.x; acc.y += v1.y;
            acc.x += v2.x; acc.y += v2.y;
            acc.x += v3.x; acc.y += v3.y;
        }
        for (; c < b; ++c) {
            const double2 v = at(c);
            acc.x += v.x;
            acc.y += v.y;
        }
    }
    red[warp][lane] = acc;
    __syncthreads();
    if (warp != 0 || !act) return;
    double2 s = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
        s.x += red[w][lane].x;
        s.y += red[w][lane].y;
    }
    const int64_t row = order[i];
    if (kShift) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) {
            const double2 qv = *reinterpret_cast<const double2*>(q + row * ld + col);
            s.x = fma(-alpha, qv.x, s.x);
            s.y = fma(-alpha, qv.y, s.y);
        }
    }
    // slab-major output (y_slab_w > 0): col and col + 1 share a slab (both even, w a multiple of 4)
    double* dst = y_slab_w > 0 ? y + ((col / y_slab_w) * y_rows + row) * y_slab_w + col % y_slab_w : y + row * ld + col;
    *reinterpret_cast<double2*>(dst) = s;
}

// Flat variant for rows with few chunks: one thread per output element, the
// chunk rows fetched eight ahead of the in-order additions.
template <bool kShift>
__global__ void split_combine_kernel(const double* __restrict__ partial, const int32_t* __restrict__ split_first,
                                     const int32_t* __restrict__ slot, const int32_t* __restrict__ order,
                                     int64_t nsplit, double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                                     const double* __restrict__ alpha_p, const int32_t* __restrict__ gate,
                                     int y_slab_w = 0, int64_t y_rows = 0) {
    if (gate_closed(gate)) return;
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= nsplit * ld) return;
    const int64_t i = e / ld, col = e - (e / ld) * ld;
    const int64_t row = order[i];
    double acc = 0.0;
    const int32_t c0 = split_first[i], c1 = split_first[i + 1];
    int32_t c = c0;
    for (; c + 8 <= c1; c += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            v[u] = partial[static_cast<int64_t>(slot != nullptr ? slot[c + u] : c + u) * ld + col];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; c < c1; ++c) acc += partial[static_cast<int64_t>(slot != nullptr ? slot[c] : c) * ld + col];
    if (kShift) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) acc = fma(-alpha, q[row * ld + col], acc);
    }
    y[y_slab_w > 0 ? ((col / y_slab_w) * y_rows + row) * y_slab_w + col % y_slab_w : row * ld + col] = acc;
}

__global__ void panel_bounds_kernel(const int32_t* __restrict__ order, const int64_t* __restrict__ off,
                                    const int32_t* __restrict__ idx, int64_t n, int npanel, int64_t panel_rows,
                                    int64_t* __restrict__ bounds) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= n * (npanel + 1)) return;
    const int64_t r = t / (npanel + 1);
    const int p = static_cast<int>(t - r * (npanel + 1));
    const int64_t row = order[r];
    int64_t lo = off[row], hi = off[row + 1];
    if (p == npanel) {
        bounds[t] = hi;
        return;
    }
    const int64_t key = p * panel_rows;
    while (lo < hi) {  // first position with idx >= key
        const int64_t mid = lo + (hi - lo) / 2;
        if (idx[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    bounds[t] = lo;
}

// ---- split-row chunk planning on the device (build_chunks) ------------------
// Split row r (order[r], r < *nsplit) of length L is cut into groups of gs
// consecutive X-row panels (gs = ceil(npanel / max(1, min(npanel, L / C)))), and
// each group's CSR range into ceil(len / C) near-equal chunks; a chunk is listed
// under the middle panel of its group. npanel == 1: one group, the whole row.

// first position in [lo, hi) of row data with idx >= key (indices ascending)
__device__ __forceinline__ int64_t lower_pos(const int32_t* __restrict__ idx, int64_t lo, int64_t hi, int64_t key) {
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (idx[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <bool kEmit>
__device__ __forceinline__ int64_t plan_row(const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                                            int64_t row, int npanel, int64_t panel_rows, int64_t C, int64_t out0,
                                            int64_t* __restrict__ p0, int64_t* __restrict__ p1,
                                            int32_t* __restrict__ panel) {
    const int64_t beg = off[row], end = off[row + 1];
    const int64_t L = end - beg;
    const int64_t groups = max(int64_t(1), min(static_cast<int64_t>(npanel), L / C));
    const int gs = static_cast<int>((npanel + groups - 1) / groups);
    int64_t nch = 0;
    int64_t b = beg;
    for (int p = 0; p < npanel; p += gs) {
        const int pe = min(npanel, p + gs);
        const int64_t e = pe == npanel ? end : lower_pos(idx, b, end, static_cast<int64_t>(pe) * panel_rows);
        const int64_t len = e - b;
        if (len > 0) {
            const int64_t n = (len + C - 1) / C, cs = (len + n - 1) / n;
            if (kEmit) {
                DSVD_DCHECK(b >= beg && e <= end);
                for (int64_t j = 0; j < n; ++j) {
                    p0[out0 + nch + j] = b + j * cs;
                    p1[out0 + nch + j] = min(e, b + (j + 1) * cs);
                    panel[out0 + nch + j] = (p + pe - 1) / 2;
                }
            }
            nch += n;
        }
        b = e;
    }
    return nch;
}

// row_nch[r] = chunks of split row r; 0 for the other rows
__global__ void chunk_count_kernel(const int32_t* __restrict__ order, const int64_t* __restrict__ off,
                                   const int32_t* __restrict__ idx, int64_t rows, const int32_t* __restrict__ nsplit,
                                   int npanel, int64_t panel_rows, int64_t C, int32_t* __restrict__ row_nch) {
    const int64_t ns = *nsplit;
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        row_nch[r] = r < ns ? static_cast<int32_t>(plan_row<false>(off, idx, order[r], npanel, panel_rows, C, 0,
                                                                   nullptr, nullptr, nullptr))
                            : 0;
}

__global__ void chunk_emit_kernel(const int32_t* __restrict__ order, const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ idx, int64_t ns, int npanel, int64_t panel_rows,
                                  int64_t C, const int32_t* __restrict__ first, int64_t* __restrict__ p0,
                                  int64_t* __restrict__ p1, int32_t* __restrict__ panel) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < ns;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        plan_row<true>(off, idx, order[r], npanel, panel_rows, C, first[r], p0, p1, panel);
}

// list position `pos` holds chunk ids[pos]: slot[id] = pos, p0/p1 in list order
__global__ void chunk_place_kernel(const int32_t* __restrict__ ids, int64_t nc, const int64_t* __restrict__ p0,
                                   const int64_t* __restrict__ p1, int32_t* __restrict__ slot,
                                   int64_t* __restrict__ q0, int64_t* __restrict__ q1) {
    for (int64_t pos = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; pos < nc;
         pos += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t id = ids[pos];
        DSVD_DCHECK(id >= 0 && id < nc);
        slot[id] = static_cast<int32_t>(pos);
        q0[pos] = p0[id];
        q1[pos] = p1[id];
    }
}

__global__ void iota32_kernel(int32_t* __restrict__ v, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<int32_t>(i);
}

__global__ void prefix_bounds_kernel(const int32_t* __restrict__ order, const int64_t* __restrict__ off,
                                     int64_t n, int64_t* beg, int64_t* end) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) {
        const int64_t r = order[i];
        beg[i] = off[r];
        end[i] = off[r + 1];
    }
}

// ---- hub rows ------------------------------------------------------------------
// One warp per (hub row, 32-column slab); one lane per column, so each lane
// runs its column's FMA chain over the row in CSR order (bitwise as above).
// Gathered X values and the (index, value) stream move through a per-warp
// shared-memory ring with cp.async: kHubNB batches of 32 nonzeros are in
// flight while the chain consumes the oldest, so a 200k-nonzero row runs at
// the FMA-latency bound instead of one L2/DRAM round trip per few nonzeros.
constexpr int kHubNB = 4;                 // gather batches in flight (ring depth)
constexpr int kHubWarps = 2;              // warps per block
constexpr int kHubWarpDoubles = kHubNB * 32 * 32 + 2 * kHubNB * 32;  // gathers + values
constexpr int kHubWarpInts = 2 * kHubNB * 32;                        // indices
constexpr size_t kHubSmem =
    kHubWarps * (sizeof(double) * kHubWarpDoubles + sizeof(int32_t) * kHubWarpInts);

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <bool kShift>
__global__ void __launch_bounds__(32 * kHubWarps)
spmm_hub_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                const double* __restrict__ val, const int32_t* __restrict__ order,
                const int32_t* __restrict__ n_hub_p, int nslab, const double* __restrict__ x,
                double* __restrict__ y, int64_t ld, const double* __restrict__ q,
                const double* __restrict__ alpha_p, const int32_t* __restrict__ gate) {
    if (gate_closed(gate)) return;
    extern __shared__ double hub_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * kHubWarps + warp;
    if (item >= static_cast<int64_t>(*n_hub_p) * nslab) return;
    const int64_t row = order[item / nslab];
    const int64_t col = static_cast<int64_t>(item % nslab) * 32 + lane;
    const bool active = col < ld;
    double* ring = hub_smem + warp * kHubWarpDoubles;        // [NB][32 nnz][32 lanes]
    double* vring = ring + kHubNB * 32 * 32;                  // [2NB][32]
    int32_t* iring = reinterpret_cast<int32_t*>(hub_smem + kHubWarps * kHubWarpDoubles) +
                     warp * kHubWarpInts;                     // [2NB][32]
    const int64_t beg = off[row], end = off[row + 1];
    const int64_t nb = (end - beg + 31) / 32;
    const double* xc = x + (active ? col : 0);

    // (index, value) batch b -> slot b % 2NB
    auto fetch_iv = [&](int64_t b) {
        const int64_t p = beg + b * 32 + lane;
        if (b < nb && p < end) {
            cp_async4(iring + (b % (2 * kHubNB)) * 32 + lane, idx + p);
            cp_async8(vring + (b % (2 * kHubNB)) * 32 + lane, val + p);
        }
    };
    // gathers of batch b -> ring slot b % NB (indices must already be in smem)
    auto gather = [&](int64_t b) {
        if (b >= nb || !active) return;
        const int cnt = static_cast<int>(min(static_cast<int64_t>(32), end - beg - b * 32));
        const int32_t* ib = iring + (b % (2 * kHubNB)) * 32;
        double* slot = ring + (b % kHubNB) * 1024;
        for (int j = 0; j < cnt; ++j) cp_async8(slot + j * 32 + lane, xc + static_cast<int64_t>(ib[j]) * ld);
    };

    // prologue: indices of batches 0..NB-1 first (one group), then gathers 0..NB-2
    for (int b = 0; b < kHubNB; ++b) fetch_iv(b);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (int b = 0; b < kHubNB - 1; ++b) {
        gather(b);
        fetch_iv(b + kHubNB);
        cp_async_commit();
    }
    double acc = 0.0;
    for (int64_t b = 0; b < nb; ++b) {
        gather(b + kHubNB - 1);      // its indices arrived with an older group
        fetch_iv(b + 2 * kHubNB - 1);
        cp_async_commit();
        cp_async_wait<kHubNB - 1>();  // batch b (gathers and values) has landed
        __syncwarp();
        const double* slot = ring + (b % kHubNB) * 1024;
        const double* vb = vring + (b % (2 * kHubNB)) * 32;
        const int cnt = static_cast<int>(min(static_cast<int64_t>(32), end - beg - b * 32));
        if (cnt == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc = fma(vb[j], slot[j * 32 + lane], acc);
        } else {
            for (int j = 0; j < cnt; ++j) acc = fma(vb[j], slot[j * 32 + lane], acc);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    if (!active) return;
    if (kShift) {
        const double alpha = *alpha_p;
        if (alpha != 0.0) acc = fma(-alpha, q[row * ld + col], acc);
    }
    y[row * ld + col] = acc;
}


__global__ void count_ge_kernel(const int32_t* __restrict__ sorted_desc, int64_t n, int64_t t,
                                int32_t* out) {
    // number of leading entries >= t in a descending array (binary search)
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (sorted_desc[mid] >= t) lo = mid + 1; else hi = mid;
    }
    *out = static_cast<int32_t>(lo);
}

__global__ void narrow_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                              int64_t nnz, int64_t cols, int32_t* bad) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t c = src[p];
        if (c < 0 || c >= cols) {
            *bad = 1;
            c = 0;
        }
        dst[p] = static_cast<int32_t>(c);
    }
}

__global__ void widen_kernel(const int32_t* __restrict__ src, int64_t* __restrict__ dst,
                             int64_t nnz) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[p] = src[p];
}

__global__ void check_offsets_kernel(const int64_t* __restrict__ off, int64_t rows, int64_t nnz,
                                     int32_t* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (off[i] > off[i + 1] || off[i] < 0 || off[i + 1] > nnz) *bad = 1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[rows] != nnz)) *bad = 1;
}

// row_of[p] = i for p in [off[i], off[i+1]) — one warp per row.
__global__ void expand_rows_kernel(const int64_t* __restrict__ off, int64_t rows,
                                   int32_t* __restrict__ row_of) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
         i < rows; i += warps) {
        for (int64_t p = off[i] + lane; p < off[i + 1]; p += 32) row_of[p] = static_cast<int32_t>(i);
    }
}

__global__ void iota_kernel(int32_t* __restrict__ v, int64_t n) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[p] = static_cast<int32_t>(p);
}

__global__ void gather_transpose_kernel(const int32_t* __restrict__ perm,
                                        const int32_t* __restrict__ row_of,
                                        const double* __restrict__ val, int32_t* __restrict__ t_idx,
                                        double* __restrict__ t_val, int64_t nnz) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t p = perm[k];
        t_idx[k] = row_of[p];
        t_val[k] = val[p];
    }
}

// t_off[c] = first position whose (sorted) column key is >= c.
__global__ void offsets_from_keys_kernel(const int32_t* __restrict__ keys, int64_t nnz,
                                         int64_t cols, int64_t* __restrict__ t_off) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t key = keys[k];
        const int64_t prev = k > 0 ? static_cast<int64_t>(keys[k - 1]) : -1;
        for (int64_t c = prev + 1; c <= key; ++c) t_off[c] = k;
        if (k == nnz - 1)
            for (int64_t c = key + 1; c <= cols; ++c) t_off[c] = nnz;
    }
}

__global__ void fill_i64_kernel(int64_t* __restrict__ p, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void order_ranges_kernel(const int32_t* __restrict__ order, const int64_t* __restrict__ off, int64_t rows,
                                    int64_t* __restrict__ obeg, int32_t* __restrict__ olen) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = order[i];
        obeg[i] = off[r];
        const int64_t n = off[r + 1] - off[r];
        olen[i] = static_cast<int32_t>(n > 0x7fffffff ? 0x7fffffff : n);
    }
}

__global__ void row_lengths_kernel(const int64_t* __restrict__ off, int64_t rows,
                                   int32_t* __restrict__ len, int32_t* __restrict__ ids) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t n = off[i + 1] - off[i];
        len[i] = static_cast<int32_t>(n > 0x7fffffff ? 0x7fffffff : n);
        ids[i] = static_cast<int32_t>(i);
    }
}

int grid_for(int64_t n, int threads = 256) {
    const int64_t g = ceil_div(n, threads);
    return static_cast<int>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

int key_bits(int64_t maxval) {
    int b = 1;
    while (b < 32 && (int64_t(1) << b) <= maxval) ++b;
    return b;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// y rows of the split rows = their chunk partials summed in chunk order (+ shift)
void combine_split(const SpmmArgs& s, cudaStream_t stream, double* partial) {
    const DevCsr& a = *s.a;
    const int yw = s.y_slab ? s.slab : 0;
    // rows with many chunks (hub columns of A^T): the 8-warp tree per row
    if (a.max_row_chunks > 32) {
        const dim3 cgrid(static_cast<unsigned>(a.nsplit), static_cast<unsigned>(ceil_div(s.ld, 64)));
        if (s.q != nullptr)
            split_combine_tree_kernel<true><<<cgrid, 256, 0, stream>>>(partial, a.split_first, a.chunk_slot, a.order,
                                                                       a.nsplit, s.y, s.ld, s.q, s.alpha, s.gate, yw,
                                                                       a.rows);
        else
            split_combine_tree_kernel<false><<<cgrid, 256, 0, stream>>>(partial, a.split_first, a.chunk_slot,
                                                                        a.order, a.nsplit, s.y, s.ld, nullptr,
                                                                        nullptr, s.gate, yw, a.rows);
    } else {
        const int64_t n = a.nsplit * s.ld;
        if (s.q != nullptr)
            split_combine_kernel<true><<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, stream>>>(
                partial, a.split_first, a.chunk_slot, a.order, a.nsplit, s.y, s.ld, s.q, s.alpha, s.gate, yw, a.rows);
        else
            split_combine_kernel<false><<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, stream>>>(
                partial, a.split_first, a.chunk_slot, a.order, a.nsplit, s.y, s.ld, nullptr, nullptr, s.gate, yw,
                a.rows);
    }
    DSVD_LAUNCH_CHECK();
}

// Rows without nonzeros (order[i], i in [ne, rows)): y = 0.0, or the shifted
// update of an empty chain, fma(-alpha, q, 0.0), unless alpha == 0 (add_scaled skipped).
__global__ void empty_rows_kernel(const int32_t* __restrict__ order, int64_t ne, int64_t rows, int64_t ld,
                                  double* __restrict__ y, const double* __restrict__ q,
                                  const double* __restrict__ alpha_p, const int32_t* __restrict__ gate, int y_slab_w) {
    if (gate_closed(gate)) return;
    const double alpha = q != nullptr ? *alpha_p : 0.0;
    const int64_t g = ld / 4, units = (rows - ne) * g;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < units;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = order[ne + e / g], col = 4 * (e % g);
        DSVD_DCHECK(row >= 0 && row < rows);
        double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
        if (alpha != 0.0) {
            const double4 qv = *reinterpret_cast<const double4*>(q + row * ld + col);
            v = make_double4(fma(-alpha, qv.x, 0.0), fma(-alpha, qv.y, 0.0), fma(-alpha, qv.z, 0.0),
                             fma(-alpha, qv.w, 0.0));
        }
        double* dst = y_slab_w > 0 ? y + ((col / y_slab_w) * rows + row) * y_slab_w + col % y_slab_w : y + row * ld + col;
        *reinterpret_cast<double4*>(dst) = v;
    }
}

// Short rows (at most kShortRow nonzeros) as whole rows: one 16-lane group per
// row gathers all of each nonzero's slab-major X row at once (round r covers
// columns 64r .. 64r + 63: one 64-column slab, or two 32-column slabs), so the
// row's metadata and index loads and its latency chain are paid once per row
// instead of once per (row, slab). Every column's FMA chain is the slab
// kernel's (CSR order, the same shift epilogue): the rows are bitwise those of
// the per-slab launch.
constexpr int kShortRounds = 5;  // ld <= 320
template <bool kShift, int W>
__global__ void __launch_bounds__(256, 2)
spmm_short_rows_kernel(const int32_t* __restrict__ idx, const double* __restrict__ val,
                       const int32_t* __restrict__ order, const int64_t* __restrict__ obeg,
                       const int32_t* __restrict__ olen, int64_t first, int64_t end, int64_t rows,
                       const double* __restrict__ x, int64_t x_rows, double* __restrict__ y, int64_t ld, bool y_slab,
                       const double* __restrict__ q, const double* __restrict__ alpha_p,
                       const int32_t* __restrict__ gate, bool uni, double uval) {
    if (gate_closed(gate)) return;
    const int lane = threadIdx.x & 31, t = lane & 15;
    const unsigned gmask = 0xffffu << (lane & 16);
    const int64_t pos = first + (static_cast<int64_t>(blockIdx.x) * 16 + (threadIdx.x >> 4));
    if (pos >= end) return;  // whole 16-lane groups leave together
    const int64_t row = order[pos];
    const int64_t beg = obeg[pos];
    const int len = olen[pos];
    DSVD_DCHECK(row >= 0 && row < rows && len <= kMidRow);
    // this lane's columns: 4t .. 4t + 3 of each 64-column round, at slab c / W, offset c % W
    int64_t xoff[kShortRounds];
#pragma unroll
    for (int r = 0; r < kShortRounds; ++r) {
        const int c = 64 * r + 4 * t;
        xoff[r] = static_cast<int64_t>(c / W) * x_rows * W + c % W;
    }
    double acc[kShortRounds][4];
#pragma unroll
    for (int r = 0; r < kShortRounds; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[r][k] = 0.0;
    int ci = 0;
    double vi = 0.0;
    for (int p = 0; p < len; ++p) {
        if ((p & 15) == 0) {  // the next 16 (index, value) pairs, one per lane
            ci = 0;
            vi = 0.0;
            if (p + t < len) {
                ci = idx[beg + p + t];
                vi = uni ? uval : val[beg + p + t];
            }
        }
        const int64_t c = __shfl_sync(gmask, ci, p & 15, 16);
        const double v = __shfl_sync(gmask, vi, p & 15, 16);
        DSVD_DCHECK(c >= 0 && c < x_rows);
        double xa[kShortRounds][4];
#pragma unroll
        for (int r = 0; r < kShortRounds; ++r)
            if (64 * r + 4 * t < ld) ld256(x + xoff[r] + c * W, xa[r]);
#pragma unroll
        for (int r = 0; r < kShortRounds; ++r)
            if (64 * r + 4 * t < ld)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[r][k] = fma(v, xa[r][k], acc[r][k]);
    }
    const double alpha = kShift ? *alpha_p : 0.0;
#pragma unroll
    for (int r = 0; r < kShortRounds; ++r) {
        const int64_t col = 64 * r + 4 * t;
        if (col >= ld) continue;
        if (kShift && alpha != 0.0) {  // solver.cpp:94 skips the update when alpha == 0
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[r][k] = fma(-alpha, q[row * ld + col + k], acc[r][k]);
        }
        double* out = y_slab ? y + ((col / W) * rows + row) * W + col % W : y + row * ld + col;
        *reinterpret_cast<double4*>(out) = make_double4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
    }
}

int g_short_whole_rows = 1;  // option "spmm_short_rows" (sparse.cuh set_spmm_short_rows)

// One slab-kernel launch over the chunks [0, nchunks) and the rows at order
// positions [first, end), slab-major.
template <int W, bool kHint, int U, int MB, bool kTag>
void launch_slab_range(const SpmmArgs& s, cudaStream_t stream, double* partial, int64_t nchunks, int64_t first,
                       int64_t end) {
    const DevCsr& a = *s.a;
    constexpr int RB = kSlabWarps * SlabCfg<W>::R;
    const int64_t items = nchunks + (end - first);
    if (items <= 0) return;
    const int64_t bps = ceil_div(items, RB);
    const int64_t nslab = ceil_div(s.ld, W);
    if (bps * nslab >= (int64_t(1) << 31)) fail(DSVD_UNSUPPORTED, "spmm: slab grid too large");
    const unsigned blocks = static_cast<unsigned>(bps * nslab);
    const int32_t* ix = kTag ? s.idx_tag : a.idx;
    if (s.q != nullptr)
        spmm_slab_kernel<true, W, U, kHint, MB, kTag><<<blocks, 32 * kSlabWarps, 0, stream>>>(
            a.off, ix, a.val, a.order, first, nchunks, a.chunk_p0, a.chunk_p1, a.rows, bps, s.x, s.y, partial,
            s.ld, s.q, s.alpha, s.gate, a.cols, s.x_slab, s.y_slab, end, a.obeg, a.olen, a.uniform, a.uval);
    else
        spmm_slab_kernel<false, W, U, kHint, MB, kTag><<<blocks, 32 * kSlabWarps, 0, stream>>>(
            a.off, ix, a.val, a.order, first, nchunks, a.chunk_p0, a.chunk_p1, a.rows, bps, s.x, s.y, partial,
            s.ld, nullptr, nullptr, s.gate, a.cols, s.x_slab, s.y_slab, end, a.obeg, a.olen, a.uniform, a.uval);
    DSVD_LAUNCH_CHECK();
}

template <int W, bool kHint, int U, int MB, bool kTag>
void launch_slab(const SpmmArgs& s, cudaStream_t stream, double* partial) {
    const DevCsr& a = *s.a;
    const int64_t nsplit = partial != nullptr ? a.nsplit : 0;
    const int64_t nchunks = partial != nullptr ? a.nchunks : 0;
    if ((s.x_slab || s.y_slab) && s.slab != W) fail(DSVD_OTHER, "spmm: slab-major block of another slab width");
    // rows with nonzeros run through the kernel; the empty tail of a.order is
    // filled below (or skipped). Rows of at most kShortRow nonzeros (their cost
    // is the per-row load chain, not bandwidth) get their own launch at 48
    // warps per SM (instead of 32) and one gather in flight per lane.
    const int64_t active = a.nonempty_rows >= 0 ? std::max(a.nonempty_rows, nsplit) : a.rows;
    const int64_t nlong = a.long_rows >= 0 ? std::min(std::max(a.long_rows, nsplit), active) : active;
    const bool whole = g_short_whole_rows && s.x_slab && !kTag && s.ld <= 64 * kShortRounds &&
                       a.obeg != nullptr && (g_short_whole_rows == 1 || a.mid_rows >= 0);
    // whole-row short rows: from position ws on (rows of at most kShortRow, or kMidRow, nonzeros)
    const int64_t ws = !whole ? nlong : (g_short_whole_rows == 1 ? nlong : std::min(std::max(a.mid_rows, nsplit), active));
    launch_slab_range<W, kHint, U, MB, kTag>(s, stream, partial, nchunks, nsplit, whole ? ws : nlong);
    if (whole && active > ws) {
        const unsigned blocks = static_cast<unsigned>(ceil_div(active - ws, 16));
        if (s.q != nullptr)
            spmm_short_rows_kernel<true, W><<<blocks, 256, 0, stream>>>(
                a.idx, a.val, a.order, a.obeg, a.olen, ws, active, a.rows, s.x, a.cols, s.y, s.ld, s.y_slab, s.q,
                s.alpha, s.gate, a.uniform, a.uval);
        else
            spmm_short_rows_kernel<false, W><<<blocks, 256, 0, stream>>>(
                a.idx, a.val, a.order, a.obeg, a.olen, ws, active, a.rows, s.x, a.cols, s.y, s.ld, s.y_slab,
                nullptr, nullptr, s.gate, a.uniform, a.uval);
        DSVD_LAUNCH_CHECK();
    } else if (!whole) {
        launch_slab_range<W, kHint, 1, 6, kTag>(s, stream, partial, 0, nlong, active);
    }
    if (active < a.rows && !s.skip_empty) {
        empty_rows_kernel<<<grid_for((a.rows - active) * (s.ld / 4)), 256, 0, stream>>>(
            a.order, active, a.rows, s.ld, s.y, s.q, s.alpha, s.gate, s.y_slab ? W : 0);
        DSVD_LAUNCH_CHECK();
    }
}

template <int W, bool kHint>
void launch_slab_u(const SpmmArgs& s, cudaStream_t stream, double* partial, int depth) {
    // gathers in flight per lane / CTAs per SM: depth 0: 4 / 3 (24 warps), 1: 8 / 2, 2: 2 / 4
    if (s.idx_tag != nullptr) {
        if (depth == 1) launch_slab<W, kHint, 8, 2, true>(s, stream, partial);
        else if (depth == 2) launch_slab<W, kHint, 2, 4, true>(s, stream, partial);
        else launch_slab<W, kHint, 4, 3, true>(s, stream, partial);
        return;
    }
    if (depth == 1) launch_slab<W, kHint, 8, 2, false>(s, stream, partial);
    else if (depth == 2) launch_slab<W, kHint, 2, 4, false>(s, stream, partial);
    else launch_slab<W, kHint, 4, 3, false>(s, stream, partial);
}

void spmm_slab(const SpmmArgs& s, cudaStream_t stream, int w, bool hint, int depth, double* partial) {
    if (s.a->rows == 0) return;
    if (w == 32) {
        if (hint) launch_slab_u<32, true>(s, stream, partial, depth);
        else launch_slab_u<32, false>(s, stream, partial, depth);
    } else {
        if (hint) launch_slab_u<64, true>(s, stream, partial, depth);
        else launch_slab_u<64, false>(s, stream, partial, depth);
    }
}

}  // namespace

void set_spmm_short_rows(int v) { g_short_whole_rows = v < 0 ? 0 : (v > 2 ? 2 : v); }

void spmm(const SpmmArgs& s, cudaStream_t stream, int variant, cudaStream_t side,
          cudaEvent_t fork, cudaEvent_t join, double* partial) {
    const DevCsr& a = *s.a;
    if (a.rows == 0) return;
    // variant bits: 16 skips the bulk rows, 32 skips the hub rows / chunks
    // (benchmarking the two halves separately)
    const bool skip_bulk = (variant & 16) != 0, skip_hub = (variant & 32) != 0;
    // bit 1024: the long-row chunks run on the main stream before the bulk rows
    // (serial) instead of beside them on the side stream
    if ((variant & 1024) != 0 && side != nullptr) side = stream;
    // the whole-row kernel takes the bulk rows and the split chunks when
    // ld <= 192; bits 64 / 128 force the 64-column slab kernel for them, bits
    // 256 / 512 raise the whole-row kernel's gather lookahead from 2 to 4 / 8
    const bool row_bulk = (variant & 64) == 0 && s.ld <= 192, row_chunk = (variant & 128) == 0 && s.ld <= 192;
    // 192 < ld <= 320: the wide whole-row kernel (same bits force the slab kernel)
    const bool wide_bulk = (variant & 64) == 0 && s.ld > 192 && s.ld <= 320,
               wide_chunk = (variant & 128) == 0 && s.ld > 192 && s.ld <= 320;
    const int ru = (variant & 256) ? 4 : (variant & 512) ? 8 : 2;
    // bits 4096 / 8192: the column-slab kernel with 32- / 64-column slabs for the
    // bulk rows AND the split chunks (one launch, slab-major); 16384: its L2
    // evict_first hints on the streaming bytes
    const int slab_w = (variant & 4096) ? 32 : (variant & 8192) ? 64 : 0;
    // bit 131072: the hint only on launches that write a slab-major Y (the A X pass)
    const bool slab_hint = (variant & 16384) != 0 && (!(variant & 131072) || s.y_slab);
    // bits 32768 / 65536: slab gather depth (launch_slab_u)
    const int slab_depth = (variant & 32768) ? 1 : (variant & 65536) ? 2 : 0;
    const bool slab_ok = slab_w > 0 && !skip_bulk && !skip_hub && (a.nsplit == 0 || partial != nullptr);
    if ((s.x_slab || s.y_slab) && !slab_ok)
        fail(DSVD_OTHER, "spmm: slab-major blocks need the column-slab kernel (split mode, slab variant bits)");
    if (slab_ok) {
        spmm_slab(s, stream, slab_w, slab_hint, slab_depth, partial);
        if (a.nsplit > 0 && partial != nullptr) combine_split(s, stream, partial);
        return;
    }
    const bool split = a.nsplit > 0 && partial != nullptr && side != nullptr;
    const int64_t hub = (!split && side != nullptr && a.d_hub_rows != nullptr) ? a.hub_rows : 0;
    if (split) {
        // chunks of the long rows (longest work first) on the side stream,
        // beside the bulk rows on the main stream; combined in chunk order
        DSVD_CUDA_CHECK(cudaEventRecord(fork, stream));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(side, fork, 0));
        const int nslab64 = static_cast<int>(ceil_div(s.ld, kSlab));
        const int64_t citems = skip_hub ? 0 : a.nchunks * nslab64;
        if (citems > 0 && row_chunk) {
            auto k = ru == 4 ? spmm_row_kernel<false, true, 4>
                     : ru == 8 ? spmm_row_kernel<false, true, 8> : spmm_row_kernel<false, true, 2>;
            k<<<static_cast<unsigned>(ceil_div(a.nchunks, kRowWarps)), 32 * kRowWarps, 0, side>>>(
                a.off, a.idx, a.val, a.order, 0, a.nchunks, s.x, partial, s.ld, nullptr, nullptr, s.gate, a.chunk_p0,
                a.chunk_p1);
            DSVD_LAUNCH_CHECK();
        } else if (citems > 0 && wide_chunk) {
            spmm_row_wide_kernel<false, true><<<static_cast<unsigned>(ceil_div(a.nchunks, kRowWarps)),
                                                32 * kRowWarps, 0, side>>>(a.off, a.idx, a.val, a.order, 0, a.nchunks,
                                                                           s.x, partial, s.ld, nullptr, nullptr,
                                                                           s.gate, a.chunk_p0, a.chunk_p1);
            DSVD_LAUNCH_CHECK();
        } else if (citems > 0) {
            spmm_bulk_kernel<false, true><<<static_cast<unsigned>(ceil_div(citems, 8)), 256, 0, side>>>(
                a.off, a.idx, a.val, a.order, 0, a.nchunks, nslab64, s.x, partial, s.ld, nullptr, nullptr,
                s.gate, a.chunk_p0, a.chunk_p1);
            DSVD_LAUNCH_CHECK();
        }
    }
    if (hub > 0) {
        {  // per launch: the attribute is per device (a process may drive several GPUs)
            DSVD_CUDA_CHECK(cudaFuncSetAttribute(spmm_hub_kernel<true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kHubSmem));
            DSVD_CUDA_CHECK(cudaFuncSetAttribute(spmm_hub_kernel<false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kHubSmem));
        }
        DSVD_CUDA_CHECK(cudaEventRecord(fork, stream));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(side, fork, 0));
    }
    if (hub > 0 && !skip_hub) {
        const int nslab32 = static_cast<int>(ceil_div(s.ld, 32));
        const unsigned blocks = static_cast<unsigned>(ceil_div(hub * nslab32, kHubWarps));
        if (s.q != nullptr)
            spmm_hub_kernel<true><<<blocks, 32 * kHubWarps, kHubSmem, side>>>(
                a.off, a.idx, a.val, a.order, a.d_hub_rows, nslab32, s.x, s.y, s.ld, s.q, s.alpha, s.gate);
        else
            spmm_hub_kernel<false><<<blocks, 32 * kHubWarps, kHubSmem, side>>>(
                a.off, a.idx, a.val, a.order, a.d_hub_rows, nslab32, s.x, s.y, s.ld, nullptr, nullptr,
                s.gate);
        DSVD_LAUNCH_CHECK();
    }
    const int nslab = static_cast<int>(ceil_div(s.ld, kSlab));
    const int warps_per_block = 8;
    const int64_t first = split ? a.nsplit : hub;  // rows handled above / in chunks
    const int64_t items = skip_bulk ? 0 : (a.rows - first) * nslab;
    if (items > 0 && wide_bulk) {
        const unsigned blocks = static_cast<unsigned>(ceil_div(a.rows - first, kRowWarps));
        if (s.q != nullptr)
            spmm_row_wide_kernel<true, false><<<blocks, 32 * kRowWarps, 0, stream>>>(
                a.off, a.idx, a.val, a.order, first, a.rows, s.x, s.y, s.ld, s.q, s.alpha, s.gate, nullptr, nullptr);
        else
            spmm_row_wide_kernel<false, false><<<blocks, 32 * kRowWarps, 0, stream>>>(
                a.off, a.idx, a.val, a.order, first, a.rows, s.x, s.y, s.ld, nullptr, nullptr, s.gate, nullptr,
                nullptr);
        DSVD_LAUNCH_CHECK();
    } else if (items > 0 && row_bulk) {
        const unsigned blocks = static_cast<unsigned>(ceil_div(a.rows - first, kRowWarps));
        if (s.q != nullptr) {
            auto k = ru == 4 ? spmm_row_kernel<true, false, 4>
                     : ru == 8 ? spmm_row_kernel<true, false, 8> : spmm_row_kernel<true, false, 2>;
            k<<<blocks, 32 * kRowWarps, 0, stream>>>(a.off, a.idx, a.val, a.order, first, a.rows, s.x, s.y, s.ld, s.q,
                                                     s.alpha, s.gate, nullptr, nullptr);
        } else {
            auto k = ru == 4 ? spmm_row_kernel<false, false, 4>
                     : ru == 8 ? spmm_row_kernel<false, false, 8> : spmm_row_kernel<false, false, 2>;
            k<<<blocks, 32 * kRowWarps, 0, stream>>>(a.off, a.idx, a.val, a.order, first, a.rows, s.x, s.y, s.ld,
                                                     nullptr, nullptr, s.gate, nullptr, nullptr);
        }
        DSVD_LAUNCH_CHECK();
    } else if (items > 0) {
        const int64_t blocks = ceil_div(items, warps_per_block);
        if (s.q != nullptr) {
            spmm_bulk_kernel<true, false><<<static_cast<unsigned>(blocks), 32 * warps_per_block, 0, stream>>>(
                a.off, a.idx, a.val, a.order, first, a.rows, nslab, s.x, s.y, s.ld, s.q, s.alpha, s.gate,
                nullptr, nullptr);
        } else {
            spmm_bulk_kernel<false, false><<<static_cast<unsigned>(blocks), 32 * warps_per_block, 0, stream>>>(
                a.off, a.idx, a.val, a.order, first, a.rows, nslab, s.x, s.y, s.ld, nullptr, nullptr,
                s.gate, nullptr, nullptr);
        }
        DSVD_LAUNCH_CHECK();
    }
    if (split) {
        DSVD_CUDA_CHECK(cudaEventRecord(join, side));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(stream, join, 0));
        combine_split(s, stream, partial);
        return;
    }
    if (hub > 0) {
        DSVD_CUDA_CHECK(cudaEventRecord(join, side));
        DSVD_CUDA_CHECK(cudaStreamWaitEvent(stream, join, 0));
    }
}

void panel_bounds(const DevCsr& m, int64_t nrows, int npanel, int64_t panel_rows, int64_t* bounds,
                  cudaStream_t stream) {
    const int64_t n = nrows * (npanel + 1);
    if (n == 0) return;
    panel_bounds_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, stream>>>(m.order, m.off, m.idx, nrows,
                                                                                   npanel, panel_rows, bounds);
    DSVD_LAUNCH_CHECK();
}

// ---- row-major <-> slab-major copies (32-byte units) --------------------------
template <bool kToSlab>
__global__ void slab_copy_kernel(const double* __restrict__ src, int64_t rows, int64_t ld, int w,
                                 double* __restrict__ dst) {
    // unit e = (slab s, row r, 4-column group t): consecutive threads walk the
    // slab-major side contiguously, the row-major side in 32-byte pieces
    const int64_t g = w / 4, nslab = (ld + w - 1) / w, units = nslab * rows * g;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < units;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t t = e % g, rs = e / g, r = rs % rows, sl = rs / rows;
        const int64_t col = sl * w + 4 * t;
        if (col >= ld) continue;  // past the last column: the slab's padding is never read
        if (kToSlab) {
            const double4 v = *reinterpret_cast<const double4*>(src + r * ld + col);
            *reinterpret_cast<double4*>(dst + 4 * e) = v;
        } else {
            const double4 v = *reinterpret_cast<const double4*>(src + 4 * e);
            *reinterpret_cast<double4*>(dst + r * ld + col) = v;
        }
    }
}

size_t chunk_plan_scratch_bytes(int64_t rows, int64_t max_chunks) {
    size_t a = 0, b = 0, c = 0;
    const int nr = static_cast<int>(rows > 0 ? rows + 1 : 1), nc = static_cast<int>(max_chunks > 0 ? max_chunks : 1);
    cub::DeviceScan::InclusiveSum(nullptr, a, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), nr);
    cub::DeviceReduce::Max(nullptr, b, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), nr);
    cub::DeviceRadixSort::SortPairs(nullptr, c, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), nc);
    return align_up(std::max({a, b, c}));
}

void chunk_plan_count(const DevCsr& m, int npanel, int64_t panel_rows, int32_t* row_nch, int32_t* first,
                      int32_t* d_total_max, void* temp, size_t temp_bytes, cudaStream_t stream) {
    DSVD_CUDA_CHECK(cudaMemsetAsync(first, 0, sizeof(int32_t), stream));
    DSVD_CUDA_CHECK(cudaMemsetAsync(d_total_max, 0, 2 * sizeof(int32_t), stream));
    if (m.rows == 0 || m.split_chunk <= 0) return;
    chunk_count_kernel<<<grid_for(m.rows), 256, 0, stream>>>(m.order, m.off, m.idx, m.rows, m.d_hub_rows, npanel,
                                                            panel_rows, m.split_chunk, row_nch);
    DSVD_LAUNCH_CHECK();
    size_t tb = temp_bytes;
    DSVD_CUDA_CHECK(cub::DeviceScan::InclusiveSum(temp, tb, row_nch, first + 1, static_cast<int>(m.rows), stream));
    DSVD_CUDA_CHECK(cudaMemcpyAsync(d_total_max, first + m.rows, sizeof(int32_t), cudaMemcpyDeviceToDevice, stream));
    tb = temp_bytes;
    DSVD_CUDA_CHECK(cub::DeviceReduce::Max(temp, tb, row_nch, d_total_max + 1, static_cast<int>(m.rows), stream));
}

void chunk_plan_emit(const DevCsr& m, int64_t ns, int npanel, int64_t panel_rows, const int32_t* first, int64_t nc,
                     int64_t* p0, int64_t* p1, int32_t* slot, int64_t* tmp0, int64_t* tmp1, int32_t* keys,
                     int32_t* keys_sorted, int32_t* ids, int32_t* ids_sorted, void* temp, size_t temp_bytes,
                     cudaStream_t stream) {
    if (nc == 0) return;
    if (npanel <= 1) {  // list order = CSR order, no slot map
        chunk_emit_kernel<<<grid_for(ns), 256, 0, stream>>>(m.order, m.off, m.idx, ns, npanel, 0, m.split_chunk, first,
                                                           p0, p1, keys);
        DSVD_LAUNCH_CHECK();
        return;
    }
    chunk_emit_kernel<<<grid_for(ns), 256, 0, stream>>>(m.order, m.off, m.idx, ns, npanel, panel_rows, m.split_chunk,
                                                       first, tmp0, tmp1, keys);
    DSVD_LAUNCH_CHECK();
    iota32_kernel<<<grid_for(nc), 256, 0, stream>>>(ids, nc);
    DSVD_LAUNCH_CHECK();
    size_t tb = temp_bytes;  // stable: chunks of one panel keep their CSR order
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys_sorted, ids, ids_sorted, static_cast<int>(nc),
                                                    0, key_bits(npanel), stream));
    chunk_place_kernel<<<grid_for(nc), 256, 0, stream>>>(ids_sorted, nc, tmp0, tmp1, slot, p0, p1);
    DSVD_LAUNCH_CHECK();
}

// hot[j] = 1 for the k most referenced X rows (the first k entries of the
// transpose's length order), then idx_tag[p] = idx[p] with the sign bit set
// when X row idx[p] is not hot.
__global__ void hot_flags_kernel(const int32_t* __restrict__ order_t, int64_t k, uint8_t* __restrict__ hot) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        hot[order_t[i]] = 1;
}
__global__ void tag_indices_kernel(const int32_t* __restrict__ idx, int64_t nnz, const uint8_t* __restrict__ hot,
                                   int32_t* __restrict__ out) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t c = idx[p];
        out[p] = hot[c] ? c : static_cast<int32_t>(static_cast<uint32_t>(c) | 0x80000000u);
    }
}

void tag_hot_indices(const DevCsr& m, const int32_t* order_x, int64_t k, uint8_t* hot, int32_t* idx_tag,
                     cudaStream_t stream) {
    DSVD_CUDA_CHECK(cudaMemsetAsync(hot, 0, static_cast<size_t>(m.cols > 0 ? m.cols : 1), stream));
    k = std::min(k, m.cols);
    if (k > 0) {
        hot_flags_kernel<<<grid_for(k), 256, 0, stream>>>(order_x, k, hot);
        DSVD_LAUNCH_CHECK();
    }
    if (m.nnz > 0) {
        tag_indices_kernel<<<grid_for(m.nnz), 256, 0, stream>>>(m.idx, m.nnz, hot, idx_tag);
        DSVD_LAUNCH_CHECK();
    }
}

void to_slab_major(const double* src, int64_t rows, int64_t ld, int w, double* dst, cudaStream_t stream) {
    if (rows == 0 || ld == 0) return;
    slab_copy_kernel<true><<<grid_for(ceil_div(ld, w) * rows * (w / 4)), 256, 0, stream>>>(src, rows, ld, w, dst);
    DSVD_LAUNCH_CHECK();
}

void from_slab_major(const double* src, int64_t rows, int64_t ld, int w, double* dst, cudaStream_t stream) {
    if (rows == 0 || ld == 0) return;
    slab_copy_kernel<false><<<grid_for(ceil_div(ld, w) * rows * (w / 4)), 256, 0, stream>>>(src, rows, ld, w, dst);
    DSVD_LAUNCH_CHECK();
}

void prefix_row_bounds(const DevCsr& m, int64_t n, int64_t* d_beg, int64_t* d_end,
                       cudaStream_t stream) {
    if (n == 0) return;
    prefix_bounds_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, stream>>>(m.order, m.off, n,
                                                                                    d_beg, d_end);
    DSVD_LAUNCH_CHECK();
}

void narrow_indices(const int64_t* src, int32_t* dst, int64_t nnz, int64_t cols, int32_t* bad,
                    cudaStream_t stream) {
    if (nnz == 0) return;
    narrow_kernel<<<grid_for(nnz), 256, 0, stream>>>(src, dst, nnz, cols, bad);
    DSVD_LAUNCH_CHECK();
}

void widen_indices(const int32_t* src, int64_t* dst, int64_t nnz, cudaStream_t stream) {
    if (nnz == 0) return;
    widen_kernel<<<grid_for(nnz), 256, 0, stream>>>(src, dst, nnz);
    DSVD_LAUNCH_CHECK();
}

namespace {
__global__ void uniform_values_kernel(const double* __restrict__ val, int64_t nnz, int32_t* nonuniform,
                                      double* first) {
    const long long v0 = __double_as_longlong(val[0]);
    if (blockIdx.x == 0 && threadIdx.x == 0) *first = val[0];
    bool diff = false;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        diff |= __double_as_longlong(__ldg(val + i)) != v0;
    if (__any_sync(kFull, diff) && (threadIdx.x & 31) == 0) *nonuniform = 1;
}
}  // namespace

void check_uniform_values(const double* val, int64_t nnz, int32_t* nonuniform, double* first,
                          cudaStream_t stream) {
    if (nnz == 0) return;
    uniform_values_kernel<<<grid_for(nnz), 256, 0, stream>>>(val, nnz, nonuniform, first);
    DSVD_LAUNCH_CHECK();
}

void check_offsets(const int64_t* off, int64_t rows, int64_t nnz, int32_t* bad,
                   cudaStream_t stream) {
    check_offsets_kernel<<<grid_for(rows), 256, 0, stream>>>(off, rows, nnz, bad);
    DSVD_LAUNCH_CHECK();
}

size_t csc_scratch_bytes(int64_t rows, int64_t cols, int64_t nnz) {
    (void)rows;
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), nnz > 0 ? nnz : 1, 0,
                                    key_bits(cols));
    return 4 * align_up(sizeof(int32_t) * (nnz > 0 ? nnz : 1)) + align_up(temp);
}

void build_transpose(const DevCsr& a, DevCsr& at, void* scratch, size_t scratch_bytes,
                     cudaStream_t stream, cudaEvent_t values_ready) {
    at.rows = a.cols;
    at.cols = a.rows;
    at.nnz = a.nnz;
    const int64_t nnz = a.nnz;
    if (nnz == 0) {
        fill_i64_kernel<<<grid_for(at.rows + 1), 256, 0, stream>>>(at.off, at.rows + 1, 0);
        DSVD_LAUNCH_CHECK();
        return;
    }
    if (nnz > 0x7fffffffLL) fail(DSVD_UNSUPPORTED, "transpose: nnz >= 2^31 is not supported");
    char* p = static_cast<char*>(scratch);
    const size_t seg = align_up(sizeof(int32_t) * nnz);
    int32_t* row_of = reinterpret_cast<int32_t*>(p);
    int32_t* keys_out = reinterpret_cast<int32_t*>(p + seg);
    int32_t* perm_in = reinterpret_cast<int32_t*>(p + 2 * seg);
    int32_t* perm_out = reinterpret_cast<int32_t*>(p + 3 * seg);
    void* temp = p + 4 * seg;
    size_t temp_bytes = scratch_bytes - 4 * seg;

    expand_rows_kernel<<<grid_for(a.rows * 32), 256, 0, stream>>>(a.off, a.rows, row_of);
    DSVD_LAUNCH_CHECK();
    iota_kernel<<<grid_for(nnz), 256, 0, stream>>>(perm_in, nnz);
    DSVD_LAUNCH_CHECK();
    // LSD radix sort is stable: equal columns keep their CSR (row-major) order,
    // exactly the counting sort's placement.
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, a.idx, keys_out, perm_in,
                                                    perm_out, nnz, 0, key_bits(a.cols), stream));
    // the values may still be on their way from the host (upload_pair)
    if (values_ready != nullptr) DSVD_CUDA_CHECK(cudaStreamWaitEvent(stream, values_ready, 0));
    gather_transpose_kernel<<<grid_for(nnz), 256, 0, stream>>>(perm_out, row_of, a.val, at.idx,
                                                               at.val, nnz);
    DSVD_LAUNCH_CHECK();
    offsets_from_keys_kernel<<<grid_for(nnz), 256, 0, stream>>>(keys_out, nnz, at.rows, at.off);
    DSVD_LAUNCH_CHECK();
}

size_t order_scratch_bytes(int64_t rows) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairsDescending(
        nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
        static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
        rows > 0 ? rows : 1, 0, 32);
    return 3 * align_up(sizeof(int32_t) * (rows > 0 ? rows : 1)) + align_up(temp);
}

void build_row_order(DevCsr& m, void* scratch, size_t scratch_bytes, cudaStream_t stream) {
    if (m.rows == 0) return;
    char* p = static_cast<char*>(scratch);
    const size_t seg = align_up(sizeof(int32_t) * m.rows);
    int32_t* len = reinterpret_cast<int32_t*>(p);
    int32_t* len_sorted = reinterpret_cast<int32_t*>(p + seg);
    int32_t* ids = reinterpret_cast<int32_t*>(p + 2 * seg);
    void* temp = p + 3 * seg;
    size_t temp_bytes = scratch_bytes - 3 * seg;
    row_lengths_kernel<<<grid_for(m.rows), 256, 0, stream>>>(m.off, m.rows, len, ids);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, len, len_sorted,
                                                              ids, m.order, m.rows, 0, 32, stream));
    if (m.d_hub_rows != nullptr) {
        count_ge_kernel<<<1, 1, 0, stream>>>(len_sorted, m.rows,
                                             m.hub_threshold > 0 ? m.hub_threshold : (int64_t(1) << 40),
                                             m.d_hub_rows);
        DSVD_LAUNCH_CHECK();
    }
    if (m.d_nonempty != nullptr) {
        count_ge_kernel<<<1, 1, 0, stream>>>(len_sorted, m.rows, 1, m.d_nonempty);
        DSVD_LAUNCH_CHECK();
    }
    if (m.d_mid != nullptr) {
        count_ge_kernel<<<1, 1, 0, stream>>>(len_sorted, m.rows, kMidRow + 1, m.d_mid);
        DSVD_LAUNCH_CHECK();
    }
    if (m.d_long != nullptr) {
        count_ge_kernel<<<1, 1, 0, stream>>>(len_sorted, m.rows, kShortRow + 1, m.d_long);
        DSVD_LAUNCH_CHECK();
    }
    if (m.obeg != nullptr) {
        order_ranges_kernel<<<grid_for(m.rows), 256, 0, stream>>>(m.order, m.off, m.rows, m.obeg, m.olen);
        DSVD_LAUNCH_CHECK();
    }
}

namespace {
__global__ void row_flags_kernel(const int64_t* __restrict__ off, int64_t rows, int32_t* __restrict__ flag) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        flag[r] = off[r + 1] > off[r] ? 1 : 0;
}
__global__ void compact_place_kernel(const int64_t* __restrict__ off, int64_t rows, const int32_t* __restrict__ flag,
                                     const int32_t* __restrict__ pos, int32_t* __restrict__ newid,
                                     int32_t* __restrict__ oldid, int64_t* __restrict__ off_c) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (flag[r]) {
            const int32_t p = pos[r];
            newid[r] = p;
            oldid[p] = static_cast<int32_t>(r);
            off_c[p] = off[r];
        } else {
            newid[r] = -1;
        }
        if (r == rows - 1) off_c[pos[r] + flag[r]] = off[rows];
    }
}
__global__ void remap_ids_kernel(const int32_t* __restrict__ in, int64_t n, const int32_t* __restrict__ map,
                                 int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t v = map[in[i]];
        DSVD_DCHECK(v >= 0);
        out[i] = v;
    }
}
__global__ void scatter_rows_kernel(const double* __restrict__ src, int64_t rows_c, int64_t k,
                                    const int32_t* __restrict__ oldid, double* __restrict__ dst, int64_t rows) {
    const int64_t total = rows_c * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = e / rows_c, i = e - c * rows_c;
        dst[c * rows + oldid[i]] = src[e];
    }
}
}  // namespace

size_t compact_scratch_bytes(int64_t rows) {
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                  static_cast<int>(rows > 0 ? rows : 1));
    return 2 * align_up(sizeof(int32_t) * (rows > 0 ? rows : 1)) + align_up(temp);
}

void compact_rows_map(const int64_t* off, int64_t rows, int32_t* newid, int32_t* oldid, int64_t* off_c,
                      void* scratch, size_t scratch_bytes, cudaStream_t stream) {
    if (rows == 0) return;
    char* p = static_cast<char*>(scratch);
    const size_t seg = align_up(sizeof(int32_t) * rows);
    int32_t* flag = reinterpret_cast<int32_t*>(p);
    int32_t* pos = reinterpret_cast<int32_t*>(p + seg);
    size_t tb = scratch_bytes - 2 * seg;
    row_flags_kernel<<<grid_for(rows), 256, 0, stream>>>(off, rows, flag);
    DSVD_LAUNCH_CHECK();
    DSVD_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(p + 2 * seg, tb, flag, pos, static_cast<int>(rows), stream));
    compact_place_kernel<<<grid_for(rows), 256, 0, stream>>>(off, rows, flag, pos, newid, oldid, off_c);
    DSVD_LAUNCH_CHECK();
}

void remap_ids(const int32_t* in, int64_t n, const int32_t* map, int32_t* out, cudaStream_t stream) {
    if (n == 0) return;
    remap_ids_kernel<<<grid_for(n), 256, 0, stream>>>(in, n, map, out);
    DSVD_LAUNCH_CHECK();
}

void scatter_rows_colmajor(const double* src, int64_t rows_c, int64_t k, const int32_t* oldid, double* dst,
                           int64_t rows, cudaStream_t stream) {
    DSVD_CUDA_CHECK(cudaMemsetAsync(dst, 0, sizeof(double) * rows * k, stream));
    if (rows_c * k == 0) return;
    scatter_rows_kernel<<<grid_for(rows_c * k), 256, 0, stream>>>(src, rows_c, k, oldid, dst, rows);
    DSVD_LAUNCH_CHECK();
}

}  // namespace dsvd
