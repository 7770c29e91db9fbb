"""Python host mirror of the reference dashSVD interface, backed by the B200
C ABI (include/dashsvd_b200.h).

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/core/include/dashsvd/*.hpp):

=====================  ==========================================================
this module            reference
=====================  ==========================================================
SparseMatrix           sparse_matrix.hpp:14-36 (canonical CSR, int64 indices)
SolverConfig           solver.hpp:22-38
Algorithm, StopReason  solver.hpp:13-18, :45
TruncatedSvd           decompositions.hpp:11-17
ShiftTrace/SolveResult solver.hpp:51-61
IterationState         solver.hpp:63-72 (observer argument)
solve / dash_svd /     solver.hpp:90-116 (the `at` overloads accept and ignore a
shifted_rsvd           precomputed transpose: the device builds its own, bitwise)
finalize_row_basis     solver.hpp:123
validate_config,       solver.cpp:15-50
update_shift,
pve_stop_check
spmm, transpose        sparse_matrix.hpp:30-36
gram, matmul           dense_kernels.hpp:21-24
eig_svd, sym_eig       decompositions.hpp:28, sym_eig.hpp:20
gaussian_matrix,       random.hpp:11-20
splitmix64_at
sparse_random          synthetic.hpp:37-38
=====================  ==========================================================

Dense matrices are numpy arrays in column-major (Fortran) order, like the
reference's DenseMatrix. Every computation runs on the GPU through the native
library; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import errors as E
from ._native import (OBSERVER, dsvd_config, dsvd_outputs, dsvd_stats, check, lib)

_P = C.c_void_p
I64 = C.c_int64


def _path(path) -> bytes:
    return os.fsencode(path)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_P)


class Algorithm(enum.IntEnum):
    basic = 0
    shifted = 1
    fixed_shift = 2
    dash = 3


class StopReason(enum.IntEnum):
    fixed_p = 0
    tol_met = 1
    p_max_reached = 2


class Orthonormalizer(enum.IntEnum):
    eigsvd = 0
    qr = 1


@dataclass
class SparseMatrix:
    """Canonical CSR (sparse_matrix.hpp:10-26)."""
    rows: int
    cols: int
    offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def validate(self) -> None:
        """Canonical-form check on the host (sparse_matrix.cpp:12-33): ShapeError /
        NumericalError for the first violation in row order, as the reference's loop."""
        if self.rows < 0 or self.cols < 0:
            raise E.ShapeError("sparse matrix with negative dimension")
        if self.offsets.shape[0] != self.rows + 1:
            raise E.ShapeError("offset array must have rows+1 entries")
        if self.offsets[0] != 0 or self.offsets[-1] != self.nnz:
            raise E.ShapeError("offsets must span [0, nnz]")
        if self.col_indices.shape[0] != self.values.shape[0]:
            raise E.ShapeError("index/value length mismatch")
        off = self.offsets
        dec = np.flatnonzero(off[:-1] > off[1:])
        first_dec = int(dec[0]) if dec.size else self.rows
        # rows before the first decrease are contiguous from 0 (the loop reaches them first)
        end = int(min(max(off[first_dec], 0), self.nnz))
        ci, v = self.col_indices[:end], self.values[:end]
        row = np.repeat(np.arange(first_dec), np.diff(off[:first_dec + 1]))[:end]
        code = np.full(end, 5, dtype=np.int8)
        notinc = np.zeros(end, dtype=bool)
        if end > 1:
            notinc[1:] = (row[1:] == row[:-1]) & (ci[:-1] >= ci[1:])
        for c, bad in ((4, v == 0.0), (3, ~np.isfinite(v)), (2, notinc), (1, (ci < 0) | (ci >= self.cols))):
            code[bad] = c
        hit = np.flatnonzero(code < 5)
        if hit.size:
            p = int(hit[0])
            i, c = int(row[p]), int(code[p])
            if c == 1:
                raise E.ShapeError(f"column index out of range in row {i}")
            if c == 2:
                raise E.ShapeError(f"column indices not strictly increasing in row {i}")
            if c == 3:
                raise E.NumericalError(f"non-finite value in row {i}")
            raise E.NumericalError(f"explicit zero stored in row {i}")
        if dec.size:
            raise E.ShapeError("offsets must be non-decreasing")

    def validate_on_device(self, device: Optional["Device"] = None) -> None:
        """The same check run by the sm_100a library (dsvd_csr_validate)."""
        if self.offsets.shape[0] != self.rows + 1:
            raise E.ShapeError("offset array must have rows+1 entries")
        if self.col_indices.shape[0] != self.values.shape[0]:
            raise E.ShapeError("index/value length mismatch")
        check(lib().dsvd_csr_validate(_dev(device).handle, self.rows, self.cols, self.nnz, _ptr(self.offsets),
                                      _ptr(self.col_indices), _ptr(self.values)))


@dataclass
class SolverConfig:
    """solver.hpp:22-38."""
    k: int = 0
    s: int = -1
    p: int = -1
    tol: float = 1e-2
    p_max: int = 1000
    alg: Algorithm = Algorithm.dash
    orth: Orthonormalizer = Orthonormalizer.eigsvd
    seed: int = 0
    deterministic: bool = True

    def effective_s(self, k_: Optional[int] = None) -> int:
        k_ = self.k if k_ is None else k_
        return self.s if self.s >= 0 else (k_ // 2 if k_ // 2 > 0 else 1)

    def sketch_width(self) -> int:
        return self.k + self.effective_s(self.k)

    def _c(self, direct: bool = False) -> dsvd_config:
        flags = (1 if direct else 0) | (2 if self.orth == Orthonormalizer.qr else 0)  # DSVD_FLAG_*
        return dsvd_config(int(self.k), int(self.s), int(self.p), float(self.tol), int(self.p_max),
                           int(self.alg), flags, int(self.seed) & 0xFFFFFFFFFFFFFFFF)


@dataclass
class TruncatedSvd:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray

    def rank(self) -> int:
        return int(self.s.shape[0])


@dataclass
class ShiftTrace:
    alphas: List[float] = field(default_factory=list)
    s_hat_history: List[np.ndarray] = field(default_factory=list)
    iterations: int = 0
    stop_reason: StopReason = StopReason.fixed_p


@dataclass
class SolveResult:
    svd: TruncatedSvd
    trace: ShiftTrace
    stats: Optional[dict] = None


@dataclass
class IterationState:
    iteration: int
    alpha: float
    s_hat: np.ndarray
    q_before: np.ndarray
    q_after: np.ndarray


@dataclass
class EigenPair:
    values: np.ndarray
    vectors: np.ndarray


IterationObserver = Callable[[IterationState], None]


# ---- device context -----------------------------------------------------------

class Device:
    """One CUDA device context (stream + workspaces) of the native library."""

    def __init__(self, index: int = 0, profiling: bool = False):
        L = lib()
        h = _P()
        check(L.dsvd_ctx_create(int(index), C.byref(h)))
        self._h = h
        self.index = index
        if profiling:
            self.set_profiling(True)

    @classmethod
    def _adopt(cls, h, rows: int, cols: int, nnz: int, device: "Device") -> "DeviceMatrix":
        m = cls(None, device)
        m._h = h
        m.rows, m.cols, m.nnz = int(rows), int(cols), int(nnz)
        return m

    @classmethod
    def load_cache(cls, path: str, device: Optional[Device] = None, validate: bool = True) -> "DeviceMatrix":
        """load_cache (matrix_market.cpp:257-275) straight into HBM: the DSH1 file is read
        into pinned memory, validated on the device and built into the device pair."""
        dev = _dev(device)
        h, dims = _P(), (I64 * 3)()
        check(lib().dsvd_matrix_load_cache(dev.handle, _path(path), 1 if validate else 0, C.byref(h), dims))
        return cls._adopt(h, dims[0], dims[1], dims[2], dev)

    @classmethod
    def from_matrix_market(cls, path: str, device: Optional[Device] = None) -> "DeviceMatrix":
        """load_matrix_market (matrix_market.cpp:117-165) with the assembly on the device
        and the device pair built from it without a host round trip."""
        dev = _dev(device)
        dims = (I64 * 3)()
        check(lib().dsvd_mtx_assemble(dev.handle, _path(path), dims))
        h = _P()
        check(lib().dsvd_matrix_from_coo(dev.handle, C.byref(h)))
        return cls._adopt(h, dims[0], dims[1], dims[2], dev)

    @property
    def handle(self):
        return self._h

    def download(self) -> SparseMatrix:
        """CSR(A) back to the host (int64 indices)."""
        off = np.empty(self.rows + 1, dtype=np.int64)
        idx = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz, dtype=np.float64)
        check(lib().dsvd_matrix_download(self._h, _ptr(off), _ptr(idx), _ptr(val)))
        return SparseMatrix(self.rows, self.cols, off, idx, val)

    def set_profiling(self, on: bool) -> None:
        check(lib().dsvd_ctx_set_profiling(self._h, 1 if on else 0))

    def set_option(self, name: str, value: int) -> None:
        check(lib().dsvd_ctx_set_option(self._h, name.encode(), int(value)))

    def stats(self) -> dict:
        st = dsvd_stats()
        check(lib().dsvd_ctx_get_stats(self._h, C.byref(st)))
        return st.as_dict()

    def synchronize(self) -> None:
        check(lib().dsvd_ctx_synchronize(self._h))

    def trim(self) -> None:
        """Free the cached device workspaces (dsvd_ctx_trim)."""
        check(lib().dsvd_ctx_trim(self._h))

    def attach_comm(self, nranks: int, rank: int, unique_id: bytes) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(lib().dsvd_ctx_attach_comm(self._h, int(nranks), int(rank), buf))

    def attach_loopback(self, group: "LoopbackGroup", rank: int) -> None:
        """Join an in-process rank group (dsvd_ctx_attach_loopback): solves on this
        context then run the row-sharded engine as `rank` of `group.nranks`, with the
        collectives summed on the host side in rank order (testing without NCCL)."""
        check(lib().dsvd_ctx_attach_loopback(self._h, group.handle, int(rank)))
        group._members.append(self)

    def set_shard(self, row_offset: int, global_rows: int) -> None:
        """The CSR given to solve() is rows [row_offset, row_offset + rows) of a
        global_rows x cols matrix (row-sharded multi-GPU solve)."""
        check(lib().dsvd_ctx_set_shard(self._h, int(row_offset), int(global_rows)))

    def timer_start(self) -> None:
        check(lib().dsvd_ctx_timer_start(self._h))

    def timer_stop(self) -> float:
        """Milliseconds since timer_start, measured with CUDA events on the context's stream."""
        ms = C.c_double()
        check(lib().dsvd_ctx_timer_stop(self._h, C.byref(ms)))
        return float(ms.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().dsvd_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pin(arr: np.ndarray) -> np.ndarray:
    """Page-lock a numpy array's memory (cudaHostRegister) so host<->device
    copies of it run at full link speed. Returns the array."""
    if arr.nbytes:
        check(lib().dsvd_host_register(arr.ctypes.data_as(_P), arr.nbytes))
    return arr


def unpin(arr: np.ndarray) -> None:
    if arr.nbytes:
        check(lib().dsvd_host_unregister(arr.ctypes.data_as(_P)))


class LoopbackGroup:
    """In-process group of `nranks` contexts (one host thread each) standing in for
    an NCCL communicator, e.g. several ranks on one GPU (dsvd_loopback_create).
    Close (or drop) every member Device before the group."""

    def __init__(self, nranks: int):
        h = _P()
        check(lib().dsvd_loopback_create(int(nranks), C.byref(h)))
        self._h = h
        self.nranks = int(nranks)
        self._members = []

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        for dev in self._members:
            dev.close()
        self._members = []
        if self._h:
            check(lib().dsvd_loopback_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().dsvd_comm_unique_id(buf))
    return bytes(buf)


_default = threading.local()


def default_device() -> Device:
    dev = getattr(_default, "dev", None)
    if dev is None:
        dev = Device(0)
        _default.dev = dev
    return dev


def _dev(device: Optional[Device]) -> Device:
    return device if device is not None else default_device()


class DeviceMatrix:
    """Device-resident CSR(A) + CSR(A^T) (upload once, solve many)."""

    def __init__(self, a: Optional[SparseMatrix], device: Optional[Device] = None):
        self.device = _dev(device)
        if a is None:  # filled in by _adopt
            self._h = None
            return
        h = _P()
        check(lib().dsvd_matrix_upload(self.device.handle, a.rows, a.cols, a.nnz, _ptr(a.offsets),
                                       _ptr(a.col_indices), _ptr(a.values), C.byref(h)))
        self._h = h
        self.rows, self.cols, self.nnz = a.rows, a.cols, a.nnz

    @classmethod
    def _adopt(cls, h, rows: int, cols: int, nnz: int, device: "Device") -> "DeviceMatrix":
        m = cls(None, device)
        m._h = h
        m.rows, m.cols, m.nnz = int(rows), int(cols), int(nnz)
        return m

    @classmethod
    def load_cache(cls, path: str, device: Optional[Device] = None, validate: bool = True) -> "DeviceMatrix":
        """load_cache (matrix_market.cpp:257-275) straight into HBM: the DSH1 file is read
        into pinned memory, validated on the device and built into the device pair."""
        dev = _dev(device)
        h, dims = _P(), (I64 * 3)()
        check(lib().dsvd_matrix_load_cache(dev.handle, _path(path), 1 if validate else 0, C.byref(h), dims))
        return cls._adopt(h, dims[0], dims[1], dims[2], dev)

    @classmethod
    def from_matrix_market(cls, path: str, device: Optional[Device] = None) -> "DeviceMatrix":
        """load_matrix_market (matrix_market.cpp:117-165) with the assembly on the device
        and the device pair built from it without a host round trip."""
        dev = _dev(device)
        dims = (I64 * 3)()
        check(lib().dsvd_mtx_assemble(dev.handle, _path(path), dims))
        h = _P()
        check(lib().dsvd_matrix_from_coo(dev.handle, C.byref(h)))
        return cls._adopt(h, dims[0], dims[1], dims[2], dev)

    @property
    def handle(self):
        return self._h

    def download(self) -> SparseMatrix:
        """CSR(A) back to the host (int64 indices)."""
        off = np.empty(self.rows + 1, dtype=np.int64)
        idx = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz, dtype=np.float64)
        check(lib().dsvd_matrix_download(self._h, _ptr(off), _ptr(idx), _ptr(val)))
        return SparseMatrix(self.rows, self.cols, off, idx, val)

    def download_rows(self, r0: int, r1: int) -> SparseMatrix:
        """Rows [r0, r1) of CSR(A) as a standalone host CSR (e.g. one rank's shard)."""
        offs = self.row_offsets()
        n = int(offs[r1] - offs[r0])
        off = np.empty(r1 - r0 + 1, dtype=np.int64)
        idx = np.empty(n, dtype=np.int64)
        val = np.empty(n, dtype=np.float64)
        check(lib().dsvd_matrix_download_rows(self._h, int(r0), int(r1), _ptr(off), _ptr(idx), _ptr(val)))
        return SparseMatrix(r1 - r0, self.cols, off, idx, val)

    def row_offsets(self) -> np.ndarray:
        off = np.empty(self.rows + 1, dtype=np.int64)
        check(lib().dsvd_matrix_row_offsets(self._h, _ptr(off)))
        return off

    def set_shard(self, row_offset: int, global_rows: int) -> None:
        check(lib().dsvd_matrix_set_shard(self._h, int(row_offset), int(global_rows)))

    def bench_spmm(self, transpose: bool, l: int, variant: int = 0, iters: int = 5) -> float:
        """Average ms of one SpMM launch on a random l-column block (see header)."""
        ms = C.c_double()
        check(lib().dsvd_matrix_bench_spmm(self._h, 1 if transpose else 0, int(l), int(variant),
                                           int(iters), C.byref(ms)))
        return float(ms.value)

    def hub_rows(self):
        a, t = C.c_int64(), C.c_int64()
        check(lib().dsvd_matrix_hub_rows(self._h, C.byref(a), C.byref(t)))
        return int(a.value), int(t.value)

    def transpose(self) -> SparseMatrix:
        off = np.empty(self.cols + 1, dtype=np.int64)
        idx = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz, dtype=np.float64)
        check(lib().dsvd_matrix_download_transpose(self._h, _ptr(off), _ptr(idx), _ptr(val)))
        return SparseMatrix(self.cols, self.rows, off, idx, val)

    def solve(self, cfg: SolverConfig, observer: Optional[IterationObserver] = None,
              out_rows: Optional[int] = None) -> SolveResult:
        return _solve_handle(self, cfg, observer, out_rows)

    def close(self):
        if getattr(self, "_h", None):
            lib().dsvd_matrix_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _trace_cap(cfg: SolverConfig) -> int:
    return max(1, (cfg.p_max if cfg.alg == Algorithm.dash else max(cfg.p, 0)))


def _make_outputs(rows, cols, cfg, out=None):
    k, l = cfg.k, cfg.sketch_width()
    cap = _trace_cap(cfg)
    if out is not None:  # caller-provided (e.g. pinned) buffers
        u, s, v = out
        if any(not isinstance(b, np.ndarray) or b.dtype != np.float64 for b in (u, s, v)):
            raise E.ConfigError("out: u, s and v must be float64 numpy arrays")
        if any(not b.flags.writeable for b in (u, s, v)):
            raise E.ConfigError("out: u, s and v must be writeable")
        if u.shape != (rows, k) or v.shape != (cols, k) or s.shape != (k,) or \
                not u.flags.f_contiguous or not v.flags.f_contiguous or not s.flags.c_contiguous:
            raise E.ShapeError("out: expected Fortran-ordered u (rows x k), v (cols x k), contiguous s (k)")
    else:
        u = np.empty((rows, k), dtype=np.float64, order="F")
        s = np.empty(k, dtype=np.float64)
        v = np.empty((cols, k), dtype=np.float64, order="F")
    alphas = np.zeros(cap)
    s_hat = np.zeros((cap, l))
    out = dsvd_outputs(_ptr(u).value, _ptr(s).value, _ptr(v).value, _ptr(alphas).value,
                       _ptr(s_hat).value, cap, 0, 0, 0)
    return out, (u, s, v, alphas, s_hat)


def _result(out, bufs, device: Device, cfg: Optional[SolverConfig] = None) -> SolveResult:
    u, s, v, alphas, s_hat = bufs
    n = int(out.iterations)
    # the qr orthonormalizer produces no surrogate spectrum: empty entries (solver.cpp:121-126)
    no_spec = cfg is not None and cfg.alg == Algorithm.basic and cfg.orth == Orthonormalizer.qr
    hist = [np.empty(0) if no_spec else s_hat[c].copy() for c in range(n)]
    trace = ShiftTrace([float(a) for a in alphas[:n]], hist, n, StopReason(int(out.stop_reason)))
    return SolveResult(TruncatedSvd(u, s, v), trace, device.stats())


def _observer_cb(observer: Optional[IterationObserver]):
    if observer is None:
        return OBSERVER(0), None
    errs = []

    def cb(it, alpha, s_hat, l, qb, qa, n, _user):
        try:
            sh = np.ctypeslib.as_array(s_hat, (l,)).copy()
            qbefore = np.ctypeslib.as_array(qb, (l * n,)).reshape((n, l), order="F").copy()
            qafter = np.ctypeslib.as_array(qa, (l * n,)).reshape((n, l), order="F").copy()
            observer(IterationState(int(it), float(alpha), sh, qbefore, qafter))
        except BaseException as exc:  # surfaced after the native call returns
            errs.append(exc)

    return OBSERVER(cb), errs


def _solve_handle(m: DeviceMatrix, cfg: SolverConfig, observer, out_rows=None,
                  direct: bool = False) -> SolveResult:
    if cfg.orth != Orthonormalizer.eigsvd and cfg.alg != Algorithm.basic:
        raise E.ConfigError("the qr orthonormalizer applies to the basic algorithm only; "
                            "shifted iterations need the surrogate spectrum")
    rows = m.rows if out_rows is None else out_rows
    out, bufs = _make_outputs(rows, m.cols, cfg)
    cb, errs = _observer_cb(observer)
    c = cfg._c(direct)
    check(lib().dsvd_solve(m.device.handle, m.handle, C.byref(c), C.byref(out), cb, None))
    if errs:
        raise errs[0]
    return _result(out, bufs, m.device, cfg)


# ---- reference-shaped entry points ---------------------------------------------

def validate_config(cfg: SolverConfig, rows: int, cols: int) -> None:
    """solver.cpp:15-32."""
    c = cfg._c()
    check(lib().dsvd_validate_config(C.byref(c), int(rows), int(cols)))
    if cfg.orth == Orthonormalizer.qr and cfg.alg != Algorithm.basic:
        raise E.ConfigError("the qr orthonormalizer applies to the basic algorithm only; "
                            "shifted iterations need the surrogate spectrum")


def update_shift(alpha: float, s_ll: float) -> float:
    """solver.cpp:34-36."""
    return float(lib().dsvd_update_shift(float(alpha), float(s_ll)))


def pve_stop_check(s_hat_prev, alpha_prev, s_hat, alpha, k, tol) -> bool:
    """solver.cpp:38-50."""
    a = np.ascontiguousarray(s_hat_prev, dtype=np.float64)
    b = np.ascontiguousarray(s_hat, dtype=np.float64)
    stop = C.c_int()
    check(lib().dsvd_pve_stop_check(_ptr(a), a.size, float(alpha_prev), _ptr(b), b.size,
                                    float(alpha), int(k), float(tol), C.byref(stop)))
    return bool(stop.value)


def solve(a: SparseMatrix, cfg: SolverConfig, at: Optional[SparseMatrix] = None,
          observer: Optional[IterationObserver] = None,
          device: Optional[Device] = None, _direct: bool = False, out=None) -> SolveResult:
    """solve(a, cfg) / solve(a, at, cfg, observer) (solver.cpp:214-227).

    `out` = (u, s, v) optionally supplies the result buffers (Fortran order),
    e.g. page-locked ones registered with `pin()`, for full-speed D2H."""
    dev = _dev(device)
    if cfg.orth != Orthonormalizer.eigsvd:
        validate_config(cfg, a.rows, a.cols)
    if observer is None:
        out, bufs = _make_outputs(a.rows, a.cols, cfg, out)
        c = cfg._c(_direct)
        check(lib().dsvd_solve_csr(dev.handle, a.rows, a.cols, a.nnz, _ptr(a.offsets),
                                   _ptr(a.col_indices), _ptr(a.values), C.byref(c), C.byref(out)))
        return _result(out, bufs, dev, cfg)
    validate_config(cfg, a.rows, a.cols)
    m = DeviceMatrix(a, dev)
    try:
        return _solve_handle(m, cfg, observer, direct=_direct)
    finally:
        m.close()


def shifted_rsvd(a: SparseMatrix, cfg: SolverConfig, at: Optional[SparseMatrix] = None,
                 observer: Optional[IterationObserver] = None,
                 device: Optional[Device] = None) -> SolveResult:
    """Fixed power count (solver.cpp:190-200): alg forced to shifted unless fixed_shift.
    Runs on `a` as given (no orientation swap), like the reference."""
    c = SolverConfig(**{**cfg.__dict__})
    if c.alg != Algorithm.fixed_shift:
        c.alg = Algorithm.shifted
    return _direct(a, c, observer, device)


def dash_svd(a: SparseMatrix, cfg: SolverConfig, at: Optional[SparseMatrix] = None,
             observer: Optional[IterationObserver] = None,
             device: Optional[Device] = None) -> SolveResult:
    """Accuracy-controlled run (solver.cpp:202-212)."""
    c = SolverConfig(**{**cfg.__dict__})
    c.alg = Algorithm.dash
    return _direct(a, c, observer, device)


def _direct(a, cfg, observer, device):
    # shifted_rsvd / dash_svd call solve_direct on `a` without the orientation
    # swap (solver.cpp:195, :207)
    validate_config(cfg, a.rows, a.cols)
    return solve(a, cfg, observer=observer, device=device, _direct=True)


def basic_rsvd(a: SparseMatrix, cfg: SolverConfig, at: Optional[SparseMatrix] = None,
               observer: Optional[IterationObserver] = None,
               device: Optional[Device] = None) -> TruncatedSvd:
    """Plain randomized subspace iteration, Alg. 1 (solver.cpp:178-188): alg forced
    to basic, run on `a` as given; returns the TruncatedSvd like the reference."""
    c = SolverConfig(**{**cfg.__dict__})
    c.alg = Algorithm.basic
    return _direct(a, c, observer, device).svd


def finalize_row_basis(a: SparseMatrix, q: np.ndarray, k: int,
                       device: Optional[Device] = None) -> TruncatedSvd:
    """solver.cpp:159-164."""
    q = np.asfortranarray(q, dtype=np.float64)
    if q.shape[0] != a.cols:
        raise E.ShapeError("finalize_row_basis: basis does not match matrix")
    l = q.shape[1]
    if k < 1 or k > l:
        raise E.ShapeError("finalize_row_basis: k out of range")
    dev = _dev(device)
    m = DeviceMatrix(a, dev)
    try:
        u = np.empty((a.rows, k), order="F")
        s = np.empty(k)
        v = np.empty((a.cols, k), order="F")
        check(lib().dsvd_finalize_row_basis(dev.handle, m.handle, _ptr(q), l, k, _ptr(u), _ptr(s),
                                            _ptr(v)))
        return TruncatedSvd(u, s, v)
    finally:
        m.close()


# ---- kernel-level entry points --------------------------------------------------

def spmm(a: SparseMatrix, x: np.ndarray, device: Optional[Device] = None) -> np.ndarray:
    """Y = A X (sparse_matrix.cpp:61-86), bitwise equal to the reference."""
    x = np.asfortranarray(x, dtype=np.float64)
    if a.cols != x.shape[0]:
        raise E.ShapeError("spmm: inner dimensions differ")
    l = x.shape[1]
    y = np.empty((a.rows, l), order="F")
    dev = _dev(device)
    check(lib().dsvd_spmm(dev.handle, a.rows, a.cols, a.nnz, _ptr(a.offsets), _ptr(a.col_indices),
                          _ptr(a.values), _ptr(x), l, _ptr(y)))
    return y


def spmm_shift(a: SparseMatrix, y: np.ndarray, alpha: float, q: np.ndarray,
               device: Optional[Device] = None) -> np.ndarray:
    """T = A Y, then T += (-alpha) Q unless alpha == 0 (solver.cpp:93-94), fused."""
    y = np.asfortranarray(y, dtype=np.float64)
    q = np.asfortranarray(q, dtype=np.float64)
    if a.cols != y.shape[0] or q.shape != (a.rows, y.shape[1]):
        raise E.ShapeError("spmm_shift: shapes differ")
    l = y.shape[1]
    t = np.empty((a.rows, l), order="F")
    dev = _dev(device)
    check(lib().dsvd_spmm_shift(dev.handle, a.rows, a.cols, a.nnz, _ptr(a.offsets),
                                _ptr(a.col_indices), _ptr(a.values), _ptr(y), l, float(alpha),
                                _ptr(q), _ptr(t)))
    return t


def transpose(a: SparseMatrix, device: Optional[Device] = None) -> SparseMatrix:
    """sparse_matrix.cpp:35-55, bitwise."""
    off = np.empty(a.cols + 1, dtype=np.int64)
    idx = np.empty(a.nnz, dtype=np.int64)
    val = np.empty(a.nnz, dtype=np.float64)
    dev = _dev(device)
    check(lib().dsvd_transpose(dev.handle, a.rows, a.cols, a.nnz, _ptr(a.offsets),
                               _ptr(a.col_indices), _ptr(a.values), _ptr(off), _ptr(idx), _ptr(val)))
    return SparseMatrix(a.cols, a.rows, off, idx, val)


def gram(c: np.ndarray, device: Optional[Device] = None) -> np.ndarray:
    c = np.asfortranarray(c, dtype=np.float64)
    g = np.empty((c.shape[1], c.shape[1]), order="F")
    dev = _dev(device)
    check(lib().dsvd_gram(dev.handle, c.shape[0], c.shape[1], _ptr(c), _ptr(g)))
    return g


def matmul(a: np.ndarray, b: np.ndarray, device: Optional[Device] = None) -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    if a.shape[1] != b.shape[0]:
        raise E.ShapeError("matmul: inner dimensions differ")
    c = np.empty((a.shape[0], b.shape[1]), order="F")
    dev = _dev(device)
    check(lib().dsvd_matmul(dev.handle, a.shape[0], a.shape[1], b.shape[1], _ptr(a), _ptr(b),
                            _ptr(c)))
    return c


def sym_eig(g: np.ndarray, device: Optional[Device] = None) -> EigenPair:
    g = np.asfortranarray(g, dtype=np.float64)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise E.ShapeError("sym_eig: matrix is not square")
    n = g.shape[0]
    w = np.empty(n)
    v = np.empty((n, n), order="F")
    dev = _dev(device)
    check(lib().dsvd_sym_eig(dev.handle, n, _ptr(g), _ptr(w), _ptr(v)))
    return EigenPair(w, v)


def eig_svd(c: np.ndarray, device: Optional[Device] = None) -> TruncatedSvd:
    c = np.asfortranarray(c, dtype=np.float64)
    m, n = c.shape
    u = np.empty((m, n), order="F")
    s = np.empty(n)
    v = np.empty((n, n), order="F")
    dev = _dev(device)
    check(lib().dsvd_eig_svd(dev.handle, m, n, _ptr(c), _ptr(u), _ptr(s), _ptr(v)))
    return TruncatedSvd(u, s, v)


def gaussian_matrix(rows: int, cols: int, seed: int, device: Optional[Device] = None) -> np.ndarray:
    out = np.empty((rows, cols), order="F")
    dev = _dev(device)
    check(lib().dsvd_gaussian_matrix(dev.handle, int(rows), int(cols),
                                     int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(out)))
    return out


def gaussian_rows(rows: int, cols: int, seed: int, global_rows: int, row_offset: int,
                  device: Optional[Device] = None) -> np.ndarray:
    """Rows [row_offset, row_offset + rows) of gaussian_matrix(global_rows, cols, seed): the
    sketch block Omega_g a row shard generates locally (random.cpp:29-36)."""
    out = np.empty((rows, cols), order="F")
    dev = _dev(device)
    check(lib().dsvd_gaussian_rows(dev.handle, int(rows), int(cols), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                   int(global_rows), int(row_offset), _ptr(out)))
    return out


def splitmix64_at(seed: int, i: int) -> int:
    return int(lib().dsvd_splitmix64_at(int(seed) & 0xFFFFFFFFFFFFFFFF, int(i) & 0xFFFFFFFFFFFFFFFF))


# ---- synthetic inputs (host generators in the native library) ---------------------

def _fetch(rows, cols, nnz) -> SparseMatrix:
    off = np.empty(rows + 1, dtype=np.int64)
    idx = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    check(lib().dsvd_synth_fetch(_ptr(off), _ptr(idx), _ptr(val)))
    return SparseMatrix(rows, cols, off, idx, val)


def sparse_random(rows: int, cols: int, nnz_per_row: int, seed: int,
                  row_decay: bool = False) -> SparseMatrix:
    """synthetic.cpp:72-120 (config 1's generator), same bits as the reference."""
    nnz = C.c_int64()
    check(lib().dsvd_synth_sparse_random(rows, cols, nnz_per_row, seed, 1 if row_decay else 0,
                                         C.byref(nnz)))
    return _fetch(rows, cols, nnz.value)


def powerlaw(rows: int, cols: int, mu: float, sigma: float, zipf_s: float, seed: int,
             ratings: bool = False) -> SparseMatrix:
    """BASELINE.json configs 2/3: lognormal row degrees, Zipf columns, no duplicates."""
    nnz = C.c_int64()
    check(lib().dsvd_synth_powerlaw(rows, cols, mu, sigma, zipf_s, 1 if ratings else 0, seed,
                                    C.byref(nnz)))
    return _fetch(rows, cols, nnz.value)


def rmat(scale: int, draws: int, a: float = 0.57, b: float = 0.19, c: float = 0.19, uniform_values: bool = False,
         seed: int = 0, device: Optional[Device] = None) -> "DeviceMatrix":
    """R-MAT graph generated on the device (BASELINE.json configs 4/5), returned as a device
    matrix (DeviceMatrix.download() for the host CSR). See dsvd_synth_rmat for the rule."""
    dev = _dev(device)
    h, nnz = _P(), I64()
    check(lib().dsvd_synth_rmat(dev.handle, int(scale), int(draws), float(a), float(b), float(c),
                                1 if uniform_values else 0, int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(h), C.byref(nnz)))
    n = 1 << int(scale)
    return DeviceMatrix._adopt(h, n, n, nnz.value, dev)


def solve_device_csr(rows: int, cols: int, nnz: int, d_offsets: int, d_col_indices: int,
                     d_values: int, cfg: SolverConfig, d_u: int, d_s: int, d_v: int,
                     device: Optional[Device] = None) -> SolveResult:
    """solve(a, cfg) with the CSR (int64 offsets / int64 indices / fp64 values)
    and the U/S/V outputs already in device memory on `device` (raw pointers,
    e.g. torch CUDA tensors' data_ptr()). Trace arrays come back on the host."""
    dev = _dev(device)
    cap = _trace_cap(cfg)
    alphas = np.zeros(cap)
    s_hat = np.zeros((cap, cfg.sketch_width()))
    out = dsvd_outputs(int(d_u), int(d_s), int(d_v), _ptr(alphas).value, _ptr(s_hat).value, cap,
                       0, 0, 1)
    c = cfg._c()
    check(lib().dsvd_solve_csr_device(dev.handle, int(rows), int(cols), int(nnz), _P(d_offsets),
                                      _P(d_col_indices), _P(d_values), C.byref(c), C.byref(out)))
    n = int(out.iterations)
    trace = ShiftTrace([float(a) for a in alphas[:n]], [s_hat[i].copy() for i in range(n)], n,
                       StopReason(int(out.stop_reason)))
    return SolveResult(None, trace, dev.stats())


# ---- validation metrics (metrics.hpp) ----------------------------

def _metric_matrix(a, device):
    """A DeviceMatrix for `a` (uploaded when a SparseMatrix is given) and whether we own it."""
    if isinstance(a, DeviceMatrix):
        return a, False
    return DeviceMatrix(a, _dev(device)), True


def _metric_call(a, device, fn, *args):
    m, own = _metric_matrix(a, device)
    try:
        out = C.c_double()
        check(fn(m.device.handle, m.handle, *args, C.byref(out)))
        return float(out.value)
    finally:
        if own:
            m.close()


def _sig(ref):
    return np.ascontiguousarray(getattr(ref, "sigmas", ref), dtype=np.float64)


def eps_pve(a, u_hat: np.ndarray, ref, device: Optional[Device] = None) -> float:
    """metrics.cpp:99-117 on the device: max_i |sigma_i^2 - ||A^T u_i||^2| / sigma_{k+1}^2."""
    u = np.asfortranarray(u_hat, dtype=np.float64)
    sg = _sig(ref)
    return _metric_call(a, device, lib().dsvd_eps_pve, _ptr(u), u.shape[1], _ptr(sg), sg.size)


def eps_res(a, approx: TruncatedSvd, ref, device: Optional[Device] = None) -> float:
    """metrics.cpp:119-134: max_i ||A^T u_i - s_i v_i|| / sigma_i."""
    u, v = np.asfortranarray(approx.u, dtype=np.float64), np.asfortranarray(approx.v, dtype=np.float64)
    s = np.ascontiguousarray(approx.s, dtype=np.float64)
    sg = _sig(ref)
    return _metric_call(a, device, lib().dsvd_eps_res, _ptr(u), _ptr(s), _ptr(v), s.size, _ptr(sg), sg.size)


def eps_spec(a, approx: TruncatedSvd, ref, power_iters: int = 300, seed: int = 0x5EED,
             device: Optional[Device] = None) -> float:
    """metrics.cpp:136-159: (||A - U S V^T||_2 estimate - sigma_{k+1}) / sigma_{k+1}, the norm by
    power iteration on the matrix-free residual operator."""
    u, v = np.asfortranarray(approx.u, dtype=np.float64), np.asfortranarray(approx.v, dtype=np.float64)
    s = np.ascontiguousarray(approx.s, dtype=np.float64)
    sg = _sig(ref)
    return _metric_call(a, device, lib().dsvd_eps_spec, _ptr(u), _ptr(s), _ptr(v), s.size, _ptr(sg), sg.size,
                        int(power_iters), int(seed) & 0xFFFFFFFFFFFFFFFF)


def max_triplet_residual(a, approx: TruncatedSvd, device: Optional[Device] = None) -> float:
    """metrics.cpp:194-206: max_i ||A v_i - s_i u_i||."""
    u, v = np.asfortranarray(approx.u, dtype=np.float64), np.asfortranarray(approx.v, dtype=np.float64)
    s = np.ascontiguousarray(approx.s, dtype=np.float64)
    return _metric_call(a, device, lib().dsvd_max_triplet_residual, _ptr(u), _ptr(s), _ptr(v), s.size)


# ---- inputs: DSH1 cache, Matrix Market, COO assembly -----------

def _fetch_coo(dev: Device, rows: int, cols: int, nnz: int) -> SparseMatrix:
    off = np.empty(rows + 1, dtype=np.int64)
    idx = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    check(lib().dsvd_coo_fetch(dev.handle, _ptr(off), _ptr(idx), _ptr(val)))
    return SparseMatrix(rows, cols, off, idx, val)


def assemble(rows: int, cols: int, r, c, v, device: Optional[Device] = None) -> SparseMatrix:
    """assemble (matrix_market.cpp:90-115) on the device: triplets sorted by (row, col),
    duplicates summed, exact zeros dropped. 0-based coordinates."""
    dev = _dev(device)
    r = np.ascontiguousarray(r, dtype=np.int64)
    c = np.ascontiguousarray(c, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if not (r.shape == c.shape == v.shape):
        raise E.ShapeError("triplet arrays differ in length")
    nnz = I64()
    check(lib().dsvd_coo_assemble(dev.handle, int(rows), int(cols), r.size, _ptr(r), _ptr(c), _ptr(v),
                                  C.byref(nnz)))
    return _fetch_coo(dev, int(rows), int(cols), int(nnz.value))


def load_matrix_market(path: str, device: Optional[Device] = None) -> SparseMatrix:
    """load_matrix_market (matrix_market.cpp:117-165): parsed on the host, assembled on the
    device, returned as a host CSR (DeviceMatrix.from_matrix_market keeps it in HBM)."""
    dev = _dev(device)
    dims = (I64 * 3)()
    check(lib().dsvd_mtx_assemble(dev.handle, _path(path), dims))
    return _fetch_coo(dev, dims[0], dims[1], dims[2])


def read_matrix_market_triplets(path: str):
    """The host parsing half of load_matrix_market (matrix_market.cpp:117-163): returns
    (rows, cols, r, c, v), 0-based triplets in file order after the symmetric expansion,
    before assembly. Raises ParseError / UnsupportedFormat / Error like the reference."""
    dims = (I64 * 3)()
    check(lib().dsvd_mtx_read(_path(path), dims))
    n = int(dims[2])
    r = np.empty(n, dtype=np.int64)
    c = np.empty(n, dtype=np.int64)
    v = np.empty(n, dtype=np.float64)
    check(lib().dsvd_mtx_fetch(_ptr(r), _ptr(c), _ptr(v)))
    return int(dims[0]), int(dims[1]), r, c, v


def write_matrix_market(path: str, a: SparseMatrix) -> None:
    """write_matrix_market (matrix_market.cpp:167-177)."""
    check(lib().dsvd_write_matrix_market(_path(path), a.rows, a.cols, _ptr(a.offsets), _ptr(a.col_indices),
                                         _ptr(a.values)))


def save_cache(path: str, a: SparseMatrix) -> None:
    """save_cache (matrix_market.cpp:241-253): DSH1 binary CSR."""
    check(lib().dsvd_save_cache(_path(path), a.rows, a.cols, a.nnz, _ptr(a.offsets), _ptr(a.col_indices),
                                _ptr(a.values)))


def load_cache(path: str, device: Optional[Device] = None) -> SparseMatrix:
    """load_cache (matrix_market.cpp:255-275): read, validated on the device, returned on
    the host. DeviceMatrix.load_cache keeps the matrix in HBM instead."""
    m = DeviceMatrix.load_cache(path, device, validate=True)
    try:
        return m.download()
    finally:
        m.close()


def load_dense_array(path: str) -> np.ndarray:
    """load_dense_array (matrix_market.cpp:179-213): column-major rows x cols array."""
    dims = (I64 * 2)()
    check(lib().dsvd_dense_read(_path(path), dims))
    out = np.empty((dims[0], dims[1]), order="F")
    check(lib().dsvd_dense_fetch(_ptr(out)))
    return out


def write_dense_array(path: str, a: np.ndarray) -> None:
    """write_dense_array (matrix_market.cpp:215-223)."""
    a = np.asfortranarray(a, dtype=np.float64)
    check(lib().dsvd_dense_write(_path(path), a.shape[0], a.shape[1], _ptr(a)))


def load_reference_spectrum(path: str) -> np.ndarray:
    """load_reference_spectrum (metrics.cpp:71-90): descending singular values."""
    n = I64()
    check(lib().dsvd_spectrum_read(_path(path), C.byref(n)))
    out = np.empty(n.value)
    check(lib().dsvd_spectrum_fetch(_ptr(out)))
    return out


def write_reference_spectrum(path: str, sigmas) -> None:
    """write_reference_spectrum (metrics.cpp:92-97)."""
    s = np.ascontiguousarray(sigmas, dtype=np.float64)
    check(lib().dsvd_spectrum_write(_path(path), _ptr(s), s.size))


def eps_sigma(s_hat, ref) -> float:
    """metrics.cpp:160-170: worst relative error of the leading k singular values."""
    s_hat = np.asarray(s_hat, dtype=np.float64)
    sg = _sig(ref)
    k = s_hat.size
    if k < 1:
        raise E.ShapeError("eps_sigma: no singular values supplied")
    if sg.size < k:
        raise E.DegenerateReference(f"reference provides {sg.size} singular values, need {k}")
    worst = 0.0
    for i in range(k):
        if sg[i] == 0.0:
            raise E.DegenerateReference("sigma_i is zero")
        worst = max(worst, abs(sg[i] - s_hat[i]) / sg[i])
    return worst
