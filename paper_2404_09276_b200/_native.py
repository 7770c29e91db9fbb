"""ctypes binding of the C ABI in include/dashsvd_b200.h.

The shared library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2404_09276_b200/csrc``) to
``paper_2404_09276_b200/_lib/libdashsvd_b200.so``. There is no CPU fallback:
if the library is missing, every entry point raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

# DSVD_CHECKED=1 selects the bounds-checked build (make -C paper_2404_09276_b200/csrc checked:
# device-side index assertions that trap on a violation; compute-sanitizer is not available
# on the GPU pool)
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "_lib_checked" if os.environ.get("DSVD_CHECKED") == "1" else "_lib", "libdashsvd_b200.so")

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double
U64 = C.c_uint64

DSVD_OK, DSVD_SHAPE, DSVD_CONFIG, DSVD_RANK, DSVD_NUMERICAL = 0, 1, 2, 3, 4
DSVD_CUDA, DSVD_OOM, DSVD_NCCL, DSVD_UNSUPPORTED, DSVD_OTHER = 5, 6, 7, 8, 9
DSVD_DEGENERATE, DSVD_FORMAT, DSVD_PARSE = 10, 11, 12


class NativeLibraryMissing(E.Error):
    """The sm_100a extension is not built; there is deliberately no fallback."""


class dsvd_config(C.Structure):
    _fields_ = [("k", I64), ("s", I64), ("p", I64), ("tol", D), ("p_max", I64), ("alg", I32),
                ("flags", I32), ("seed", U64)]


class dsvd_outputs(C.Structure):
    _fields_ = [("u", P), ("s", P), ("v", P), ("alphas", P), ("s_hat", P), ("trace_cap", I64),
                ("iterations", I64), ("stop_reason", I32), ("outputs_on_device", I32)]


class dsvd_stats(C.Structure):
    _fields_ = [("total_ms", D), ("h2d_ms", D), ("csc_ms", D), ("omega_ms", D), ("sketch_ms", D),
                ("loop_ms", D), ("finalize_ms", D), ("d2h_ms", D), ("spmm_ms", D), ("gram_ms", D),
                ("eig_ms", D), ("rescale_ms", D), ("allreduce_ms", D), ("spmm_launches", I64),
                ("kernel_launches", I64), ("eig_sweeps", I64), ("spmm_bytes", I64),
                ("spmm_pass_ms", D * 2), ("spmm_pass_bytes", I64 * 2),
                ("spmm_pass_launches", I64 * 2), ("pipelined", I64)]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out


OBSERVER = C.CFUNCTYPE(None, I64, D, C.POINTER(D), I64, C.POINTER(D), C.POINTER(D), I64, P)

# (name, restype, argtypes) for every exported entry point of dashsvd_b200.h
SIGNATURES = [
    ("dsvd_last_error", C.c_char_p, []),
    ("dsvd_last_error_index", C.c_longlong, []),
    ("dsvd_version", C.c_char_p, []),
    ("dsvd_ctx_create", C.c_int, [C.c_int, C.POINTER(P)]),
    ("dsvd_ctx_destroy", C.c_int, [P]),
    ("dsvd_ctx_set_profiling", C.c_int, [P, C.c_int]),
    ("dsvd_ctx_get_stats", C.c_int, [P, C.POINTER(dsvd_stats)]),
    ("dsvd_ctx_synchronize", C.c_int, [P]),
    ("dsvd_ctx_trim", C.c_int, [P]),
    ("dsvd_ctx_set_option", C.c_int, [P, C.c_char_p, I64]),
    ("dsvd_comm_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("dsvd_ctx_attach_comm", C.c_int, [P, C.c_int, C.c_int, C.POINTER(C.c_uint8)]),
    ("dsvd_ctx_set_shard", C.c_int, [P, I64, I64]),
    ("dsvd_loopback_create", C.c_int, [C.c_int, C.POINTER(P)]),
    ("dsvd_loopback_destroy", C.c_int, [P]),
    ("dsvd_ctx_attach_loopback", C.c_int, [P, P, C.c_int]),
    ("dsvd_host_register", C.c_int, [P, C.c_size_t]),
    ("dsvd_host_unregister", C.c_int, [P]),
    ("dsvd_matrix_upload", C.c_int, [P, I64, I64, I64, P, P, P, C.POINTER(P)]),
    ("dsvd_matrix_from_device", C.c_int, [P, I64, I64, I64, P, P, P, C.POINTER(P)]),
    ("dsvd_matrix_destroy", C.c_int, [P]),
    ("dsvd_matrix_set_shard", C.c_int, [P, I64, I64]),
    ("dsvd_matrix_shape", C.c_int, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
    ("dsvd_matrix_download_transpose", C.c_int, [P, P, P, P]),
    ("dsvd_matrix_download", C.c_int, [P, P, P, P]),
    ("dsvd_matrix_download_rows", C.c_int, [P, I64, I64, P, P, P]),
    ("dsvd_matrix_row_offsets", C.c_int, [P, P]),
    ("dsvd_matrix_bench_spmm", C.c_int, [P, C.c_int, I64, C.c_int, C.c_int, C.POINTER(D)]),
    ("dsvd_matrix_hub_rows", C.c_int, [P, C.POINTER(I64), C.POINTER(I64)]),
    ("dsvd_solve", C.c_int, [P, P, C.POINTER(dsvd_config), C.POINTER(dsvd_outputs), OBSERVER, P]),
    ("dsvd_solve_csr", C.c_int, [P, I64, I64, I64, P, P, P, C.POINTER(dsvd_config),
                                 C.POINTER(dsvd_outputs)]),
    ("dsvd_solve_csr_device", C.c_int, [P, I64, I64, I64, P, P, P, C.POINTER(dsvd_config),
                                        C.POINTER(dsvd_outputs)]),
    ("dsvd_ctx_timer_start", C.c_int, [P]),
    ("dsvd_ctx_timer_stop", C.c_int, [P, C.POINTER(D)]),
    ("dsvd_finalize_row_basis", C.c_int, [P, P, P, I64, I64, P, P, P]),
    ("dsvd_eps_pve", C.c_int, [P, P, P, I64, P, I64, C.POINTER(D)]),
    ("dsvd_eps_res", C.c_int, [P, P, P, P, P, I64, P, I64, C.POINTER(D)]),
    ("dsvd_eps_spec", C.c_int, [P, P, P, P, P, I64, P, I64, I64, U64, C.POINTER(D)]),
    ("dsvd_csr_validate", C.c_int, [P, I64, I64, I64, P, P, P]),
    ("dsvd_save_cache", C.c_int, [C.c_char_p, I64, I64, I64, P, P, P]),
    ("dsvd_matrix_load_cache", C.c_int, [P, C.c_char_p, C.c_int, C.POINTER(P), C.POINTER(I64)]),
    ("dsvd_coo_assemble", C.c_int, [P, I64, I64, I64, P, P, P, C.POINTER(I64)]),
    ("dsvd_coo_fetch", C.c_int, [P, P, P, P]),
    ("dsvd_matrix_from_coo", C.c_int, [P, C.POINTER(P)]),
    ("dsvd_mtx_assemble", C.c_int, [P, C.c_char_p, C.POINTER(I64)]),
    ("dsvd_mtx_read", C.c_int, [C.c_char_p, C.POINTER(I64)]),
    ("dsvd_mtx_fetch", C.c_int, [P, P, P]),
    ("dsvd_write_matrix_market", C.c_int, [C.c_char_p, I64, I64, P, P, P]),
    ("dsvd_dense_read", C.c_int, [C.c_char_p, C.POINTER(I64)]),
    ("dsvd_dense_fetch", C.c_int, [P]),
    ("dsvd_dense_write", C.c_int, [C.c_char_p, I64, I64, P]),
    ("dsvd_spectrum_read", C.c_int, [C.c_char_p, C.POINTER(I64)]),
    ("dsvd_spectrum_fetch", C.c_int, [P]),
    ("dsvd_spectrum_write", C.c_int, [C.c_char_p, P, I64]),
    ("dsvd_max_triplet_residual", C.c_int, [P, P, P, P, P, I64, C.POINTER(D)]),
    ("dsvd_validate_config", C.c_int, [C.POINTER(dsvd_config), I64, I64]),
    ("dsvd_update_shift", D, [D, D]),
    ("dsvd_pve_stop_check", C.c_int, [P, I64, D, P, I64, D, I64, D, C.POINTER(C.c_int)]),
    ("dsvd_spmm", C.c_int, [P, I64, I64, I64, P, P, P, P, I64, P]),
    ("dsvd_spmm_shift", C.c_int, [P, I64, I64, I64, P, P, P, P, I64, D, P, P]),
    ("dsvd_transpose", C.c_int, [P, I64, I64, I64, P, P, P, P, P, P]),
    ("dsvd_gram", C.c_int, [P, I64, I64, P, P]),
    ("dsvd_sym_eig", C.c_int, [P, I64, P, P, P]),
    ("dsvd_eig_svd", C.c_int, [P, I64, I64, P, P, P, P]),
    ("dsvd_matmul", C.c_int, [P, I64, I64, I64, P, P, P]),
    ("dsvd_gaussian_matrix", C.c_int, [P, I64, I64, U64, P]),
    ("dsvd_gaussian_rows", C.c_int, [P, I64, I64, U64, I64, I64, P]),
    ("dsvd_splitmix64_at", U64, [U64, U64]),
    ("dsvd_synth_sparse_random", C.c_int, [I64, I64, I64, U64, C.c_int, C.POINTER(I64)]),
    ("dsvd_synth_powerlaw", C.c_int, [I64, I64, D, D, D, C.c_int, U64, C.POINTER(I64)]),
    ("dsvd_synth_fetch", C.c_int, [P, P, P]),
    ("dsvd_synth_rmat", C.c_int, [P, C.c_int, I64, D, D, D, C.c_int, U64, C.POINTER(P), C.POINTER(I64)]),
]

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the native library, or raise NativeLibraryMissing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `make -C paper_2404_09276_b200/csrc` "
                "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib


def check(rc: int) -> None:
    """Translate a C-ABI status into the reference's exception types."""
    if rc == DSVD_OK:
        return
    L = lib()
    msg = (L.dsvd_last_error() or b"").decode(errors="replace")
    if rc == DSVD_SHAPE:
        raise E.ShapeError(msg)
    if rc == DSVD_CONFIG:
        raise E.ConfigError(msg)
    if rc == DSVD_RANK:
        raise E.RankDeficient(int(L.dsvd_last_error_index()), msg.split(" (index")[0])
    if rc == DSVD_NUMERICAL:
        raise E.NumericalError(msg)
    if rc == DSVD_UNSUPPORTED:
        raise E.UnsupportedOnDevice(msg)
    if rc == DSVD_DEGENERATE:
        raise E.DegenerateReference(msg)
    if rc == DSVD_FORMAT:
        raise E.UnsupportedFormat(msg)
    if rc == DSVD_PARSE:
        raise E.ParseError(int(L.dsvd_last_error_index()), msg)
    if rc == DSVD_OTHER:
        raise E.Error(msg)
    raise E.DeviceError(f"[status {rc}] {msg}")
