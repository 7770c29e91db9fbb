"""ctypes bindings for the CHECKERS (test infrastructure only).

- ``Oracle``   — oracle/_build/liboracle.so, the C restatement (oracle/dashsvd_oracle.c)
- ``Reference`` — oracle/_ref/libdashsvd_ref.so, the unmodified reference core
  compiled from /root/reference plus oracle/ref_harness.cpp (present when it was
  built in the dev container; it travels to the GPU box as a built file).
- ``InputsGen`` — oracle/_build/libinputs.so (oracle/inputs_gen.c): the synthetic
  matrices of BASELINE.json configs 2-5 built on the host without the product
  library (bench.py's reference arm).

Both expose the same Python surface: column-major numpy arrays in and out, the
reference's status codes turned into the exceptions of
``paper_2404_09276_b200.errors``. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdashsvd_ref.so")
INPUTS_SO = os.path.join(ROOT, "oracle", "_build", "libinputs.so")

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_U64 = C.c_uint64


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


@dataclass
class Csr:
    rows: int
    cols: int
    offsets: np.ndarray  # int64 rows+1
    col_indices: np.ndarray  # int64 nnz
    values: np.ndarray  # float64 nnz

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])


class _orc_csr(C.Structure):
    _fields_ = [("rows", _I64), ("cols", _I64), ("nnz", _I64), ("offsets", _P),
                ("col_indices", _P), ("values", _P)]


class _orc_config(C.Structure):
    _fields_ = [("k", _I64), ("s", _I64), ("p", _I64), ("tol", _D), ("p_max", _I64),
                ("alg", C.c_int), ("seed", _U64), ("orth_qr", C.c_int)]


ALG = {"basic": 0, "shifted": 1, "fixed_shift": 2, "dash": 3}
STOP = {0: "fixed_p", 1: "tol_met", 2: "p_max_reached"}


def _raise(code, msg, index):
    from paper_2404_09276_b200 import errors as E
    if code == 0:
        return
    if code == 3:
        raise E.RankDeficient(int(index), msg)
    if code == 12:
        raise E.ParseError(int(index), msg.split(": ", 1)[1] if msg.startswith("parse error") else msg)
    raise {1: E.ShapeError, 2: E.ConfigError, 4: E.NumericalError, 11: E.UnsupportedFormat}.get(code, E.Error)(msg)


def transpose_np(a: Csr) -> Csr:
    """Counting-sort transpose (same rule as sparse_matrix.cpp:35-55), numpy."""
    order = np.argsort(a.col_indices, kind="stable")
    rows_of = np.repeat(np.arange(a.rows, dtype=np.int64), np.diff(a.offsets))
    off = np.zeros(a.cols + 1, dtype=np.int64)
    np.cumsum(np.bincount(a.col_indices, minlength=a.cols), out=off[1:])
    return Csr(a.cols, a.rows, off, rows_of[order].astype(np.int64), a.values[order].copy())


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.path = path

    def f(self, name, res, *args):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = res
        fn.argtypes = list(args)
        return fn

    def err(self):
        msg = self.f("last_error", C.c_char_p)().decode()
        idx = self.f("last_error_index", C.c_longlong)()
        return msg, idx

    def check(self, rc):
        if rc != 0:
            msg, idx = self.err()
            _raise(rc, msg, idx)

    # --- RNG -----------------------------------------------------------
    def splitmix64_at(self, seed, i):
        return int(self.f("splitmix64_at", _U64, _U64, _U64)(seed, i))

    def normal_at(self, seed, i):
        return float(self.f("normal_at", _D, _U64, _U64)(seed, i))

    def gaussian_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        self.f("gaussian_matrix", None, _I64, _I64, _U64, _P)(rows, cols, seed, _ptr(out))
        return out

    # --- dense ---------------------------------------------------------
    def gram(self, c):
        c = np.asfortranarray(c, dtype=np.float64)
        g = np.empty((c.shape[1], c.shape[1]), order="F")
        self._gram(c, g)
        return g

    def matmul(self, a, b):
        a = np.asfortranarray(a, dtype=np.float64)
        b = np.asfortranarray(b, dtype=np.float64)
        c = np.empty((a.shape[0], b.shape[1]), order="F")
        self._matmul(a, b, c)
        return c

    def sym_eig(self, g):
        g = np.asfortranarray(g, dtype=np.float64)
        n = g.shape[0]
        w = np.empty(n)
        v = np.empty((n, n), order="F")
        self.check(self.f("sym_eig", C.c_int, _I64, _P, _P, _P)(n, _ptr(g), _ptr(w), _ptr(v)))
        return w, v

    def eig_svd(self, c):
        c = np.asfortranarray(c, dtype=np.float64)
        m, n = c.shape
        u = np.empty((m, n), order="F")
        s = np.empty(n)
        v = np.empty((n, n), order="F")
        self.check(self.f("eig_svd", C.c_int, _I64, _I64, _P, _P, _P, _P)(
            m, n, _ptr(c), _ptr(u), _ptr(s), _ptr(v)))
        return u, s, v

    def update_shift(self, alpha, s_ll):
        return float(self.f("update_shift", _D, _D, _D)(alpha, s_ll))


class Oracle(_Lib):
    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)

    @staticmethod
    def _csr(a: Csr):
        return _orc_csr(a.rows, a.cols, a.nnz, _ptr(a.offsets), _ptr(a.col_indices),
                        _ptr(a.values))

    def sparse_random(self, rows, cols, npr, seed, decay=False) -> Csr:
        nnz = _I64()
        po, pi, pv = _P(), _P(), _P()
        fn = self.f("sparse_random", C.c_int, _I64, _I64, _I64, _U64, C.c_int, C.POINTER(_I64),
                    C.POINTER(_P), C.POINTER(_P), C.POINTER(_P))
        self.check(fn(rows, cols, npr, seed, 1 if decay else 0, C.byref(nnz), C.byref(po),
                      C.byref(pi), C.byref(pv)))
        n = nnz.value
        off = np.ctypeslib.as_array(C.cast(po, C.POINTER(_I64)), (rows + 1,)).copy()
        idx = np.ctypeslib.as_array(C.cast(pi, C.POINTER(_I64)), (max(n, 1),))[:n].copy()
        val = np.ctypeslib.as_array(C.cast(pv, C.POINTER(_D)), (max(n, 1),))[:n].copy()
        free = self.f("free", None, _P)
        for p in (po, pi, pv):
            free(p)
        return Csr(rows, cols, off, idx, val)

    def transpose(self, a: Csr) -> Csr:
        to = np.empty(a.cols + 1, dtype=np.int64)
        ti = np.empty(a.nnz, dtype=np.int64)
        tv = np.empty(a.nnz, dtype=np.float64)
        cs = self._csr(a)
        self.check(self.f("transpose", C.c_int, _P, _P, _P, _P)(C.byref(cs), _ptr(to), _ptr(ti),
                                                              _ptr(tv)))
        return Csr(a.cols, a.rows, to, ti, tv)

    def spmm(self, a: Csr, x):
        x = np.asfortranarray(x, dtype=np.float64)
        l = x.shape[1]
        y = np.empty((a.rows, l), order="F")
        cs = self._csr(a)
        self.check(self.f("spmm", C.c_int, _P, _P, _I64, _P)(C.byref(cs), _ptr(x), l, _ptr(y)))
        return y

    def add_scaled(self, y, alpha, x):
        y = np.array(y, dtype=np.float64, order="F", copy=True)
        x = np.asfortranarray(x, dtype=np.float64)
        self.f("add_scaled", None, _I64, _P, _D, _P)(y.size, _ptr(y), alpha, _ptr(x))
        return y

    def _gram(self, c, g):
        self.f("gram", None, _I64, _I64, _P, _P)(c.shape[0], c.shape[1], _ptr(c), _ptr(g))

    def _matmul(self, a, b, c):
        self.f("matmul", None, _I64, _I64, _I64, _P, _P, _P)(a.shape[0], a.shape[1], b.shape[1],
                                                           _ptr(a), _ptr(b), _ptr(c))

    def validate_config(self, rows, cols, k, s=-1, p=-1, tol=1e-2, p_max=1000, alg="dash"):
        cfg = _orc_config(k, s, p, tol, p_max, ALG[alg], 0, 0)
        self.check(self.f("validate_config", C.c_int, _P, _I64, _I64)(C.byref(cfg), rows, cols))

    def pve_stop_check(self, prev, alpha_prev, cur, alpha, k, tol):
        prev = np.ascontiguousarray(prev, dtype=np.float64)
        cur = np.ascontiguousarray(cur, dtype=np.float64)
        stop = C.c_int()
        fn = self.f("pve_stop_check", C.c_int, _P, _I64, _D, _P, _I64, _D, _I64, _D,
                    C.POINTER(C.c_int))
        self.check(fn(_ptr(prev), prev.size, alpha_prev, _ptr(cur), cur.size, alpha, k, tol,
                      C.byref(stop)))
        return bool(stop.value)

    def finalize_row_basis(self, a: Csr, q, k):
        q = np.asfortranarray(q, dtype=np.float64)
        l = q.shape[1]
        u = np.empty((a.rows, k), order="F")
        s = np.empty(k)
        v = np.empty((a.cols, k), order="F")
        cs = self._csr(a)
        self.check(self.f("finalize_row_basis", C.c_int, _P, _P, _I64, _I64, _P, _P, _P)(
            C.byref(cs), _ptr(q), l, k, _ptr(u), _ptr(s), _ptr(v)))
        return u, s, v

    def qr_orth(self, c):
        c = np.asfortranarray(c, dtype=np.float64)
        q = np.empty_like(c, order="F")
        self.check(self.f("qr_orth", C.c_int, _I64, _I64, _P, _P)(c.shape[0], c.shape[1], _ptr(c), _ptr(q)))
        return q

    def solve(self, a: Csr, k, s=-1, p=-1, tol=1e-2, p_max=1000, alg="dash", seed=0, at=None, orth="eigsvd"):
        at = at if at is not None else self.transpose(a)
        sw = k + (s if s >= 0 else max(1, k // 2))
        cap = (p_max if alg == "dash" else max(p, 0)) + 1
        u = np.empty((a.rows, k), order="F")
        sv = np.empty(k)
        v = np.empty((a.cols, k), order="F")
        alphas = np.zeros(cap)
        s_hat = np.zeros((cap, sw))
        it = _I64()
        sr = C.c_int()
        cfg = _orc_config(k, s, p, tol, p_max, ALG[alg], seed, 1 if orth == "qr" else 0)
        ca, cat = self._csr(a), self._csr(at)
        fn = self.f("solve", C.c_int, _P, _P, _P, _P, _P, _P, _P, _P, _I64, C.POINTER(_I64),
                    C.POINTER(C.c_int))
        self.check(fn(C.byref(ca), C.byref(cat), C.byref(cfg), _ptr(u), _ptr(sv), _ptr(v),
                      _ptr(alphas), _ptr(s_hat), cap, C.byref(it), C.byref(sr)))
        n = it.value
        return dict(u=u, s=sv, v=v, alphas=alphas[:n].copy(), s_hat=s_hat[:n].copy(),
                    iterations=n, stop_reason=STOP[sr.value])


class Reference(_Lib):
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)

    def set_threads(self, n):
        self.f("set_threads", None, C.c_int)(n)

    def thread_count(self):
        return int(self.f("thread_count", C.c_int)())

    def metrics(self, a: Csr, u, s, v, sigmas, power_iters=300, seed=0x5EED):
        """[eps_pve, eps_res, eps_spec, max_triplet_residual] (metrics.cpp:99-206)."""
        u, v = np.asfortranarray(u, dtype=np.float64), np.asfortranarray(v, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.float64)
        sg = np.ascontiguousarray(sigmas, dtype=np.float64)
        out = np.zeros(4)
        fn = self.f("metrics", C.c_int, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _P, _I64, _I64, _U64, _P)
        self.check(fn(*self._a(a), _ptr(u), _ptr(s), _ptr(v), s.size, _ptr(sg), sg.size, power_iters, seed,
                      _ptr(out)))
        return out

    # --- inputs (matrix_market.cpp, sparse_matrix.cpp:12-33) ---------------
    def validate(self, a: Csr):
        self.check(self.f("validate", C.c_int, _I64, _I64, _I64, _P, _P, _P)(*self._a(a)))

    def _fetch_csr(self, dims) -> Csr:
        rows, cols, n = dims[0], dims[1], dims[2]
        off = np.empty(rows + 1, dtype=np.int64)
        idx = np.empty(n, dtype=np.int64)
        val = np.empty(n, dtype=np.float64)
        self.f("csr_fetch", None, _P, _P, _P)(_ptr(off), _ptr(idx), _ptr(val))
        return Csr(rows, cols, off, idx, val)

    def load_matrix_market(self, path) -> Csr:
        dims = (_I64 * 3)()
        self.check(self.f("load_matrix_market", C.c_int, C.c_char_p, _P)(os.fsencode(path), dims))
        return self._fetch_csr(dims)

    def load_cache(self, path) -> Csr:
        dims = (_I64 * 3)()
        self.check(self.f("load_cache", C.c_int, C.c_char_p, _P)(os.fsencode(path), dims))
        return self._fetch_csr(dims)

    def save_cache(self, path, a: Csr):
        self.check(self.f("save_cache", C.c_int, C.c_char_p, _I64, _I64, _I64, _P, _P, _P)(os.fsencode(path),
                                                                                       *self._a(a)))

    def load_dense_array(self, path):
        dims = (_I64 * 2)()
        self.check(self.f("load_dense_array", C.c_int, C.c_char_p, _P)(os.fsencode(path), dims))
        out = np.empty((dims[0], dims[1]), order="F")
        self.f("dense_fetch", None, _P)(_ptr(out))
        return out

    def write_dense_array(self, path, a):
        a = np.asfortranarray(a, dtype=np.float64)
        self.check(self.f("write_dense_array", C.c_int, C.c_char_p, _I64, _I64, _P)(os.fsencode(path), a.shape[0],
                                                                                 a.shape[1], _ptr(a)))

    def load_spectrum(self, path):
        n = _I64()
        self.check(self.f("load_spectrum", C.c_int, C.c_char_p, C.POINTER(_I64))(os.fsencode(path), C.byref(n)))
        out = np.empty(n.value)
        self.f("spectrum_fetch", None, _P)(_ptr(out))
        return out

    def write_spectrum(self, path, s):
        s = np.ascontiguousarray(s, dtype=np.float64)
        self.check(self.f("write_spectrum", C.c_int, C.c_char_p, _P, _I64)(os.fsencode(path), _ptr(s), s.size))

    def write_matrix_market(self, path, a: Csr):
        self.check(self.f("write_matrix_market", C.c_int, C.c_char_p, _I64, _I64, _I64, _P, _P, _P)(
            os.fsencode(path), *self._a(a)))

    def sparse_random(self, rows, cols, npr, seed, decay=False) -> Csr:
        nnz = _I64()
        self.check(self.f("sparse_random", C.c_int, _I64, _I64, _I64, _U64, C.c_int,
                          C.POINTER(_I64))(rows, cols, npr, seed, 1 if decay else 0, C.byref(nnz)))
        n = nnz.value
        off = np.empty(rows + 1, dtype=np.int64)
        idx = np.empty(n, dtype=np.int64)
        val = np.empty(n, dtype=np.float64)
        self.f("sparse_random_fetch", None, _P, _P, _P)(_ptr(off), _ptr(idx), _ptr(val))
        return Csr(rows, cols, off, idx, val)

    def _a(self, a: Csr):
        return (a.rows, a.cols, a.nnz, _ptr(a.offsets), _ptr(a.col_indices), _ptr(a.values))

    def transpose(self, a: Csr) -> Csr:
        to = np.empty(a.cols + 1, dtype=np.int64)
        ti = np.empty(a.nnz, dtype=np.int64)
        tv = np.empty(a.nnz, dtype=np.float64)
        self.check(self.f("transpose", C.c_int, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P)(
            *self._a(a), _ptr(to), _ptr(ti), _ptr(tv)))
        return Csr(a.cols, a.rows, to, ti, tv)

    def spmm(self, a: Csr, x):
        x = np.asfortranarray(x, dtype=np.float64)
        l = x.shape[1]
        y = np.empty((a.rows, l), order="F")
        self.check(self.f("spmm", C.c_int, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _P)(
            *self._a(a), _ptr(x), l, _ptr(y)))
        return y

    def add_scaled(self, y, alpha, x):
        y = np.array(y, dtype=np.float64, order="F", copy=True)
        x = np.asfortranarray(x, dtype=np.float64)
        self.check(self.f("add_scaled", C.c_int, _I64, _I64, _P, _D, _P)(
            y.shape[0], y.shape[1], _ptr(y), alpha, _ptr(x)))
        return y

    def _gram(self, c, g):
        self.check(self.f("gram", C.c_int, _I64, _I64, _P, _P)(c.shape[0], c.shape[1], _ptr(c),
                                                             _ptr(g)))

    def _matmul(self, a, b, c):
        self.check(self.f("matmul", C.c_int, _I64, _I64, _I64, _P, _P, _P)(
            a.shape[0], a.shape[1], b.shape[1], _ptr(a), _ptr(b), _ptr(c)))

    def validate_config(self, rows, cols, k, s=-1, p=-1, tol=1e-2, p_max=1000, alg="dash"):
        self.check(self.f("validate_config", C.c_int, _I64, _I64, _I64, _I64, _I64, _D, _I64,
                          C.c_int)(rows, cols, k, s, p, tol, p_max, ALG[alg]))

    def pve_stop_check(self, prev, alpha_prev, cur, alpha, k, tol):
        prev = np.ascontiguousarray(prev, dtype=np.float64)
        cur = np.ascontiguousarray(cur, dtype=np.float64)
        stop = C.c_int()
        fn = self.f("pve_stop_check", C.c_int, _P, _I64, _D, _P, _I64, _D, _I64, _D,
                    C.POINTER(C.c_int))
        self.check(fn(_ptr(prev), prev.size, alpha_prev, _ptr(cur), cur.size, alpha, k, tol,
                      C.byref(stop)))
        return bool(stop.value)

    def finalize_row_basis(self, a: Csr, q, k):
        q = np.asfortranarray(q, dtype=np.float64)
        l = q.shape[1]
        u = np.empty((a.rows, k), order="F")
        s = np.empty(k)
        v = np.empty((a.cols, k), order="F")
        self.check(self.f("finalize_row_basis", C.c_int, _I64, _I64, _I64, _P, _P, _P, _P, _I64,
                          _I64, _P, _P, _P)(*self._a(a), _ptr(q), l, k, _ptr(u), _ptr(s), _ptr(v)))
        return u, s, v

    def solve(self, a: Csr, k, s=-1, p=-1, tol=1e-2, p_max=1000, alg="dash", seed=0,
              times=False, orth="eigsvd"):
        self.f("set_orth", None, C.c_int)(1 if orth == "qr" else 0)
        sw = k + (s if s >= 0 else max(1, k // 2))
        cap = (p_max if alg == "dash" else max(p, 0)) + 1
        u = np.empty((a.rows, k), order="F")
        sv = np.empty(k)
        v = np.empty((a.cols, k), order="F")
        alphas = np.zeros(cap)
        s_hat = np.zeros((cap, sw))
        it = _I64()
        sr = C.c_int()
        tm = np.zeros(cap + 2) if times else None
        fn = self.f("solve", C.c_int, _I64, _I64, _I64, _P, _P, _P, _I64, _I64, _I64, _D, _I64,
                    C.c_int, _U64, _P, _P, _P, _P, _P, _I64, C.POINTER(_I64), C.POINTER(C.c_int),
                    _P)
        self.check(fn(*self._a(a), k, s, p, tol, p_max, ALG[alg], seed, _ptr(u), _ptr(sv),
                      _ptr(v), _ptr(alphas), _ptr(s_hat), cap, C.byref(it), C.byref(sr),
                      _ptr(tm)))
        n = it.value
        out = dict(u=u, s=sv, v=v, alphas=alphas[:n].copy(), s_hat=s_hat[:n].copy(),
                   iterations=n, stop_reason=STOP[sr.value])
        if times:
            out["times"] = dict(transpose=float(tm[0]), solve=float(tm[1]),
                                stamps=tm[2:2 + n].copy())
        return out


class InputsGen:
    """oracle/inputs_gen.c: R-MAT (configs 4/5) and power-law (configs 2/3) inputs,
    bit-identical to the product's generators (tests/test_inputs_gen.py)."""

    def __init__(self, path=INPUTS_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.lib.gen_rmat.restype = C.c_int
        self.lib.gen_rmat.argtypes = [C.c_int, _I64, _D, _D, _D, C.c_int, _U64, C.POINTER(_I64)]
        self.lib.gen_powerlaw.restype = C.c_int
        self.lib.gen_powerlaw.argtypes = [_I64, _I64, _D, _D, _D, C.c_int, _U64, C.POINTER(_I64)]
        self.lib.gen_fetch.restype = None
        self.lib.gen_fetch.argtypes = [_P, _P, _P]

    def _fetch(self, rows, cols, nnz) -> Csr:
        off = np.empty(rows + 1, dtype=np.int64)
        idx = np.empty(nnz, dtype=np.int64)
        val = np.empty(nnz, dtype=np.float64)
        self.lib.gen_fetch(_ptr(off), _ptr(idx), _ptr(val))
        return Csr(rows, cols, off, idx, val)

    def rmat(self, scale, draws, a=0.57, b=0.19, c=0.19, uniform=False, seed=0) -> Csr:
        nnz = _I64()
        rc = self.lib.gen_rmat(int(scale), int(draws), a, b, c, 1 if uniform else 0, int(seed), C.byref(nnz))
        if rc != 0:
            raise RuntimeError(f"gen_rmat failed ({rc})")
        n = 1 << int(scale)
        return self._fetch(n, n, nnz.value)

    def powerlaw(self, rows, cols, mu, sigma, zipf_s, seed, ratings=False) -> Csr:
        nnz = _I64()
        rc = self.lib.gen_powerlaw(int(rows), int(cols), mu, sigma, zipf_s, 1 if ratings else 0, int(seed),
                                   C.byref(nnz))
        if rc != 0:
            raise RuntimeError(f"gen_powerlaw failed ({rc})")
        return self._fetch(rows, cols, nnz.value)
