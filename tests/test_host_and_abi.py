"""CPU tests of the host side: the C-ABI library loads and exports every symbol
include/dashsvd_b200.h declares, the pure host functions behave like the
reference's, the synthetic generators are deterministic, sharding is sound.
No CUDA compute runs here (there is no GPU in the dev container)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2404_09276_b200 as d
from paper_2404_09276_b200 import _native
from paper_2404_09276_b200.sharding import shard_bounds, shard_csr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            with open(os.path.join(ROOT, "include", fn)) as f:
                names |= set(re.findall(r"DSVD_API\s+[\w\s\*]+?\b(dsvd_\w+)\s*\(", f.read()))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    bound = {n for n, _, _ in _native.SIGNATURES}
    assert set(names) <= bound, set(names) - bound


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(d.DeviceError):
        d.Device(0)


def test_host_update_shift_and_stop_rule():
    # test_rsvd.cpp:33-84 through the C ABI's host functions
    assert d.update_shift(0.0, 0.5) == 0.25
    assert d.update_shift(0.3, 0.2) == 0.3
    assert d.update_shift(0.25, 0.35) == pytest.approx(0.30, rel=1e-15)
    assert not d.pve_stop_check([3.90, 1.00], 0.0, [4.00, 1.00], 0.05, 1, 0.01)
    assert d.pve_stop_check([4.0, 1.0], 0.05, [4.0, 1.0], 0.05, 1, 1e-12)
    assert d.pve_stop_check([4.00, 1.00], 0.05, [4.005, 1.00], 0.05, 1, 0.01)
    assert not d.pve_stop_check([2.0, 0.0], 0.0, [1.0, 0.0], 0.0, 1, 0.01)
    assert not d.pve_stop_check([1.0, 0.0], 0.0, [1.0, 0.0], 0.0, 1, 0.01)
    with pytest.raises(d.ShapeError):
        d.pve_stop_check([4.0], 0.0, [4.0], 0.0, 1, 0.01)


def test_host_update_shift_matches_oracle(oracle):
    rng = np.random.default_rng(0)
    for _ in range(500):
        a, s = rng.random(2)
        assert d.update_shift(a, s) == oracle.update_shift(a, s)


def cfg(alg, k, s, p=-1, **kw):
    return d.SolverConfig(k=k, s=s, p=p, alg=d.Algorithm[alg], **kw)


def test_validate_config_matches_reference_rules():
    # test_rsvd.cpp:86-133
    bad = [cfg("dash", 0, 1), cfg("shifted", 25, 10, 4), cfg("dash", 4, 0),
           cfg("basic", 4, 2, -1), cfg("shifted", 4, 2, -1), cfg("fixed_shift", 4, 2, -1),
           cfg("dash", 4, 2, tol=0.0), cfg("dash", 4, 2, tol=-1.0), cfg("dash", 4, 2, p_max=0),
           cfg("dash", 4, 2, orth=d.Orthonormalizer.qr),
           cfg("shifted", 4, 2, 3, orth=d.Orthonormalizer.qr)]
    for c in bad:
        with pytest.raises(d.ConfigError):
            d.validate_config(c, 40, 30)
    d.validate_config(cfg("dash", 4, 2), 40, 30)
    d.validate_config(cfg("basic", 4, 2, 0, orth=d.Orthonormalizer.qr), 40, 30)
    with pytest.raises(d.ShapeError):
        d.validate_config(cfg("dash", 4, 2), 0, 30)
    c = d.SolverConfig()
    assert c.effective_s(1) == 1 and c.effective_s(7) == 3 and c.effective_s(2) == 1
    c.k = 7
    assert c.sketch_width() == 10
    c.s = 0
    assert c.sketch_width() == 7


def test_validate_config_agrees_with_oracle(oracle):
    from paper_2404_09276_b200 import ConfigError
    rng = np.random.default_rng(1)
    for _ in range(300):
        k, s = int(rng.integers(0, 12)), int(rng.integers(-1, 8))
        p, p_max = int(rng.integers(-1, 4)), int(rng.integers(0, 3))
        tol = float(rng.choice([-1.0, 0.0, 1e-2]))
        alg = str(rng.choice(["shifted", "fixed_shift", "dash"]))
        rows, cols = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        c = d.SolverConfig(k=k, s=s, p=p, tol=tol, p_max=p_max, alg=d.Algorithm[alg])
        try:
            oracle.validate_config(rows, cols, k=k, s=s, p=p, tol=tol, p_max=p_max, alg=alg)
            ok_ref = True
        except ConfigError:
            ok_ref = False
        try:
            d.validate_config(c, rows, cols)
            ok = True
        except ConfigError:
            ok = False
        assert ok == ok_ref, (c, rows, cols)


def test_splitmix_host_pins():
    assert d.splitmix64_at(0, 0) == 0xe220a8397b1dcdaf
    assert d.splitmix64_at(0x8000000000000000, 5) == 0x4d7e6a268a67c5ff


def test_sparse_random_generator_bitwise_reference(oracle):
    # the native host generator reproduces synthetic.cpp:72-120 bit for bit
    a = d.sparse_random(10000, 5000, 25, 0, True)
    b = oracle.sparse_random(10000, 5000, 25, 0, True)
    assert a.nnz == b.nnz == 249377
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))
    a.validate()


def test_powerlaw_generator_deterministic_and_canonical():
    a = d.powerlaw(3000, 2000, 3.0, 1.0, 1.1, 5)
    b = d.powerlaw(3000, 2000, 3.0, 1.0, 1.1, 5)
    assert np.array_equal(a.col_indices, b.col_indices) and np.array_equal(a.values, b.values)
    a.validate()  # strictly increasing columns = sampled without replacement
    deg = np.diff(a.offsets)
    assert deg.min() >= 1
    counts = np.bincount(a.col_indices, minlength=2000)
    assert counts.max() > 20 * np.median(counts[counts > 0])  # Zipf hub columns
    r = d.powerlaw(2000, 1000, 3.0, 1.0, 1.0, 9, ratings=True)
    assert set(np.unique(r.values)) <= {1.0, 2.0, 3.0, 4.0, 5.0}


def test_sparse_validate_catches_violations():
    ok = d.SparseMatrix(2, 3, [0, 1, 2], [0, 2], [1.0, 2.0])
    ok.validate()
    with pytest.raises(d.ShapeError):
        d.SparseMatrix(2, 3, [0, 2, 2], [1, 1], [1.0, 2.0]).validate()
    with pytest.raises(d.ShapeError):
        d.SparseMatrix(2, 3, [0, 1, 2], [0, 3], [1.0, 2.0]).validate()
    with pytest.raises(d.NumericalError):
        d.SparseMatrix(2, 3, [0, 1, 2], [0, 1], [1.0, 0.0]).validate()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_bounds_cover_and_balance(world):
    a = d.powerlaw(5000, 1000, 3.0, 1.0, 1.1, 3)
    b = shard_bounds(a.offsets, world)
    assert b[0] == 0 and b[-1] == a.rows and all(x <= y for x, y in zip(b, b[1:]))
    shards = [shard_csr(a, b[g], b[g + 1]) for g in range(world)]
    assert sum(s.nnz for s in shards) == a.nnz
    assert np.array_equal(np.concatenate([s.col_indices for s in shards]), a.col_indices)
    per = [s.nnz for s in shards]
    assert max(per) - min(per) <= int(np.diff(a.offsets).max()) + 1
    for s in shards:
        s.validate()


def test_loopback_group_lifecycle_on_the_host():
    """The in-process rank group is host state only: create / destroy and the
    argument checks need no GPU."""
    g = d.LoopbackGroup(3)
    assert g.nranks == 3
    g.close()
    for bad in (0, 9):
        with pytest.raises(d.ConfigError):
            d.LoopbackGroup(bad)

