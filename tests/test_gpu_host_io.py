"""Staged host copies (engine.cu copy_h2d / copy_d2h): a solve whose CSR inputs
and U/S/V outputs live in PAGEABLE host memory (std::vector / numpy — what the
reference-shaped API hands out) moves them through a ring of pinned slots with
host threads, instead of a cudaMemcpyAsync through the driver's bounce buffer.
The bytes must be exactly those of the pinned-buffer solve and of the unstaged
copy, for every entry point that writes host factors (the shifted / dash row
basis with column and row compaction, the basic algorithm), with slots small
enough that every array spans many of them."""
import numpy as np
import pytest

import paper_2404_09276_b200 as d

pytestmark = pytest.mark.gpu

CHUNK = 1 << 16  # 64 KB slots: U and V below span hundreds of slots


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def _rmat(scale, draws, seed):
    dv = d.Device(0)
    m = d.rmat(scale, draws, seed=seed, device=dv)
    a = m.download()
    m.close()
    dv.close()
    return a


def _copy(a):
    return d.SparseMatrix(a.rows, a.cols, a.offsets.copy(), a.col_indices.copy(), a.values.copy())


def _solve(a, cfg, staging, pinned, threads=0):
    a = _copy(a)
    k = cfg.k
    u = np.empty((a.rows, k), order="F")
    s = np.empty(k)
    v = np.empty((a.cols, k), order="F")
    arrays = (a.offsets, a.col_indices, a.values, u, s, v)
    if pinned:
        for x in arrays:
            d.pin(x)
    dv = d.Device(0)
    dv.set_option("host_staging", staging)
    dv.set_option("host_stage_chunk", CHUNK)
    dv.set_option("host_copy_threads", threads)
    try:
        r = d.solve(a, cfg, device=dv, out=(u, s, v))
    finally:
        dv.close()
        if pinned:
            for x in arrays:
                d.unpin(x)
    return r


def _same(r0, r1):
    assert r0.trace.iterations == r1.trace.iterations
    for name in ("u", "s", "v"):
        assert np.array_equal(bits(getattr(r0.svd, name)), bits(getattr(r1.svd, name))), name


@pytest.mark.parametrize("alg,kw", [("shifted", dict(p=3)), ("dash", dict(tol=1e-2)),
                                    ("basic", dict(p=2))])
def test_pageable_buffers_staged_are_bitwise_the_pinned_solve(alg, kw):
    a = _rmat(15, 400000, 7)  # ~half the rows / columns empty: compaction on both sides
    assert a.nnz * 8 > 16 * CHUNK
    cfg = d.SolverConfig(k=40, s=20, alg=d.Algorithm[alg], seed=5, **kw)
    pinned = _solve(a, cfg, staging=1, pinned=True)
    staged = _solve(a, cfg, staging=1, pinned=False)
    plain = _solve(a, cfg, staging=0, pinned=False)
    _same(pinned, staged)
    _same(pinned, plain)


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_staged_copies_any_thread_count(threads):
    """Odd thread counts and slices that do not divide the slot: same bytes."""
    a = d.powerlaw(30000, 12000, 2.0, 1.2, 1.1, 3)
    cfg = d.SolverConfig(k=30, s=10, p=2, alg=d.Algorithm.shifted, seed=1)
    ref = _solve(a, cfg, staging=0, pinned=False)
    _same(ref, _solve(a, cfg, staging=1, pinned=False, threads=threads))


def test_staging_options_are_validated():
    dv = d.Device(0)
    for name, value in (("host_staging", 2), ("host_stage_chunk", 1000), ("host_stage_chunk", 1 << 31),
                        ("host_copy_threads", -1)):
        with pytest.raises(d.ConfigError):
            dv.set_option(name, value)
    dv.close()
