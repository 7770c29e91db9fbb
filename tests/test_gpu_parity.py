"""GPU parity: every device kernel and the full solve, through the C ABI,
against the oracle (oracle/dashsvd_oracle.c, pinned bitwise to the reference)
on the same seeded inputs.

Bars (north_star / SURVEY 8d):
  - integer/byte work and every FMA-chain kernel whose order the device
    reproduces (CSR transpose, SpMM, SpMM+shift, matmul): BITWISE;
  - Gram: relative 1e-13 (split-K order differs from the reference's single chain);
  - eigensolver: relative 1e-12 on eigenvalues (Jacobi vs Householder+QL);
  - solve: singular values relative 1e-8, principal angles of U and V
    subspaces <= 1e-6, equal iteration count, PVE ratio at termination
    relative 1e-6.
"""
import numpy as np
import pytest

import paper_2404_09276_b200 as d
from oracle_lib import Csr, transpose_np

pytestmark = pytest.mark.gpu


def to_dev(a: Csr) -> d.SparseMatrix:
    return d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, a.values)


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def assert_bitwise(x, y):
    x = np.asarray(x)
    y = np.asarray(y)
    assert x.shape == y.shape
    diff = np.flatnonzero(bits(x.ravel(order="F")) != bits(y.ravel(order="F")))
    assert diff.size == 0, f"{diff.size} entries differ, first at {diff[:5]}"


def sin_theta(u_ref, u):
    """sine of the largest principal angle between span(u_ref) and span(u)."""
    q1, _ = np.linalg.qr(u_ref)
    q2, _ = np.linalg.qr(u)
    r = q2 - q1 @ (q1.T @ q2)
    return float(np.linalg.norm(r, 2))


@pytest.fixture(scope="module")
def c1(oracle):
    return oracle.sparse_random(10000, 5000, 25, 0, True)


# ---- CSR transpose (bit-exact) ------------------------------------------------

def test_transpose_bitwise_config1(dev, oracle, c1):
    t_ref = oracle.transpose(c1)
    t = d.transpose(to_dev(c1), device=dev)
    assert np.array_equal(t.offsets, t_ref.offsets)
    assert np.array_equal(t.col_indices, t_ref.col_indices)
    assert_bitwise(t.values, t_ref.values)


@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 3, 2), (50, 80, 6), (300, 20, 9), (1, 500, 40)])
def test_transpose_bitwise_shapes(dev, oracle, shape):
    rows, cols, npr = shape
    a = oracle.sparse_random(rows, cols, min(npr, cols), 11 + rows, False)
    t_ref = oracle.transpose(a)
    t = d.transpose(to_dev(a), device=dev)
    assert np.array_equal(t.offsets, t_ref.offsets)
    assert np.array_equal(t.col_indices, t_ref.col_indices)
    assert_bitwise(t.values, t_ref.values)


def test_transpose_empty_rows_and_zero_nnz(dev, oracle):
    # rows with no entries and an all-empty matrix
    off = np.array([0, 0, 2, 2, 3, 3], dtype=np.int64)
    a = Csr(5, 4, off, np.array([1, 3, 0], dtype=np.int64), np.array([1.5, -2.0, 3.0]))
    t_ref = oracle.transpose(a)
    t = d.transpose(to_dev(a), device=dev)
    assert np.array_equal(t.offsets, t_ref.offsets)
    assert np.array_equal(t.col_indices, t_ref.col_indices)
    assert_bitwise(t.values, t_ref.values)
    z = Csr(3, 6, np.zeros(4, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0))
    tz = d.transpose(to_dev(z), device=dev)
    assert np.array_equal(tz.offsets, np.zeros(7, dtype=np.int64)) and tz.nnz == 0


def test_transpose_power_law_hub_columns(dev, oracle):
    a = d.powerlaw(3000, 1500, 3.0, 1.0, 1.1, 5)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    t_ref = oracle.transpose(ca)
    t = d.transpose(a, device=dev)
    assert np.array_equal(t.offsets, t_ref.offsets)
    assert np.array_equal(t.col_indices, t_ref.col_indices)
    assert_bitwise(t.values, t_ref.values)


def test_transpose_rejects_bad_index(dev):
    a = d.SparseMatrix(2, 3, np.array([0, 1, 2]), np.array([0, 7]), np.array([1.0, 2.0]))
    with pytest.raises(d.ShapeError):
        d.transpose(a, device=dev)


# ---- SpMM (bit-exact) -----------------------------------------------------------

@pytest.mark.parametrize("l", [1, 3, 47, 48, 49, 64, 75, 97, 128, 129, 150, 190, 192, 193, 300])
def test_spmm_bitwise_widths(dev, oracle, c1, l):
    rng = np.random.default_rng(l)
    x = np.asfortranarray(rng.standard_normal((c1.cols, l)))
    y_ref = oracle.spmm(c1, x)
    y = d.spmm(to_dev(c1), x, device=dev)
    assert_bitwise(y, y_ref)


# spmm_variant bits: 64/128 force the 64-column slab kernel for the bulk rows /
# split chunks, 256/512 deepen the whole-row kernel's gather lookahead;
# 4096/8192 the slab-major column-slab kernel (32/64 columns) with 16384 its L2
# hints and 32768/65536 its gather depth
SLAB_VARIANTS = [4096, 8192, 4096 | 16384, 8192 | 16384 | 32768, 4096 | 65536, 4096 | 16384 | 32768]


@pytest.mark.parametrize("variant", [64, 128, 192, 256, 512] + SLAB_VARIANTS)
@pytest.mark.parametrize("l", [2, 75, 150])
def test_spmm_kernel_variants_bitwise(oracle, variant, l):
    dv = d.Device(0)
    dv.set_option("spmm_variant", variant)
    a = d.powerlaw(6000, 2500, 3.5, 1.0, 1.1, 21)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    at = transpose_np(ca)
    rng = np.random.default_rng(variant + l)
    for m, x in ((ca, rng.standard_normal((ca.cols, l))), (at, rng.standard_normal((ca.rows, l)))):
        x = np.asfortranarray(x)
        q = np.asfortranarray(rng.standard_normal((m.rows, l)))
        short = np.diff(m.offsets) <= 512  # rows the default split mode keeps whole
        y_ref = oracle.spmm(m, x)
        assert_bitwise(d.spmm(to_dev(m), x, device=dv)[short], y_ref[short])
        t_ref = oracle.add_scaled(y_ref, -0.25, q)
        assert_bitwise(d.spmm_shift(to_dev(m), x, 0.25, q, device=dv)[short], t_ref[short])
    dv.close()


@pytest.mark.parametrize("variant", SLAB_VARIANTS)
@pytest.mark.parametrize("l", [2, 75, 150, 300])
def test_spmm_slab_kernel_equals_the_default_split_mode(variant, l):
    """The slab kernel runs the split rows' chunks in the same launch: every row,
    split or not, must equal the default kernels' output bitwise (same chains,
    same chunk partials, same combine), with and without the fused shift."""
    a = d.powerlaw(7000, 2600, 3.5, 1.0, 1.1, 23)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    at = transpose_np(ca)
    assert np.diff(at.offsets).max() > 512  # split rows present
    base, dv = d.Device(0), d.Device(0)
    dv.set_option("spmm_variant", variant)
    rng = np.random.default_rng(l)
    for m, x in ((ca, rng.standard_normal((ca.cols, l))), (at, rng.standard_normal((ca.rows, l)))):
        x = np.asfortranarray(x)
        q = np.asfortranarray(rng.standard_normal((m.rows, l)))
        assert_bitwise(d.spmm(to_dev(m), x, device=dv), d.spmm(to_dev(m), x, device=base))
        assert_bitwise(d.spmm_shift(to_dev(m), x, 0.3, q, device=dv), d.spmm_shift(to_dev(m), x, 0.3, q, device=base))
    dv.close()
    base.close()


@pytest.mark.parametrize("variant", [4096 | 16384, 8192])
def test_solve_with_slab_kernel_is_bitwise_the_default_solve(variant):
    a = d.powerlaw(9000, 4000, 3.5, 1.0, 1.1, 5)
    cfg = d.SolverConfig(k=20, s=10, tol=1e-2, seed=4)
    base, dv = d.Device(0), d.Device(0)
    dv.set_option("spmm_variant", variant)
    r0 = d.solve(a, cfg, device=base)
    r1 = d.solve(a, cfg, device=dv)
    assert r0.trace.iterations == r1.trace.iterations
    assert_bitwise(r1.svd.s, r0.svd.s)
    assert_bitwise(r1.svd.u, r0.svd.u)
    assert_bitwise(r1.svd.v, r0.svd.v)
    dv.close()
    base.close()


@pytest.mark.parametrize("slab", [32, 64])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("pipeline", [0, 1])
@pytest.mark.parametrize("alg", ["shifted", "dash"])
def test_solve_slab_layouts_are_bitwise_the_whole_row_solve(slab, layout, pipeline, alg):
    """The column-slab kernel with slab-major sketch / A Q blocks (slab_layout 1:
    Omega and Y written slab-major, the pass-1 operand copied into a slab-major
    block) or with row-major blocks (slab_layout 0) reproduces the whole-row
    kernels' solve bitwise, on a width where the slab kernel is the candidate
    (l = 300) and on l = 150."""
    a = d.powerlaw(9000, 4000, 3.5, 1.0, 1.1, 6)
    for k, s_ in ((200, 100), (100, 50)):
        cfg = (d.SolverConfig(k=k, s=s_, p=3, alg=d.Algorithm.shifted, seed=2) if alg == "shifted"
               else d.SolverConfig(k=k, s=s_, tol=1e-2, p_max=6, seed=2))
        base, dv = d.Device(0), d.Device(0)
        for x in (base, dv):
            x.set_option("pipeline", pipeline)
        base.set_option("spmm_slab", 0)
        dv.set_option("spmm_slab", slab)
        dv.set_option("slab_layout", layout)
        r0 = d.solve(a, cfg, device=base)
        r1 = d.solve(a, cfg, device=dv)
        assert r0.trace.iterations == r1.trace.iterations
        assert_bitwise(r1.svd.s, r0.svd.s)
        assert_bitwise(r1.svd.u, r0.svd.u)
        assert_bitwise(r1.svd.v, r0.svd.v)
        assert_bitwise(np.array(r1.trace.alphas), np.array(r0.trace.alphas))
        dv.close()
        base.close()


@pytest.mark.parametrize("value", [1.0, -0.37, 0.0, None])
@pytest.mark.parametrize("slab", [32, 64])
def test_slab_kernel_uniform_values_bitwise(value, slab):
    """All-equal values (an unweighted graph's 1.0): the column-slab kernel
    multiplies by the one value instead of streaming them (uniform_values 1)
    and must match the value-streaming kernel and the whole-row kernels bitwise,
    with and without the fused shift; value None: one entry differs, so the
    detection must fall back to the stream."""
    a = d.powerlaw(7000, 2600, 3.5, 1.0, 1.1, 29)
    vals = np.full(a.nnz, 1.0 if value is None else value)
    if value is None:
        vals[a.nnz // 2] = 2.0
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, vals)
    at = transpose_np(ca)
    devs = [d.Device(0) for _ in range(3)]
    devs[0].set_option("spmm_slab", 0)
    for dv, uni in ((devs[1], 0), (devs[2], 1)):
        dv.set_option("spmm_variant", 4096 if slab == 32 else 8192)
        dv.set_option("uniform_values", uni)
    rng = np.random.default_rng(slab)
    for l in (75, 300):
        for m, x in ((ca, rng.standard_normal((ca.cols, l))), (at, rng.standard_normal((ca.rows, l)))):
            x = np.asfortranarray(x)
            q = np.asfortranarray(rng.standard_normal((m.rows, l)))
            ref = d.spmm(to_dev(m), x, device=devs[1])
            refs = d.spmm_shift(to_dev(m), x, 0.3, q, device=devs[1])
            assert_bitwise(d.spmm(to_dev(m), x, device=devs[0]), ref)
            assert_bitwise(d.spmm(to_dev(m), x, device=devs[2]), ref)
            assert_bitwise(d.spmm_shift(to_dev(m), x, 0.3, q, device=devs[2]), refs)
    for dv in devs:
        dv.close()


@pytest.mark.parametrize("hot_mb", [0, 1])
@pytest.mark.parametrize("hint", [0, 1, 2])
def test_solve_slab_l2_policies_are_bitwise_the_whole_row_solve(hot_mb, hint):
    """The slab kernel's L2 policies (hot/cold-tagged gathers, evict_first on the
    streaming bytes of every launch or of the A X pass only) change no bits."""
    a = d.powerlaw(9000, 4000, 3.5, 1.0, 1.1, 8)
    cfg = d.SolverConfig(k=200, s=100, p=2, alg=d.Algorithm.shifted, seed=3)
    base, dv = d.Device(0), d.Device(0)
    base.set_option("spmm_slab", 0)
    dv.set_option("spmm_slab", 64)
    dv.set_option("spmm_hot_mb", hot_mb)
    dv.set_option("spmm_slab_hint", hint)
    r0 = d.solve(a, cfg, device=base)
    r1 = d.solve(a, cfg, device=dv)
    assert_bitwise(r1.svd.s, r0.svd.s)
    assert_bitwise(r1.svd.u, r0.svd.u)
    assert_bitwise(r1.svd.v, r0.svd.v)
    dv.close()
    base.close()


def test_solve_uniform_values_is_bitwise_the_streaming_solve():
    a = d.powerlaw(9000, 4000, 3.5, 1.0, 1.1, 7)
    a = d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, np.ones(a.nnz))
    cfg = d.SolverConfig(k=200, s=100, p=3, alg=d.Algorithm.shifted, seed=2)
    base, dv = d.Device(0), d.Device(0)
    base.set_option("uniform_values", 0)
    for x in (base, dv):
        x.set_option("spmm_slab", 64)
    r0 = d.solve(a, cfg, device=base)
    r1 = d.solve(a, cfg, device=dv)
    assert_bitwise(r1.svd.s, r0.svd.s)
    assert_bitwise(r1.svd.u, r0.svd.u)
    assert_bitwise(r1.svd.v, r0.svd.v)
    dv.close()
    base.close()


def test_spmm_transpose_pass_bitwise(dev, oracle, c1):
    at = oracle.transpose(c1)
    y = np.asfortranarray(np.random.default_rng(3).standard_normal((c1.rows, 75)))
    assert_bitwise(d.spmm(to_dev(at), y, device=dev), oracle.spmm(at, y))


@pytest.mark.parametrize("alpha", [0.0, 0.17816024588547713, -2.5])
def test_spmm_shift_bitwise(dev, oracle, c1, alpha):
    at = oracle.transpose(c1)
    rng = np.random.default_rng(9)
    y = np.asfortranarray(rng.standard_normal((c1.rows, 75)))
    q = np.asfortranarray(rng.standard_normal((c1.cols, 75)))
    t_ref = oracle.spmm(at, y)
    if alpha != 0.0:
        t_ref = oracle.add_scaled(t_ref, -alpha, q)
    t = d.spmm_shift(to_dev(at), y, alpha, q, device=dev)
    assert_bitwise(t, t_ref)


def test_spmm_power_law_long_rows_bitwise(oracle):
    dv = d.Device(0)
    dv.set_option("split_chunk", 0)  # whole chains: bit-exact
    a = d.powerlaw(4000, 2000, 3.5, 1.0, 1.1, 8)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    at = transpose_np(ca)
    x = np.asfortranarray(np.random.default_rng(1).standard_normal((ca.rows, 150)))
    assert_bitwise(d.spmm(to_dev(at), x, device=dv), oracle.spmm(at, x))


@pytest.mark.parametrize("panel", [0, 777])
@pytest.mark.parametrize("chunk", [7, 32, 100, 2048])
@pytest.mark.parametrize("l", [1, 75, 150])
def test_spmm_split_rows_match(oracle, chunk, l, panel):
    """Split mode: long rows as chunk partials summed in chunk order. Not the
    reference's single chain, so checked against the rounding-error scale
    (|A| |X|) rather than bitwise. panel: the transpose's chunks are also cut
    at multiples of `panel` gathered rows and listed panel by panel."""
    dv = d.Device(0)
    dv.set_option("split_chunk", chunk)
    dv.set_option("split_panel_rows", panel)  # no effect here: panels apply to the transpose of a solve
    a = d.powerlaw(6000, 2500, 3.5, 1.0, 1.1, 21)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    at = transpose_np(ca)
    rng = np.random.default_rng(chunk + l)
    for m, x in ((ca, rng.standard_normal((ca.cols, l))), (at, rng.standard_normal((ca.rows, l)))):
        x = np.asfortranarray(x)
        y_ref = oracle.spmm(m, x)
        scale = oracle.spmm(Csr(m.rows, m.cols, m.offsets, m.col_indices, np.abs(m.values)),
                            np.asfortranarray(np.abs(x)))
        y = d.spmm(to_dev(m), x, device=dv)
        assert np.all(np.abs(y - y_ref) <= 1e-13 * scale + 1e-300)
        q = np.asfortranarray(rng.standard_normal((m.rows, l)))
        t = d.spmm_shift(to_dev(m), x, 0.25, q, device=dv)
        t_ref = oracle.add_scaled(y_ref, -0.25, q)
        assert np.all(np.abs(t - t_ref) <= 1e-13 * (scale + 0.25 * np.abs(q)) + 1e-300)
        # rows that were not split keep their exact chains
        short = np.diff(m.offsets) <= chunk
        assert_bitwise(y[short], y_ref[short])


def test_solve_power_law_split_vs_bitwise(oracle):
    a = d.powerlaw(8000, 3000, 3.5, 1.0, 1.1, 4)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    ref = oracle.solve(ca, 20, 10, p=6, alg="shifted", seed=1)
    cfg = d.SolverConfig(k=20, s=10, p=6, alg=d.Algorithm.shifted, seed=1)
    # (split_chunk, split_panel_rows): whole chains; chunks; chunks cut and
    # ordered by 500- / 333-row panels of the gathered Y (pass 2)
    for chunk, panel in ((0, 0), (64, 0), (64, 500), (7, 333)):
        dv = d.Device(0)
        dv.set_option("split_chunk", chunk)
        dv.set_option("split_panel_rows", panel)
        res = d.solve(a, cfg, device=dv)
        check_solve(res, ref, 20)


@pytest.fixture()
def hub_dev():
    """A context whose SpMM sends every row with >= threshold nonzeros down the
    hub (cp.async ring) path, so small matrices exercise it."""
    dv = d.Device(0)
    dv.set_option("split_chunk", 0)
    yield dv
    dv.close()


@pytest.mark.parametrize("threshold", [1, 9, 33, 200])
@pytest.mark.parametrize("l", [1, 31, 75, 150, 300])
def test_spmm_hub_path_bitwise(hub_dev, oracle, c1, threshold, l):
    hub_dev.set_option("hub_threshold", threshold)
    at = oracle.transpose(c1)
    rng = np.random.default_rng(threshold + l)
    y = np.asfortranarray(rng.standard_normal((c1.rows, l)))
    q = np.asfortranarray(rng.standard_normal((c1.cols, l)))
    assert_bitwise(d.spmm(to_dev(at), y, device=hub_dev), oracle.spmm(at, y))
    t_ref = oracle.add_scaled(oracle.spmm(at, y), -0.37, q)
    assert_bitwise(d.spmm_shift(to_dev(at), y, 0.37, q, device=hub_dev), t_ref)


def test_spmm_hub_power_law_bitwise(hub_dev, oracle):
    hub_dev.set_option("hub_threshold", 64)
    a = d.powerlaw(20000, 3000, 3.5, 1.0, 1.1, 12)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    at = transpose_np(ca)
    assert np.diff(at.offsets).max() > 5000  # real hub rows
    x = np.asfortranarray(np.random.default_rng(2).standard_normal((ca.rows, 150)))
    assert_bitwise(d.spmm(to_dev(at), x, device=hub_dev), oracle.spmm(at, x))
    x = np.asfortranarray(np.random.default_rng(3).standard_normal((ca.cols, 150)))
    assert_bitwise(d.spmm(a, x, device=hub_dev), oracle.spmm(ca, x))


def test_solve_hub_path(hub_dev, oracle, c1):
    hub_dev.set_option("hub_threshold", 40)
    ref = oracle.solve(c1, 50, 25, p=10, alg="shifted", seed=0)
    res = d.solve(to_dev(c1), d.SolverConfig(k=50, s=25, p=10, alg=d.Algorithm.shifted, seed=0),
                  device=hub_dev)
    check_solve(res, ref, 50)


# ---- RNG ------------------------------------------------------------------------

def test_splitmix_pins():
    # test_dense_core.cpp:23-30
    assert d.splitmix64_at(0, 0) == 0xe220a8397b1dcdaf
    assert d.splitmix64_at(0, 1) == 0x6e789e6aa1b965f4
    assert d.splitmix64_at(42, 0) == 0xbdd732262feb6e95
    assert d.splitmix64_at(2026, 0) == 0xdb9c559891948d23
    assert d.splitmix64_at(0x8000000000000000, 5) == 0x4d7e6a268a67c5ff


def test_gaussian_pins(dev):
    # normal_at pins (test_dense_core.cpp:36-41) through the device generator
    g = d.gaussian_matrix(4, 1, 42, device=dev)
    assert g[0, 0] == float.fromhex("0x1.a8ac4b546f505p-2")
    assert g[1, 0] == float.fromhex("-0x1.c8a54f4e91a80p-1")
    assert g[2, 0] == float.fromhex("0x1.bac69cd4142c4p+0")
    assert g[3, 0] == float.fromhex("0x1.175b8fd2de8c7p-1")
    assert d.gaussian_matrix(1, 1, 7, device=dev)[0, 0] == float.fromhex("0x1.5d70229cdee62p+0")
    assert d.gaussian_matrix(1, 1, 2026, device=dev)[0, 0] == float.fromhex("-0x1.170735b18c9d6p-1")
    # checksum pin (test_dense_core.cpp:59-61)
    g = d.gaussian_matrix(8, 4, 2026, device=dev)
    assert int(bits(g.ravel(order="F")).sum(dtype=np.uint64)) == 0x7bb02d1fc95596ff


def test_gaussian_config1_sketch_agreement(dev, oracle):
    g_ref = oracle.gaussian_matrix(10000, 75, 0)
    g = d.gaussian_matrix(10000, 75, 0, device=dev)
    mism = int(np.count_nonzero(bits(g.ravel(order="F")) != bits(g_ref.ravel(order="F"))))
    # every entry within 2 ulp; the count of 1-ulp differences is reported
    np.testing.assert_allclose(g, g_ref, rtol=5e-16, atol=0)
    print(f"config-1 Omega: {mism} of {g.size} entries differ from glibc by <= 1 ulp")
    assert int(bits(g_ref.ravel(order="F")).sum(dtype=np.uint64)) == 0xab4330ec8cf8afc5


# ---- dense kernels -----------------------------------------------------------------

@pytest.fixture(params=[0, 1], ids=["dmma", "dfma"])
def dense_dev(request):
    """Gram / rescale on FP64 tensor cores (dense_method 0) or DFMA (1)."""
    dv = d.Device(0)
    dv.set_option("dense_method", request.param)
    yield dv
    dv.close()


@pytest.mark.parametrize("shape", [(10000, 75), (777, 150), (5000, 300), (40, 3), (200003, 150), (9, 160),
                                   (1000, 8), (1000, 1), (4000, 161), (3001, 257), (2500, 512), (70, 300),
                                   (300001, 300), (6000, 312), (3000, 320), (2000, 216), (2000, 184)])
def test_gram_matches_oracle(dense_dev, oracle, shape):
    c = np.asfortranarray(np.random.default_rng(shape[1]).standard_normal(shape))
    g_ref = oracle.gram(c)
    g = d.gram(c, device=dense_dev)
    assert np.array_equal(g, g.T)  # exactly symmetric
    np.testing.assert_allclose(g, g_ref, rtol=1e-13, atol=1e-13 * np.abs(g_ref).max())


@pytest.mark.parametrize("shape", [(5000, 300), (70, 300), (300001, 300), (6000, 312), (3000, 320),
                                   (2000, 216), (2000, 184), (4000, 161), (3001, 257), (1000, 170)])
def test_wide_gram_tile_shapes_are_bitwise_equal(oracle, shape):
    """The wide DMMA Gram with 2x2 tiles of 8x8 blocks (default) and with 4x4
    tiles issues the same block products in the same k order: bitwise equal."""
    c = np.asfortranarray(np.random.default_rng(shape[1] + 7).standard_normal(shape))
    dv = d.Device(0)
    try:
        dv.set_option("gram_tiles", 4)
        g4 = d.gram(c, device=dv)
        dv.set_option("gram_tiles", 2)
        g2 = d.gram(c, device=dv)
    finally:
        dv.set_option("gram_tiles", 2)
        dv.close()
    assert_bitwise(g2, g4)
    g_ref = oracle.gram(c)
    np.testing.assert_allclose(g2, g_ref, rtol=1e-13, atol=1e-13 * np.abs(g_ref).max())


@pytest.mark.parametrize("shape", [(300, 75, 75), (1000, 150, 100), (17, 5, 3)])
def test_matmul_bitwise(dev, oracle, shape):
    m, kk, n = shape
    rng = np.random.default_rng(m)
    a = np.asfortranarray(rng.standard_normal((m, kk)))
    b = np.asfortranarray(rng.standard_normal((kk, n)))
    assert_bitwise(d.matmul(a, b, device=dev), oracle.matmul(a, b))


@pytest.mark.parametrize("n", [1, 2, 3, 20, 75, 150, 161, 200, 257, 300, 320])
def test_sym_eig_matches_oracle(dev, oracle, n):
    g0 = np.random.default_rng(n).standard_normal((n, n))
    g = np.asfortranarray(g0 + g0.T)
    w_ref, v_ref = oracle.sym_eig(g)
    e = d.sym_eig(g, device=dev)
    scale = np.abs(w_ref).max()
    np.testing.assert_allclose(e.values, w_ref, rtol=0, atol=1e-12 * scale)
    assert np.all(np.diff(e.values) >= 0)
    np.testing.assert_allclose(e.vectors.T @ e.vectors, np.eye(n), atol=1e-12)
    np.testing.assert_allclose(g @ e.vectors, e.vectors * e.values, atol=1e-11 * scale)


def test_sym_eig_known_cases(dev):
    # test_dense_core.cpp:88-104
    e = d.sym_eig(np.array([[2.0, 0.0], [0.0, 5.0]]), device=dev)
    assert e.values[0] == pytest.approx(2.0, rel=1e-14) and e.values[1] == pytest.approx(5.0, rel=1e-14)
    e = d.sym_eig(np.array([[0.0, 1.0], [1.0, 0.0]]), device=dev)
    assert e.values[0] == pytest.approx(-1.0, rel=1e-14) and e.values[1] == pytest.approx(1.0, rel=1e-14)
    e = d.sym_eig(np.array([[4.0]]), device=dev)
    assert e.values[0] == 4.0 and abs(e.vectors[0, 0]) == 1.0
    with pytest.raises(d.ShapeError):
        d.sym_eig(np.array([[1.0, 2.0], [1.0, 1.0]]), device=dev)


def test_eig_svd_clustered_spectrum_falls_back(eig_dev):
    # identity-like and repeated singular values: the tridiagonal path must
    # hand over to Jacobi and still return orthonormal factors
    f = d.eig_svd(np.eye(40), device=eig_dev)
    np.testing.assert_allclose(f.s, np.ones(40), rtol=1e-13)
    np.testing.assert_allclose(f.u @ f.v.T, np.eye(40), atol=1e-12)
    q, _ = np.linalg.qr(np.random.default_rng(5).standard_normal((300, 30)))
    sv = np.repeat([5.0, 3.0, 1.0], 10)
    c = np.asfortranarray(q * sv)
    f = d.eig_svd(c, device=eig_dev)
    np.testing.assert_allclose(f.s, sv, rtol=1e-12)
    np.testing.assert_allclose(f.v.T @ f.v, np.eye(30), atol=1e-12)
    np.testing.assert_allclose((f.u * f.s) @ f.v.T, c, atol=1e-11)


@pytest.mark.parametrize("gap", [1e-9, 1e-10, 1e-11, 3e-12])
def test_eig_svd_close_pairs_stay_accurate(dev, oracle, gap):
    # nearly repeated pairs (relative gaps 1e-9 .. 3e-12, as the R-MAT Gram
    # matrices of C4 have): the tridiagonal path keeps them (no fallback above
    # 1e-12) and the factors stay orthonormal and accurate
    rng = np.random.default_rng(int(-np.log10(gap) * 10))
    n, l = 3000, 200
    q, _ = np.linalg.qr(rng.standard_normal((n, l)))
    w, _ = np.linalg.qr(rng.standard_normal((l, l)))
    sv = np.sort(rng.uniform(1.0, 10.0, l))[::-1]
    for i in range(0, 40, 4):  # ten pairs whose squares differ by gap * sigma_1^2
        sv[i + 1] = np.sqrt(sv[i] ** 2 - gap * sv[0] ** 2)
    c = np.asfortranarray((q * sv) @ w.T)
    f = d.eig_svd(c, device=dev)
    u_ref, s_ref, v_ref = oracle.eig_svd(c)
    # eigenvalues of the Gram to ~l eps ||G||: sigma to ~1e-12 relative at sigma_1 / sigma_l = 10
    np.testing.assert_allclose(f.s, s_ref, rtol=1e-11)
    np.testing.assert_allclose(f.v.T @ f.v, np.eye(l), atol=1e-12)
    np.testing.assert_allclose(f.u.T @ f.u, np.eye(l), atol=1e-10)
    np.testing.assert_allclose((f.u * f.s) @ f.v.T, c, atol=1e-11 * sv[0])


def test_solve_config1_both_eigensolvers(oracle, c1, eig_dev):
    ref = oracle.solve(c1, 50, 25, tol=1e-2, alg="dash", seed=0)
    res = d.solve(to_dev(c1), d.SolverConfig(k=50, s=25, tol=1e-2, seed=0), device=eig_dev)
    check_solve(res, ref, 50)


@pytest.mark.parametrize("k,s", [(50, 25), (100, 50), (7, 3), (140, 20)])
def test_solve_config1_dense_methods(oracle, c1, dense_dev, k, s):
    # l = k + s spans the tensor-core shapes: odd widths, l = 160, tiny l
    ref = oracle.solve(c1, k, s, p=6, alg="shifted", seed=3)
    res = d.solve(to_dev(c1), d.SolverConfig(k=k, s=s, p=6, alg=d.Algorithm.shifted, seed=3), device=dense_dev)
    check_solve(res, ref, k)


def test_eig_svd_known_cases(dev):
    # test_dense_core.cpp:134-154
    f = d.eig_svd(np.array([[3.0, 0.0], [0.0, 4.0], [0.0, 0.0]]), device=dev)
    np.testing.assert_allclose(f.s, [4.0, 3.0], rtol=1e-14)
    np.testing.assert_allclose(f.v, [[0.0, 1.0], [1.0, 0.0]], atol=1e-14)
    np.testing.assert_allclose(f.u, [[0.0, 1.0], [1.0, 0.0], [0.0, 0.0]], atol=1e-14)
    f = d.eig_svd(np.array([[3.0, 0.0], [4.0, 5.0]]), device=dev)
    np.testing.assert_allclose(f.s, [np.sqrt(45.0), np.sqrt(5.0)], rtol=1e-13)


def test_eig_svd_rank_deficient(dev):
    # test_dense_core.cpp:173-193
    from oracle_lib import Oracle
    c = Oracle().gaussian_matrix(6, 2, 1)
    c[:, 1] = 0.0
    with pytest.raises(d.RankDeficient) as ei:
        d.eig_svd(c, device=dev)
    assert ei.value.index == 1
    with pytest.raises(d.RankDeficient) as ei:
        d.eig_svd(np.zeros((5, 2)), device=dev)
    assert ei.value.index == 0
    with pytest.raises(d.ShapeError):
        d.eig_svd(np.zeros((2, 3)), device=dev)


@pytest.fixture(params=[0, 1], ids=["tridiagonal", "jacobi"])
def eig_dev(request):
    dv = d.Device(0)
    dv.set_option("eig_method", request.param)
    yield dv
    dv.close()


@pytest.mark.parametrize("shape", [(10000, 75), (5000, 150), (2000, 300), (400, 3), (900, 64), (3000, 200),
                                   (4000, 320)])
def test_eig_svd_matches_oracle(eig_dev, oracle, shape):
    c = np.asfortranarray(np.random.default_rng(shape[0]).standard_normal(shape))
    u_ref, s_ref, v_ref = oracle.eig_svd(c)
    f = d.eig_svd(c, device=eig_dev)
    np.testing.assert_allclose(f.s, s_ref, rtol=1e-12)
    # same sign convention -> same vectors up to roundoff
    np.testing.assert_allclose(f.v, v_ref, atol=1e-10)
    np.testing.assert_allclose(f.u, u_ref, atol=1e-10)


# ---- solver (tolerance parity, north_star bars) --------------------------------------

def _pve_ratio(res, k):
    s = res["s_hat"] if isinstance(res, dict) else np.array(res.trace.s_hat_history)
    a = res["alphas"] if isinstance(res, dict) else np.array(res.trace.alphas)
    n = len(a)
    if n < 2:
        return None
    prev, cur = s[n - 2], s[n - 1]
    ap = a[n - 1]  # alpha_stored after iteration n-1 == alpha used in iteration n
    denom = cur[k] + a[n - 1]
    return float(np.max(np.abs(prev[:k] + ap - cur[:k] - a[n - 1]) / denom))


def check_solve(res, ref, k, sv_rtol=1e-8, angle=1e-6):
    np.testing.assert_allclose(res.svd.s, ref["s"], rtol=sv_rtol)
    assert sin_theta(ref["u"], res.svd.u) <= angle
    assert sin_theta(ref["v"], res.svd.v) <= angle
    assert res.trace.iterations == ref["iterations"]
    assert res.trace.stop_reason.name == ref["stop_reason"]
    np.testing.assert_allclose(res.trace.alphas, ref["alphas"], rtol=1e-8, atol=1e-300)
    if ref["iterations"]:
        np.testing.assert_allclose(np.array(res.trace.s_hat_history), ref["s_hat"], rtol=1e-8)


def test_solve_config1_shifted(dev, oracle, c1):
    ref = oracle.solve(c1, 50, 25, p=10, alg="shifted", seed=0)
    res = d.solve(to_dev(c1), d.SolverConfig(k=50, s=25, p=10, alg=d.Algorithm.shifted, seed=0),
                  device=dev)
    check_solve(res, ref, 50)
    # the published probe values
    assert res.svd.s[0] == pytest.approx(4.3734243453278507, rel=1e-12)
    assert res.svd.s[49] == pytest.approx(0.73000858905607624, rel=1e-10)


def test_solve_config1_dash(dev, oracle, c1):
    ref = oracle.solve(c1, 50, 25, tol=1e-2, alg="dash", seed=0)
    res = d.dash_svd(to_dev(c1), d.SolverConfig(k=50, s=25, tol=1e-2, seed=0), device=dev)
    check_solve(res, ref, 50)
    assert res.trace.iterations == 7
    r_ref = _pve_ratio(ref, 50)
    r = _pve_ratio(res, 50)
    assert r == pytest.approx(r_ref, rel=1e-6)


def test_solve_fixed_shift(dev, oracle):
    a = oracle.sparse_random(50, 35, 6, 21, True)
    ref = oracle.solve(a, 5, 3, p=4, alg="fixed_shift")
    res = d.shifted_rsvd(to_dev(a), d.SolverConfig(k=5, s=3, p=4, alg=d.Algorithm.fixed_shift),
                         device=dev)
    check_solve(res, ref, 5)
    assert res.trace.alphas[2] == res.trace.alphas[1] == res.trace.alphas[3]


def test_solve_wide_orientation(dev, oracle):
    wide = oracle.sparse_random(60, 100, 8, 44, True)
    cfg = d.SolverConfig(k=8, s=4, seed=2)
    ref = oracle.solve(wide, 8, 4, tol=1e-2, alg="dash", seed=2)
    res = d.solve(to_dev(wide), cfg, device=dev)
    assert res.svd.u.shape == (60, 8) and res.svd.v.shape == (100, 8)
    check_solve(res, ref, 8)


def test_solve_p0_and_tiny(dev, oracle):
    a = oracle.sparse_random(40, 25, 6, 77, True)
    ref = oracle.solve(a, 5, 5, p=0, alg="shifted")
    res = d.solve(to_dev(a), d.SolverConfig(k=5, s=5, p=0, alg=d.Algorithm.shifted), device=dev)
    check_solve(res, ref, 5)


def test_solve_stop_reasons(dev, oracle):
    a = oracle.sparse_random(60, 40, 6, 5, True)
    r = d.dash_svd(to_dev(a), d.SolverConfig(k=5, s=3, tol=1e9), device=dev)
    assert r.trace.iterations == 1 and r.trace.stop_reason == d.StopReason.tol_met
    r = d.dash_svd(to_dev(a), d.SolverConfig(k=5, s=3, tol=1e-15, p_max=3), device=dev)
    assert r.trace.iterations == 3 and r.trace.stop_reason == d.StopReason.p_max_reached


def test_solve_dash_equals_shifted_at_stop(dev):
    # test_rsvd.cpp:317-339: the accuracy-controlled run is bitwise the
    # fixed-count run at the same iteration count (same device path)
    from oracle_lib import Oracle
    a = to_dev(Oracle().sparse_random(150, 90, 8, 6, True))
    dr = d.dash_svd(a, d.SolverConfig(k=12, s=6, tol=1e-2, seed=17), device=dev)
    assert dr.trace.stop_reason == d.StopReason.tol_met
    fr = d.shifted_rsvd(a, d.SolverConfig(k=12, s=6, p=dr.trace.iterations, seed=17), device=dev)
    assert_bitwise(dr.svd.u, fr.svd.u)
    assert_bitwise(dr.svd.s, fr.svd.s)
    assert_bitwise(dr.svd.v, fr.svd.v)
    assert_bitwise(dr.trace.alphas, fr.trace.alphas)


def test_solve_deterministic(dev, c1):
    cfg = d.SolverConfig(k=50, s=25, p=4, alg=d.Algorithm.shifted)
    r1 = d.solve(to_dev(c1), cfg, device=dev)
    r2 = d.solve(to_dev(c1), cfg, device=dev)
    assert_bitwise(r1.svd.u, r2.svd.u)
    assert_bitwise(r1.svd.v, r2.svd.v)
    assert_bitwise(r1.svd.s, r2.svd.s)


def test_concurrent_contexts_on_threads(c1):
    """One context per thread (the documented pattern for concurrent solves,
    dashsvd_b200.h): four threads solving at once on one GPU give the same bits
    as a solve alone."""
    import threading
    a = to_dev(c1)
    cfgs = [d.SolverConfig(k=20, s=10, p=3, alg=d.Algorithm.shifted, seed=s) for s in range(4)]
    alone = [d.solve(a, c, device=d.Device(0)) for c in cfgs]
    out = [None] * 4
    errors = []

    def work(t):
        try:
            dv = d.Device(0)
            out[t] = d.solve(a, cfgs[t], device=dv)
            dv.close()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for r, r0 in zip(out, alone):
        assert_bitwise(r.svd.s, r0.svd.s)
        assert_bitwise(r.svd.u, r0.svd.u)


@pytest.mark.parametrize("alg", ["shifted", "dash"])
def test_sharded_path_single_rank(oracle, c1, alg):
    """The multi-GPU code path (NCCL communicator, shard bookkeeping, all-reduce
    of the n x l partials, shift after the sum, all-reduced finalize Gram) run
    with a one-rank communicator on the one GPU: it must reproduce the
    single-GPU solve bitwise (one rank's all-reduce is the identity and the
    separate shift kernel does the same fma as the fused epilogue)."""
    cfg = (d.SolverConfig(k=50, s=25, p=6, alg=d.Algorithm.shifted, seed=0) if alg == "shifted"
           else d.SolverConfig(k=50, s=25, tol=1e-2, seed=0))
    plain = d.Device(0)
    r_ref = d.solve(to_dev(c1), cfg, device=plain)
    sh = d.Device(0)
    sh.attach_comm(1, 0, d.comm_unique_id())
    sh.set_shard(0, c1.rows)
    r = d.solve(to_dev(c1), cfg, device=sh)
    assert r.trace.iterations == r_ref.trace.iterations
    assert_bitwise(r.svd.s, r_ref.svd.s)
    assert_bitwise(r.svd.u, r_ref.svd.u)
    assert_bitwise(r.svd.v, r_ref.svd.v)
    ref = oracle.solve(c1, 50, 25, p=6, alg="shifted", seed=0) if alg == "shifted" else \
        oracle.solve(c1, 50, 25, tol=1e-2, alg="dash", seed=0)
    check_solve(r, ref, 50)
    sh.close()
    plain.close()


def test_observer_and_snapshot_finalize(dev, oracle):
    # test_rsvd.cpp:341-389 + :424-458 on the device path
    a = oracle.sparse_random(60, 40, 6, 33, True)
    seen = []
    cfg = d.SolverConfig(k=6, s=3, p=5, alg=d.Algorithm.shifted)
    full = d.shifted_rsvd(to_dev(a), cfg, observer=lambda st: seen.append(st), device=dev)
    assert [s.iteration for s in seen] == [1, 2, 3, 4, 5]
    for c, st in enumerate(seen):
        assert st.alpha == full.trace.alphas[c]
        assert_bitwise(st.s_hat, full.trace.s_hat_history[c])
        assert st.q_after.shape == (40, 9)
        np.testing.assert_allclose(st.q_after.T @ st.q_after, np.eye(9), atol=1e-9)
        if c:
            assert_bitwise(st.q_before, seen[c - 1].q_after)
    short = d.shifted_rsvd(to_dev(a), d.SolverConfig(k=6, s=3, p=3, alg=d.Algorithm.shifted),
                           device=dev)
    fin = d.finalize_row_basis(to_dev(a), seen[2].q_after, 6, device=dev)
    assert_bitwise(fin.u, short.svd.u)
    assert_bitwise(fin.s, short.svd.s)
    assert_bitwise(fin.v, short.svd.v)


def test_config_errors(dev):
    a = d.SparseMatrix(40, 30, np.arange(41) * 0, np.zeros(0), np.zeros(0))
    with pytest.raises(d.ConfigError):
        d.solve(a, d.SolverConfig(k=25, s=10, p=4, alg=d.Algorithm.shifted), device=dev)
    with pytest.raises(d.ConfigError):
        d.solve(a, d.SolverConfig(k=4, s=0), device=dev)
    with pytest.raises(d.ConfigError):
        d.solve(a, d.SolverConfig(k=4, s=2, alg=d.Algorithm.shifted), device=dev)


def test_rank_one_raises_rank_deficient(dev):
    # test_rsvd.cpp:152-175: a wider sketch than the rank hits the rank floor
    u = np.array([[2 / 3], [-1 / 3], [2 / 3]])
    v = np.array([[0.6], [0.8]])
    dense = 6.0 * u @ v.T
    rows, cols = np.nonzero(dense)
    off = np.zeros(4, dtype=np.int64)
    np.add.at(off, rows + 1, 1)
    off = np.cumsum(off)
    a = d.SparseMatrix(3, 2, off, cols, dense[rows, cols])
    with pytest.raises(d.RankDeficient):
        d.solve(a, d.SolverConfig(k=1, s=1, p=1, alg=d.Algorithm.shifted), device=dev)


# ---- basic algorithm (Alg. 1) -------------------------------------

@pytest.mark.parametrize("shape", [(3000, 1800), (1500, 2600)])
@pytest.mark.parametrize("p", [0, 1, 4])
def test_solve_basic_eigsvd(dev, oracle, shape, p):
    a = oracle.sparse_random(shape[0], shape[1], 12, 5, True)
    ref = oracle.solve(a, 20, 10, p=p, alg="basic", seed=4)
    res = d.solve(to_dev(a), d.SolverConfig(k=20, s=10, p=p, alg=d.Algorithm.basic, seed=4), device=dev)
    check_solve(res, ref, 20)
    assert np.all(np.asarray(res.trace.alphas) == 0.0) and len(res.trace.alphas) == p
    assert res.trace.stop_reason.name == "fixed_p"


def test_basic_rsvd_direct_and_observer(dev, oracle, c1):
    # basic_rsvd runs on `a` as given (solver.cpp:178-184); observer sees q (m x l)
    ref = oracle.solve(c1, 30, 10, p=3, alg="basic", seed=1)
    seen = []
    cfg = d.SolverConfig(k=30, s=10, p=3, seed=1)
    f = d.basic_rsvd(to_dev(c1), cfg, observer=lambda st: seen.append(st), device=dev)
    np.testing.assert_allclose(f.s, ref["s"], rtol=1e-8)
    assert sin_theta(ref["u"], f.u) <= 1e-6 and sin_theta(ref["v"], f.v) <= 1e-6
    assert [st.iteration for st in seen] == [1, 2, 3]
    for j, st in enumerate(seen):
        assert st.alpha == 0.0 and st.q_after.shape == (c1.rows, 40)
        np.testing.assert_allclose(st.q_after.T @ st.q_after, np.eye(40), atol=1e-9)
        np.testing.assert_allclose(st.s_hat, ref["s_hat"][j], rtol=1e-8)


@pytest.mark.parametrize("shape", [(3000, 1800), (1500, 2600)])
@pytest.mark.parametrize("p", [0, 2])
def test_solve_basic_qr(dev, oracle, shape, p):
    """Basic algorithm with the QR orthonormalizer: CholeskyQR2 + Householder
    sign reconstruction on the device vs the reference's Householder qr_orth."""
    a = oracle.sparse_random(shape[0], shape[1], 12, 6, True)
    ref = oracle.solve(a, 20, 10, p=p, alg="basic", seed=2, orth="qr")
    cfg = d.SolverConfig(k=20, s=10, p=p, alg=d.Algorithm.basic, seed=2, orth=d.Orthonormalizer.qr)
    res = d.solve(to_dev(a), cfg, device=dev)
    np.testing.assert_allclose(res.svd.s, ref["s"], rtol=1e-8)
    assert sin_theta(ref["u"], res.svd.u) <= 1e-6 and sin_theta(ref["v"], res.svd.v) <= 1e-6
    assert res.trace.iterations == p and all(len(h) == 0 for h in res.trace.s_hat_history)
    np.testing.assert_allclose(res.trace.alphas, np.zeros(p))


def test_basic_qr_observer_q_matches_householder(dev, oracle):
    """The iterate q of the device QR orthonormalizer equals the reference's
    Householder Q column for column (signs included)."""
    a = oracle.sparse_random(900, 500, 10, 3, True)
    at = oracle.transpose(a)
    seen = []
    cfg = d.SolverConfig(k=12, s=6, p=2, alg=d.Algorithm.basic, seed=5, orth=d.Orthonormalizer.qr)
    d.basic_rsvd(to_dev(a), cfg, observer=lambda st: seen.append(st), device=dev)
    assert len(seen) == 2
    for st in seen:
        # the reference's qr_orth of the same block (A A^T q_before)
        y = oracle.spmm(a, oracle.spmm(at, np.asfortranarray(st.q_before)))
        q_ref = oracle.qr_orth(y)
        np.testing.assert_allclose(st.q_after, q_ref, atol=1e-10)


def test_basic_qr_rank_deficient(dev):
    # identical columns -> dependent sketch columns -> RankDeficient like qr_orth
    off = np.arange(0, 2 * 401, 2, dtype=np.int64)
    idx = np.tile(np.array([0, 1], dtype=np.int64), 400)
    val = np.ones(800)
    a = d.SparseMatrix(400, 60, off, idx, val)
    cfg = d.SolverConfig(k=4, s=2, p=1, alg=d.Algorithm.basic, seed=1, orth=d.Orthonormalizer.qr)
    with pytest.raises(d.errors.RankDeficient):
        d.solve(a, cfg, device=dev)


# ---- validation metrics on the device ---------------------------

def _dense(a):
    m = np.zeros((a.rows, a.cols))
    for i in range(a.rows):
        for p in range(a.offsets[i], a.offsets[i + 1]):
            m[i, a.col_indices[p]] += a.values[p]
    return m


@pytest.mark.parametrize("p", [0, 2])
def test_metrics_match_reference(dev, oracle, reference, p):
    a = oracle.sparse_random(1200, 700, 9, 8, True)
    sig = np.linalg.svd(_dense(a), compute_uv=False)
    res = d.solve(to_dev(a), d.SolverConfig(k=20, s=10, p=p, alg=d.Algorithm.shifted, seed=3), device=dev)
    f = res.svd
    ref = reference.metrics(a, f.u, f.s, f.v, sig, power_iters=120, seed=11)
    got = np.array([d.eps_pve(to_dev(a), f.u, sig, device=dev), d.eps_res(to_dev(a), f, sig, device=dev),
                    d.eps_spec(to_dev(a), f, sig, power_iters=120, seed=11, device=dev),
                    d.max_triplet_residual(to_dev(a), f, device=dev)])
    # reductions differ from the reference's sequential sums only by rounding
    np.testing.assert_allclose(got[[0, 1, 3]], ref[[0, 1, 3]], rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-6, atol=1e-9)


def test_metrics_degenerate_reference(dev, oracle):
    a = oracle.sparse_random(300, 200, 6, 2, True)
    f = d.solve(to_dev(a), d.SolverConfig(k=5, s=5, p=1, alg=d.Algorithm.shifted), device=dev).svd
    with pytest.raises(d.DegenerateReference):
        d.eps_pve(to_dev(a), f.u, f.s, device=dev)  # needs k + 1 values
    with pytest.raises(d.DegenerateReference):
        d.eps_spec(to_dev(a), f, np.r_[f.s, 0.0], device=dev)  # sigma_{k+1} == 0
    assert d.max_triplet_residual(to_dev(a), f, device=dev) < 1e-3 * f.s[0]


@pytest.mark.parametrize("alg,kw", [("shifted", dict(p=8)), ("dash", dict(tol=1e-2)),
                                    ("fixed_shift", dict(p=5))])
def test_loop_schedules_agree(oracle, alg, kw):
    """The pipelined loop (deferred rescale: both SpMM passes on T_{j-1}, the
    l x l eig on the priority stream beside the A T pass; engine.cu solve_tall,
    option pipeline = 1, the default) and the serial loop in the reference's
    order (pipeline = 0) both meet the solve bars against the oracle, take the
    same stop decisions, and agree with each other far inside them."""
    a = d.powerlaw(6000, 2500, 3.5, 1.0, 1.1, 9)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    ref = oracle.solve(ca, 24, 12, alg=alg, seed=5, **kw)
    cfg = d.SolverConfig(k=24, s=12, alg=d.Algorithm[alg], seed=5, **kw)
    out = []
    for pipe in (1, 0):
        dv = d.Device(0)
        dv.set_option("pipeline", pipe)
        res = d.solve(a, cfg, device=dv)
        check_solve(res, ref, 24)
        out.append(res)
        dv.close()
    p1, p0 = out
    assert p1.trace.iterations == p0.trace.iterations
    np.testing.assert_allclose(p1.svd.s, p0.svd.s, rtol=1e-11)
    assert sin_theta(p0.svd.u, p1.svd.u) <= 1e-9
    assert sin_theta(p0.svd.v, p1.svd.v) <= 1e-9


def test_loop_options_validated():
    dv = d.Device(0)
    for name, bad in (("pipeline", 2), ("pipeline", -2), ("gram_async", 2), ("shift_after", -1),
                      ("eig_priority", 3), ("eig_overlap", 3), ("eig_overlap", -2)):
        with pytest.raises(d.ConfigError):
            dv.set_option(name, bad)
    for name, good in (("pipeline", -1), ("pipeline", 0), ("pipeline", 1), ("gram_async", 0),
                       ("shift_after", 0), ("eig_priority", 1), ("eig_priority", 0), ("eig_overlap", -1),
                       ("eig_overlap", 0), ("eig_overlap", 1), ("eig_overlap", 2)):
        dv.set_option(name, good)
    with pytest.raises(d.ConfigError):
        dv.set_option("no_such_option", 1)
    dv.close()


@pytest.mark.parametrize("base,opts", [({}, dict(shift_after=1)), ({}, dict(gram_async=1)),
                                       ({}, dict(eig_priority=0)), ({}, dict(eig_overlap=0)),
                                       ({}, dict(eig_overlap=2)),
                                       # Jacobi: no tridiagonalisation to split, 2 acts as 1
                                       (dict(eig_method=1), dict(eig_method=1, eig_overlap=2))])
def test_pipelined_variants_are_bitwise_equal(oracle, base, opts):
    """The schedule variants of the pipelined loop move work between streams but
    compute the same values in the same order: bitwise equal factors."""
    a = d.powerlaw(5000, 2000, 3.5, 1.0, 1.1, 2)
    cfg = d.SolverConfig(k=16, s=8, tol=1e-2, seed=2)
    res = []
    for extra in (base, opts):
        dv = d.Device(0)
        dv.set_option("pipeline", 1)
        for k_, v_ in extra.items():
            dv.set_option(k_, v_)
        res.append(d.solve(a, cfg, device=dv))
        dv.close()
    assert res[0].trace.iterations == res[1].trace.iterations
    for name in ("u", "s", "v"):
        assert_bitwise(getattr(res[0].svd, name), getattr(res[1].svd, name))


@pytest.mark.parametrize("alg,kw", [("dash", dict(tol=2e-2)), ("shifted", dict(p=5))])
def test_eig_overlap_wide_sketch(oracle, alg, kw):
    """l = 180 (> 160: the wide tridiagonalisation, where the default splits the
    eig chain: tridiagonalisation beside the A T pass, the rest after it on the
    main stream). Every placement of the chain gives the same bits, and the
    solve meets the bars against the oracle (dash: the deferred stop flags keep
    N_p and the stop reason)."""
    a = d.powerlaw(3000, 1500, 3.0, 1.0, 1.1, 5)
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    ref = oracle.solve(ca, 120, 60, alg=alg, seed=5, **kw)
    cfg = d.SolverConfig(k=120, s=60, alg=d.Algorithm[alg], seed=5, **kw)
    res = []
    for eov in (-1, 1, 0):
        dv = d.Device(0)
        dv.set_option("pipeline", 1)
        dv.set_option("eig_overlap", eov)
        res.append(d.solve(a, cfg, device=dv))
        dv.close()
    check_solve(res[0], ref, 120)
    for r in res[1:]:
        assert r.trace.iterations == res[0].trace.iterations
        for name in ("u", "s", "v"):
            assert_bitwise(getattr(res[0].svd, name), getattr(r.svd, name))


def _rmat_host(scale, draws, seed):
    dv = d.Device(0)
    m = d.rmat(scale, draws, seed=seed, device=dv)
    a = m.download()
    m.close()
    dv.close()
    return a


@pytest.mark.parametrize("alg,kw", [("shifted", dict(p=4)), ("dash", dict(tol=1e-2))])
def test_compact_cols_matches_oracle_and_the_full_solve(oracle, alg, kw):
    """An R-MAT graph with ~half of its columns empty: the solve runs on the
    non-empty columns only (compact_cols = 1, default) and scatters V back.
    Against the oracle (which computes every zero row) and the uncompacted
    device solve: the same N_p, sigma and subspaces to rounding, and V exactly
    zero on the empty columns."""
    a = _rmat_host(13, 60000, 3)
    empty = np.bincount(a.col_indices, minlength=a.cols) == 0
    assert 0.2 * a.cols < empty.sum() < 0.8 * a.cols
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    ref = oracle.solve(ca, 40, 20, alg=alg, seed=4, **kw)
    cfg = d.SolverConfig(k=40, s=20, alg=d.Algorithm[alg], seed=4, **kw)
    out = []
    for cc in (1, 0):
        dv = d.Device(0)
        dv.set_option("compact_cols", cc)
        out.append(d.solve(a, cfg, device=dv))
        dv.close()
    res, full = out
    check_solve(res, ref, 40)
    assert np.all(res.svd.v[empty] == 0.0)
    assert res.trace.iterations == full.trace.iterations
    np.testing.assert_allclose(res.svd.s, full.svd.s, rtol=1e-12)
    assert sin_theta(full.svd.u, res.svd.u) <= 1e-10
    assert sin_theta(full.svd.v, res.svd.v) <= 1e-10


def test_compact_cols_wide_orientation(oracle):
    """A wide matrix (rows < cols) is solved on its transpose, whose empty
    columns are A's empty rows: U is the scattered factor there."""
    a = _rmat_host(13, 60000, 8)
    r = 3000  # the first rows: a 3000 x 8192 wide matrix with empty rows
    w = d.SparseMatrix(r, a.cols, a.offsets[:r + 1].copy(), a.col_indices[:a.offsets[r]].copy(),
                       a.values[:a.offsets[r]].copy())
    empty_rows = np.diff(w.offsets) == 0
    assert empty_rows.sum() > 0.05 * r
    ref = oracle.solve(Csr(w.rows, w.cols, w.offsets, w.col_indices, w.values), 30, 15, p=3, alg="shifted",
                       seed=1)
    dv = d.Device(0)
    res = d.solve(w, d.SolverConfig(k=30, s=15, p=3, alg=d.Algorithm.shifted, seed=1), device=dv)
    dv.close()
    check_solve(res, ref, 30)
    assert np.all(res.svd.u[empty_rows] == 0.0)


def test_compact_cols_device_outputs_are_the_host_outputs():
    """The device-resident entry point (dsvd_solve_csr_device, bench.py's `value`
    path) with column compaction: V is scattered into the caller's device buffer
    with zero rows, bitwise the host-output solve. (Device buffers through
    cuda-python: importing torch after NCCL was dlopen'd by an earlier test
    would clash with its bundled NCCL.)"""
    rt = pytest.importorskip("cuda.bindings.runtime")
    a = _rmat_host(12, 30000, 11)
    k = 20
    cfg = d.SolverConfig(k=k, s=10, p=3, alg=d.Algorithm.shifted, seed=2)
    dv = d.Device(0)
    host = d.solve(a, cfg, device=dv)
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
    bufs = []

    def up(x):
        err, p = rt.cudaMalloc(max(x.nbytes, 8))
        assert err == rt.cudaError_t.cudaSuccess
        bufs.append(p)
        if x.nbytes:
            assert rt.cudaMemcpy(p, x.ctypes.data, x.nbytes, H2D)[0] == rt.cudaError_t.cudaSuccess
        return p

    off = up(np.ascontiguousarray(a.offsets, dtype=np.int64))
    idx = up(np.ascontiguousarray(a.col_indices, dtype=np.int64))
    val = up(np.ascontiguousarray(a.values))
    u_h = np.full((a.rows, k), np.nan, order="F")
    v_h = np.full((a.cols, k), np.nan, order="F")
    s_h = np.empty(k)
    du, dvv, ds = up(u_h), up(v_h), up(s_h)
    res = d.api.solve_device_csr(a.rows, a.cols, a.nnz, off, idx, val, cfg, du, ds, dvv, device=dv)
    for hb, db in ((u_h, du), (v_h, dvv), (s_h, ds)):
        assert rt.cudaMemcpy(hb.ctypes.data, db, hb.nbytes, D2H)[0] == rt.cudaError_t.cudaSuccess
    for p in bufs:
        rt.cudaFree(p)
    dv.close()
    assert res.trace.iterations == host.trace.iterations
    assert_bitwise(s_h, host.svd.s)
    assert_bitwise(u_h, host.svd.u)
    assert_bitwise(v_h, host.svd.v)
    assert (np.bincount(a.col_indices, minlength=a.cols) == 0).sum() > 0.05 * a.cols


@pytest.mark.parametrize("slab,k,s_", [(64, 200, 100), (32, 100, 50)])
@pytest.mark.parametrize("mode", [1, 2])
def test_short_rows_whole_row_kernel_is_bitwise_the_per_slab_launch(slab, k, s_, mode):
    """spmm_short_rows (default 1): the column-slab SpMM's rows of at most 8 (mode 2: 32)
    nonzeros run as whole rows, one 16-lane group gathering every slab of a nonzero at
    once, instead of one (row, slab) item each. Same FMA chains: bitwise the per-slab
    launch (mode 0), for 64- and 32-column slabs, on both passes of a shifted solve."""
    a = d.powerlaw(9000, 4000, 2.0, 1.2, 1.1, 13)  # many rows of 1..8 and 9..32 nonzeros
    deg = np.diff(a.offsets)
    assert ((deg > 0) & (deg <= 8)).sum() > 1000 and ((deg > 8) & (deg <= 32)).sum() > 500
    cfg = d.SolverConfig(k=k, s=s_, p=3, alg=d.Algorithm.shifted, seed=2)
    out = []
    for m in (0, mode):
        dv = d.Device(0)
        dv.set_option("spmm_slab", slab)
        dv.set_option("spmm_short_rows", m)
        out.append(d.solve(a, cfg, device=dv))
        dv.close()
    for name in ("u", "s", "v"):
        assert_bitwise(getattr(out[0].svd, name), getattr(out[1].svd, name))
    d.Device(0).set_option("spmm_short_rows", 1)  # process-wide knob: back to the default


@pytest.mark.parametrize("slab", [64, 32])
def test_compact_rows_in_the_finalize(oracle, slab):
    """Column-slab path (forced here at l = 60): the finalize forms B = A Q on the
    non-empty rows of A only (a view of A with its length order renumbered), runs
    the Gram and U = B V' diag(1/s) on them and scatters U back. Against the oracle
    and the uncompacted solve; U exactly zero on A's empty rows."""
    a = _rmat_host(13, 60000, 21)
    empty_rows = np.diff(a.offsets) == 0
    assert 0.2 * a.rows < empty_rows.sum() < 0.8 * a.rows
    assert np.diff(a.offsets).max() > 512  # hub rows: the split-row chunks run on the compacted view
    ca = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    ref = oracle.solve(ca, 40, 20, p=3, alg="shifted", seed=3)
    cfg = d.SolverConfig(k=40, s=20, p=3, alg=d.Algorithm.shifted, seed=3)
    out = []
    for cc in (1, 0):
        dv = d.Device(0)
        dv.set_option("spmm_slab", slab)
        dv.set_option("compact_cols", cc)
        out.append(d.solve(a, cfg, device=dv))
        dv.close()
    res, full = out
    check_solve(res, ref, 40)
    assert np.all(res.svd.u[empty_rows] == 0.0)
    np.testing.assert_allclose(res.svd.s, full.svd.s, rtol=1e-12)
    assert sin_theta(full.svd.u, res.svd.u) <= 1e-10
    assert sin_theta(full.svd.v, res.svd.v) <= 1e-10
