"""GPU: the row-sharded engine (engine.cu solve_tall with a communicator)
executed natively at world size 2 and 3 on ONE B200.

Each rank is a device context on its own host thread, attached to an
in-process loopback group (comm.cu): its collectives synchronise the rank's
stream, meet the other ranks at a host barrier and sum their device buffers in
fixed rank order, so no kernel ever waits on another rank's kernel. Every
sharded branch of the engine runs for real: Omega_g with the global index
formula at row_offset > 0 (random.cpp:29-36), the reduced n x l partials and
the shift applied once after the sum (solver.cpp:93-95), the v2 slab Gram +
l x l all-reduce + slab rescale + all-gather, the all-reduced finalize Gram with
the global rank floor (decompositions.cpp:52-62) and the U row shards.

Bars (the same as tests/test_dist_gloo.py, against the single-process oracle
solve): singular values relative 1e-10, largest principal angle of U (the
stacked shards) and V <= 1e-8, identical iteration count and stop reason;
Omega_g bitwise.
"""
import threading

import numpy as np
import pytest

import paper_2404_09276_b200 as d
from oracle_lib import Csr
from paper_2404_09276_b200.sharding import shard_bounds, shard_csr

pytestmark = pytest.mark.gpu


def to_dev(a: Csr) -> d.SparseMatrix:
    return d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, a.values)


def sin_theta(u_ref, u):
    q1, _ = np.linalg.qr(u_ref)
    q2, _ = np.linalg.qr(u)
    r = q2 - q1 @ (q1.T @ q2)
    return float(np.linalg.norm(r, 2))


def run_sharded(a: d.SparseMatrix, cfg: d.SolverConfig, bounds, options=None):
    """Solve `a` row-sharded at `bounds` (r_0 = 0 <= ... <= r_G = rows), one host
    thread and context per rank on device 0. Returns the per-rank results."""
    world = len(bounds) - 1
    group = d.LoopbackGroup(world)
    out = [None] * world
    errors = []

    def rank_main(r):
        try:
            dv = d.Device(0, profiling=True)
            for name, value in (options or {}).items():
                dv.set_option(name, value)
            dv.attach_loopback(group, r)
            r0, r1 = bounds[r], bounds[r + 1]
            dv.set_shard(r0, a.rows)
            out[r] = d.solve(shard_csr(a, r0, r1), cfg, device=dv)
        except Exception as exc:  # surfaced below
            errors.append((r, exc))

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    group.close()
    assert not errors, errors
    return out


def check_against(res, ref, k):
    u = np.vstack([r.svd.u for r in res])
    for r in res:  # every rank holds the same replicated factors
        assert r.trace.iterations == ref["iterations"]
        assert r.trace.stop_reason.name == ref["stop_reason"]
        np.testing.assert_allclose(r.svd.s, ref["s"], rtol=1e-10)
        assert sin_theta(ref["v"], r.svd.v) <= 1e-8
        np.testing.assert_array_equal(r.svd.s, res[0].svd.s)  # identical decisions and sums
    assert sin_theta(ref["u"], u) <= 1e-8
    np.testing.assert_allclose(res[0].trace.alphas, ref["alphas"], rtol=1e-9, atol=1e-300)


@pytest.fixture(scope="module")
def c1(oracle):
    return oracle.sparse_random(10000, 5000, 25, 0, True)


@pytest.fixture(scope="module")
def plaw():
    # power-law rows (lognormal degrees) and Zipf columns: hub columns make the
    # transpose's split-chunk path run on every rank
    return d.powerlaw(30000, 12000, 3.0, 1.0, 1.1, 7)


def test_shard_sketch_is_the_global_sketch_bitwise(oracle):
    """Omega_g = rows [r0, r1) of the global sketch: bitwise the device's full
    gaussian_matrix rows, and the reference's draws to <= 2 ulp (the device's
    log/cos are correctly rounded, glibc's are not always; DESIGN 2)."""
    m, l = 997, 37
    dv = d.Device(0)
    full = d.gaussian_matrix(m, l, 2026, device=dv)
    ref = oracle.gaussian_matrix(m, l, 2026)
    np.testing.assert_allclose(full, ref, rtol=5e-16, atol=0)
    for r0, r1 in ((0, 400), (400, 997), (123, 124), (996, 997)):
        blk = d.gaussian_rows(r1 - r0, l, 2026, m, r0, device=dv)
        assert np.array_equal(blk.view(np.uint64), np.asfortranarray(full[r0:r1]).view(np.uint64))
    dv.close()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("pipeline", [0, 1])
@pytest.mark.parametrize("alg", ["shifted", "dash"])
def test_sharded_c1_matches_oracle(oracle, c1, world, mode, pipeline, alg):
    k, s = 50, 25
    if alg == "shifted":
        cfg = d.SolverConfig(k=k, s=s, p=6, alg=d.Algorithm.shifted, seed=0)
        ref = oracle.solve(c1, k, s, p=6, alg="shifted", seed=0)
    else:
        cfg = d.SolverConfig(k=k, s=s, tol=1e-2, seed=0)
        ref = oracle.solve(c1, k, s, tol=1e-2, alg="dash", seed=0)
    a = to_dev(c1)
    bounds = shard_bounds(a.offsets, world)
    res = run_sharded(a, cfg, bounds, {"mgpu_mode": mode, "pipeline": pipeline})
    check_against(res, ref, k)
    assert all(r.stats["pipelined"] == pipeline for r in res)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("pipeline", [0, 1])
def test_sharded_power_law_matches_oracle(oracle, plaw, mode, pipeline):
    k, s = 40, 20
    cfg = d.SolverConfig(k=k, s=s, tol=1e-2, p_max=30, seed=3)
    ref = oracle.solve(Csr(plaw.rows, plaw.cols, plaw.offsets, plaw.col_indices, plaw.values), k, s,
                       tol=1e-2, p_max=30, alg="dash", seed=3)
    bounds = shard_bounds(plaw.offsets, 2)
    res = run_sharded(plaw, cfg, bounds, {"mgpu_mode": mode, "pipeline": pipeline})
    check_against(res, ref, k)


@pytest.mark.parametrize("mode", [1, 2])
def test_sharded_unbalanced_and_tiny_shards(oracle, c1, mode):
    """Shards far from the nnz balance: a one-row shard and a shard with most rows."""
    k, s = 30, 15
    cfg = d.SolverConfig(k=k, s=s, p=4, alg=d.Algorithm.shifted, seed=5)
    ref = oracle.solve(c1, k, s, p=4, alg="shifted", seed=5)
    res = run_sharded(to_dev(c1), cfg, [0, 1, 9000, 10000], {"mgpu_mode": mode})
    check_against(res, ref, k)


def test_auto_schedule_is_taken_from_the_global_nnz(oracle, c1):
    """with the auto schedule, ranks whose LOCAL nnz fall on opposite
    sides of the bound used to pick different loop schedules (which reduce
    different partials). The bound below splits the shards' local counts but not
    the global one: every rank must take the serial schedule and match the oracle."""
    k, s = 30, 15
    a = to_dev(c1)
    bounds = [0, 8000, 10000]
    nnz_local = [int(a.offsets[bounds[r + 1]] - a.offsets[bounds[r]]) for r in range(2)]
    bound = (max(nnz_local) + min(nnz_local)) // 2
    assert min(nnz_local) <= bound < max(nnz_local) < a.nnz
    cfg = d.SolverConfig(k=k, s=s, p=5, alg=d.Algorithm.shifted, seed=1)
    ref = oracle.solve(c1, k, s, p=5, alg="shifted", seed=1)
    res = run_sharded(a, cfg, bounds, {"pipeline": -1, "pipeline_auto_nnz": bound})
    assert [r.stats["pipelined"] for r in res] == [0, 0]
    check_against(res, ref, k)


def test_sharded_v1_and_v2_agree(c1):
    cfg = d.SolverConfig(k=20, s=10, p=3, alg=d.Algorithm.shifted, seed=9)
    a = to_dev(c1)
    bounds = shard_bounds(a.offsets, 2)
    r1 = run_sharded(a, cfg, bounds, {"mgpu_mode": 1})
    r2 = run_sharded(a, cfg, bounds, {"mgpu_mode": 2})
    np.testing.assert_allclose(r1[0].svd.s, r2[0].svd.s, rtol=1e-12)
    assert sin_theta(r1[0].svd.v, r2[0].svd.v) <= 1e-10


def test_sharded_rerun_is_deterministic(c1):
    cfg = d.SolverConfig(k=20, s=10, tol=1e-2, seed=2)
    a = to_dev(c1)
    bounds = shard_bounds(a.offsets, 3)
    x = run_sharded(a, cfg, bounds)
    y = run_sharded(a, cfg, bounds)
    for rx, ry in zip(x, y):
        assert np.array_equal(rx.svd.s.view(np.uint64), ry.svd.s.view(np.uint64))
        assert np.array_equal(rx.svd.u.view(np.uint64), ry.svd.u.view(np.uint64))


def assert_same_bits(x, y):
    for rx, ry in zip(x, y):
        assert rx.trace.iterations == ry.trace.iterations
        for name in ("u", "s", "v"):
            a, b = getattr(rx.svd, name), getattr(ry.svd, name)
            assert np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("pipeline", [0, 1])
def test_exchange_overlap_is_bitwise_the_whole_pass_exchange(plaw, mode, pipeline):
    """mgpu_overlap = 1 (default): the A^T pass runs in G row panels and each
    panel's partial is reduced on the communication stream while the next panel
    computes (v2: ncclReduce to the panel's owner; v1: a per-panel all-reduce).
    The panels' rows (split hub columns included) are computed exactly as in the
    whole pass, so the factors are bitwise those of the whole-pass exchange."""
    cfg = d.SolverConfig(k=24, s=12, tol=1e-2, p_max=20, seed=4)
    bounds = shard_bounds(plaw.offsets, 3)
    x = run_sharded(plaw, cfg, bounds, {"mgpu_mode": mode, "pipeline": pipeline, "mgpu_overlap": 0})
    y = run_sharded(plaw, cfg, bounds, {"mgpu_mode": mode, "pipeline": pipeline, "mgpu_overlap": 1})
    assert_same_bits(x, y)


def test_exchange_overlap_wide_sketch_matches_oracle(oracle, plaw):
    """l = 200 (> 192: the column-slab SpMM with slab-major Y) with the panelled
    exchange: against the oracle and bitwise the whole-pass exchange."""
    k, s = 120, 80
    cfg = d.SolverConfig(k=k, s=s, p=3, alg=d.Algorithm.shifted, seed=6)
    ref = oracle.solve(Csr(plaw.rows, plaw.cols, plaw.offsets, plaw.col_indices, plaw.values), k, s, p=3,
                       alg="shifted", seed=6)
    bounds = shard_bounds(plaw.offsets, 2)
    y = run_sharded(plaw, cfg, bounds, {"mgpu_overlap": 1})
    check_against(y, ref, k)
    x = run_sharded(plaw, cfg, bounds, {"mgpu_overlap": 0})
    assert_same_bits(x, y)


@pytest.mark.parametrize("pipeline", [0, 1])
@pytest.mark.parametrize("alg", ["dash", "shifted"])
def test_fused_exchange_is_bitwise_the_reduce_scatter(plaw, pipeline, alg):
    """mgpu_overlap = 2 (v2): each row panel of the A^T pass is stored straight
    into its owner's landing buffer (slot = the source rank; peer memory — here the
    loopback group's own pointers), then a barrier and the owner's rank-order sum
    of its slots. Bitwise the loopback reduce-scatter (same rank-order sums)."""
    kw = dict(tol=1e-2, p_max=20) if alg == "dash" else dict(p=4)
    cfg = d.SolverConfig(k=24, s=12, alg=d.Algorithm[alg], seed=4, **kw)
    bounds = shard_bounds(plaw.offsets, 3)
    x = run_sharded(plaw, cfg, bounds, {"pipeline": pipeline, "mgpu_overlap": 0})
    y = run_sharded(plaw, cfg, bounds, {"pipeline": pipeline, "mgpu_overlap": 2})
    assert_same_bits(x, y)


def test_fused_exchange_wide_sketch_matches_oracle(oracle, plaw):
    """The fused exchange on the column-slab SpMM (l = 200), 2 ranks, twice in a row
    on the same contexts (the landing buffers are reused), against the oracle."""
    k, s = 120, 80
    cfg = d.SolverConfig(k=k, s=s, p=3, alg=d.Algorithm.shifted, seed=6)
    ref = oracle.solve(Csr(plaw.rows, plaw.cols, plaw.offsets, plaw.col_indices, plaw.values), k, s, p=3,
                       alg="shifted", seed=6)
    bounds = shard_bounds(plaw.offsets, 2)
    y = run_sharded(plaw, cfg, bounds, {"mgpu_overlap": 2})
    check_against(y, ref, k)
    x = run_sharded(plaw, cfg, bounds, {"mgpu_overlap": 0})
    assert_same_bits(x, y)
