"""GPU: the reference's property tests of the solver (proj/tests/test_rsvd.cpp:177-501),
restated on the device path with numpy's dense SVD as the truth (the reference uses its
own oracle_svd, a one-sided Jacobi SVD; either is exact to ~1e-15 at these sizes).
"""
import numpy as np
import pytest

import paper_2404_09276_b200 as d

pytestmark = pytest.mark.gpu


def dense(a):
    m = np.zeros((a.rows, a.cols))
    rows = np.repeat(np.arange(a.rows), np.diff(a.offsets))
    m[rows, a.col_indices] = a.values
    return m


def cfg(alg, k, s, p, **kw):
    return d.SolverConfig(k=k, s=s, p=p, alg=d.Algorithm[alg], **kw)


def orthonormality_error(x):
    return float(np.abs(x.T @ x - np.eye(x.shape[1])).max())


def test_singular_values_sit_at_or_below_the_truth(dev):
    # test_rsvd.cpp:177-201
    a = d.sparse_random(100, 60, 6, 515, True)
    truth = np.linalg.svd(dense(a), compute_uv=False)
    k = 10
    results = [
        d.basic_rsvd(a, cfg("basic", k, 5, 2), device=dev),
        d.basic_rsvd(a, cfg("basic", k, 5, 2, orth=d.Orthonormalizer.qr), device=dev),
        d.shifted_rsvd(a, cfg("shifted", k, 5, 2), device=dev).svd,
        d.shifted_rsvd(a, cfg("fixed_shift", k, 5, 2), device=dev).svd,
        d.dash_svd(a, cfg("dash", k, 5, -1), device=dev).svd,
    ]
    for f in results:
        assert f.s.size == k
        assert np.all(f.s <= truth[:k] * (1.0 + 1e-10))
        assert np.all(f.s >= 0.0)
        assert np.all(np.diff(f.s) <= 1e-12)


def test_shift_trace_on_an_exactly_captured_invariant_subspace(dev):
    # test_rsvd.cpp:203-227: rank(A) = 4 = l, the first basis spans the row space
    diag = [4.0, 3.0, 2.0, 1.0]
    a = d.SparseMatrix(6, 6, [0, 1, 2, 3, 4, 4, 4], [0, 1, 2, 3], diag)
    r = d.shifted_rsvd(a, cfg("shifted", 2, 2, 3), device=dev)
    assert r.trace.iterations == 3 and r.trace.stop_reason == d.StopReason.fixed_p
    al = r.trace.alphas
    assert len(al) == 3 and al[0] == 0.0 and al[1] > 0.0
    assert all(al[c] >= al[c - 1] for c in range(1, 3))
    first = r.trace.s_hat_history[0]
    assert len(first) == 4
    assert first[0] == pytest.approx(16.0, rel=1e-12)
    assert first[3] == pytest.approx(1.0, rel=1e-12)
    assert al[1] == pytest.approx(0.5, rel=1e-12)
    assert abs(r.svd.s[0] - 4.0) <= 1e-10 and abs(r.svd.s[1] - 3.0) <= 1e-10


def test_frozen_shift_keeps_the_shift_from_iteration_two(dev):
    # test_rsvd.cpp:229-241
    a = d.sparse_random(50, 35, 6, 21, True)
    r = d.shifted_rsvd(a, cfg("fixed_shift", 5, 3, 4), device=dev)
    al = r.trace.alphas
    assert len(al) == 4 and al[0] == 0.0 and al[1] > 0.0 and al[2] == al[1] and al[3] == al[1]
    dyn = d.shifted_rsvd(a, cfg("shifted", 5, 3, 4), device=dev)
    assert dyn.trace.alphas[1] == al[1] and dyn.trace.alphas[3] >= dyn.trace.alphas[1]


def test_shifts_never_exceed_half_the_lth_squared_singular_value(dev):
    # test_rsvd.cpp:243-249
    a = d.sparse_random(80, 50, 8, 99, True)
    truth = np.linalg.svd(dense(a), compute_uv=False)
    r = d.shifted_rsvd(a, cfg("shifted", 8, 4, 6), device=dev)
    sigma_l = truth[11]  # l = 12
    assert all(alpha <= sigma_l * sigma_l / 2.0 + 1e-9 for alpha in r.trace.alphas)


def test_surrogate_spectrum_is_sandwiched(dev):
    # test_rsvd.cpp:460-478: projected spectrum <= s_hat + alpha <= truth, every iteration
    a = d.sparse_random(40, 25, 6, 77, True)
    ad = dense(a)
    truth = np.linalg.svd(ad, compute_uv=False)
    k, s = 5, 5
    l = k + s
    calls = []

    def obs(st):
        calls.append(st.iteration)
        projected = np.linalg.svd(ad @ st.q_before, compute_uv=False)
        unshifted = np.asarray(st.s_hat) + st.alpha
        assert np.all(projected[:l] ** 2 <= unshifted[:l] + 1e-8)
        assert np.all(unshifted[:l] <= truth[:l] ** 2 + 1e-8)

    d.shifted_rsvd(a, cfg("shifted", k, s, 3), observer=obs, device=dev)
    assert len(calls) == 3


def test_returned_factors_are_well_formed_for_every_algorithm(dev):
    # test_rsvd.cpp:480-501
    a = d.sparse_random(120, 70, 8, 13, True)
    k = 9

    def check(f, row_basis_family):
        assert f.s.size == k
        assert f.u.shape == (120, k) and f.v.shape == (70, k)
        assert orthonormality_error(f.u) <= 1e-8 and orthonormality_error(f.v) <= 1e-8
        assert np.all(f.s > 0.0) and np.all(np.diff(f.s) <= 1e-12)
        if row_basis_family:
            assert d.max_triplet_residual(a, f, device=dev) <= 1e-10 * f.s[0]

    check(d.basic_rsvd(a, cfg("basic", k, 4, 3), device=dev), False)
    check(d.shifted_rsvd(a, cfg("shifted", k, 4, 3), device=dev).svd, True)
    check(d.dash_svd(a, cfg("dash", k, 4, -1), device=dev).svd, True)


def test_dash_stops_at_the_first_passage_of_the_rule(dev):
    # acceptance.cpp:213-261 (criterion 3): the first iteration whose PVE ratio is
    # <= tol is the stop, none before it, and the result's eps_pve is small
    a = d.sparse_random(2000, 800, 12, 5, True)
    k, s, tol = 20, 10, 1e-2
    r = d.dash_svd(a, d.SolverConfig(k=k, s=s, tol=tol), device=dev)
    assert r.trace.stop_reason == d.StopReason.tol_met
    sh, al = np.array(r.trace.s_hat_history), np.array(r.trace.alphas)
    n = r.trace.iterations
    for j in range(1, n):
        ratio = np.max(np.abs(sh[j - 1][:k] + al[j] - sh[j][:k] - al[j]) / (sh[j][k] + al[j]))
        assert (ratio <= tol) == (j == n - 1), (j, ratio)
    truth = np.linalg.svd(dense(a), compute_uv=False)
    assert d.eps_pve(a, r.svd.u, truth, device=dev) <= 5e-2


def test_acceptance_criterion4_underestimation_sweep(dev):
    # acceptance.cpp:270-309: 50 matrices x 5 algorithm variants, sigma_hat <= sigma (1 + 1e-10)
    worst = 0.0
    for g in range(1, 51):
        a = d.sparse_random(200, 100, 10, g, True)
        truth = np.linalg.svd(dense(a), compute_uv=False)
        for variant in range(5):
            alg = ["basic", "basic", "shifted", "fixed_shift", "dash"][variant]
            c = d.SolverConfig(k=10, s=5, p=-1 if alg == "dash" else 3, tol=1e-2, seed=100 + g,
                               alg=d.Algorithm[alg],
                               orth=d.Orthonormalizer.qr if variant == 1 else d.Orthonormalizer.eigsvd)
            s = d.solve(a, c, device=dev).svd.s
            worst = max(worst, float(np.max(s / truth[:10] - 1.0)))
    assert worst <= 1e-10, worst


def test_acceptance_criterion7_eig_svd_against_an_independent_svd(dev):
    # acceptance.cpp:423-433: 100 Gaussian 2n x n matrices, sigma relative error <= 1e-8
    worst = 0.0
    for i in range(100):
        n = 10 + (i % 45)
        x = d.gaussian_matrix(2 * n, n, 1000 + i, device=dev)
        fast = d.eig_svd(x, device=dev).s
        slow = np.linalg.svd(x, compute_uv=False)
        worst = max(worst, float(np.max(np.abs(fast - slow) / slow)))
    assert worst <= 1e-8, worst


@pytest.fixture(scope="module")
def planted(oracle):
    # dense2_matrix(1000, 0) (synthetic.cpp:51-70): U diag(1/sqrt(i+1)) V^T with U, V the
    # Householder Q of seeded Gaussian matrices (the oracle's restatements of
    # gaussian_matrix and qr_orth; the product is formed in numpy)
    n = 1000
    sig = 1.0 / np.sqrt(np.arange(1, n + 1, dtype=np.float64))
    u = oracle.qr_orth(oracle.gaussian_matrix(n, n, oracle.splitmix64_at(0, 0)))
    v = oracle.qr_orth(oracle.gaussian_matrix(n, n, oracle.splitmix64_at(0, 1)))
    m = (u * sig) @ v.T
    off = np.arange(0, n * n + 1, n, dtype=np.int64)
    idx = np.tile(np.arange(n, dtype=np.int64), n)
    return d.SparseMatrix(n, n, off, idx, np.ascontiguousarray(m).ravel()), sig


def _eps(m, sig, alg, p, seed, dev):
    r = m.solve(d.SolverConfig(k=100, s=50, p=p, seed=seed, alg=d.Algorithm[alg]))
    return d.eps_pve(m, r.svd.u, sig, device=dev)


def test_acceptance_criteria1_2_shifted_beats_basic_and_frozen(planted, dev):
    # acceptance.cpp:96-189: on the planted 1000 x 1000 spectrum (k = 100, s = 50),
    # criterion 1: shifted eps_pve < basic eps_pve in >= 90% of (seed, p) pairs,
    #   p in {4, 8, 12, 16, 20}, 10 seeds, and the median ratio at p = 20 is <= 0.1;
    # criterion 2: shifted <= frozen shift at p = 8 and 16 on >= 8 of 10 seeds
    a, sig = planted
    m = d.DeviceMatrix(a, dev)
    wins = pairs = c2 = 0
    ratios = []
    for seed in range(1, 11):
        e_s, e_b, e_f = {}, {}, {}
        for p in (4, 8, 12, 16, 20):
            e_s[p] = _eps(m, sig, "shifted", p, seed, dev)
            e_b[p] = _eps(m, sig, "basic", p, seed, dev)
            pairs += 1
            wins += e_s[p] < e_b[p]
        for p in (8, 16):
            e_f[p] = _eps(m, sig, "fixed_shift", p, seed, dev)
        ratios.append(e_s[20] / e_b[20])
        c2 += all(e_s[p] <= e_f[p] for p in (8, 16))
    m.close()
    assert wins >= int(0.9 * pairs + 0.5), (wins, pairs)
    assert float(np.median(ratios)) <= 0.1, ratios
    assert c2 >= 8, c2
