"""GPU: the device half of the input path, through the C ABI.

- COO -> canonical CSR assembly on the device (ingest.cu) against the reference's
  load_matrix_market outcomes (tests/golden/input_golden.json) and, when oracle/_ref is
  present, the reference itself on larger random files: BITWISE;
- device CSR validation (dsvd_csr_validate) against SparseMatrix::validate: same first
  violation, same error type and message;
- DSH1 cache loaded straight into HBM (validate on the device) against the reference's
  load_cache, including its UnsupportedFormat / Error cases;
- full-size property: the C2 matrix, scattered into shuffled triplets, assembles back to
  itself bit for bit (assembly is idempotent on canonical input);
- a solve on a matrix loaded from a file equals the solve on the same matrix uploaded.
"""
import zlib

import numpy as np
import pytest

import paper_2404_09276_b200 as d
from input_cases import MTX_CASES, assemble_np, corrupt_csr
from paper_2404_09276_b200 import errors as E
from test_inputs import gold, outcome, write_case  # noqa: F401  (fixture re-export)

pytestmark = pytest.mark.gpu


def to_dev(a):
    return d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, a.values)


def same_csr(a, b):
    assert (a.rows, a.cols) == (b.rows, b.cols)
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(np.asarray(a.values).view(np.uint64), np.asarray(b.values).view(np.uint64))


@pytest.mark.parametrize("name", sorted(MTX_CASES))
def test_load_matrix_market_matches_reference(tmp_path, gold, dev, name):  # noqa: F811
    path = write_case(tmp_path, name)
    assert outcome(lambda: d.load_matrix_market(path, device=dev)) == gold["mtx"][name]


def test_device_matrix_from_matrix_market(tmp_path, dev):
    path = write_case(tmp_path, "symmetric")
    m = d.DeviceMatrix.from_matrix_market(path, device=dev)
    host = d.load_matrix_market(path, device=dev)
    same_csr(m.download(), host)
    t = m.transpose()
    assert t.rows == host.cols and t.nnz == host.nnz
    m.close()


def random_mtx(rng, rows, cols, n, sym="general", field="real", dup_frac=0.2):
    r = rng.integers(1, rows + 1, n)
    c = rng.integers(1, cols + 1, n)
    if sym != "general":
        keep = r >= c if sym == "symmetric" else r > c
        r, c = r[keep], c[keep]
    ndup = int(dup_frac * r.size)
    if ndup:
        pick = rng.integers(0, r.size, ndup)
        r, c = np.concatenate([r, r[pick]]), np.concatenate([c, c[pick]])
    # integer-valued doubles: duplicate sums are exact in any order, so the
    # reference's unstable sort and the device's stable one agree bit for bit
    v = rng.integers(-8, 9, r.size).astype(np.float64) * 0.5
    lines = [f"%%MatrixMarket matrix coordinate {field} {sym}", f"{rows} {cols} {r.size}"]
    if field == "pattern":
        lines += [f"{i} {j}" for i, j in zip(r, c)]
    else:
        lines += [f"{i} {j} {x:g}" for i, j, x in zip(r, c, v)]
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("sym,field", [("general", "real"), ("symmetric", "real"),
                                       ("skew-symmetric", "real"), ("general", "pattern"),
                                       ("symmetric", "integer")])
def test_random_files_match_reference(tmp_path, dev, reference, sym, field):
    rng = np.random.default_rng(zlib.crc32(f"{sym}/{field}".encode()))
    rows = cols = 700 if sym != "general" else 0
    rows, cols = (rows, cols) if rows else (900, 600)
    text = random_mtx(rng, rows, cols, 20000, sym, field)
    path = tmp_path / "r.mtx"
    path.write_text(text)
    same_csr(d.load_matrix_market(str(path), device=dev), reference.load_matrix_market(str(path)))


def test_assemble_against_numpy_restatement(dev):
    rng = np.random.default_rng(11)
    rows, cols, n = 3000, 2000, 200000
    r = rng.integers(0, rows, n)
    c = rng.integers(0, cols, n)
    v = rng.integers(-3, 4, n).astype(np.float64)  # many exact cancellations
    got = d.assemble(rows, cols, r, c, v, device=dev)
    same_csr(got, assemble_np(rows, cols, r, c, v))
    assert np.all(got.values != 0.0)


def test_assemble_duplicates_sum_in_input_order(dev):
    # non-associative sums: the device adds duplicates in input order (stable sort)
    r = np.array([1, 0, 1, 1, 1])
    c = np.array([2, 0, 2, 2, 2])
    v = np.array([1e16, 1.0, 1.0, -1e16, 1.0])
    got = d.assemble(2, 3, r, c, v, device=dev)
    assert got.offsets.tolist() == [0, 1, 2]
    assert got.values.tolist() == [1.0, ((1e16 + 1.0) - 1e16) + 1.0]


def test_assemble_edge_cases(dev):
    e = d.assemble(4, 5, [], [], [], device=dev)
    assert e.offsets.tolist() == [0] * 5 and e.nnz == 0
    z = d.assemble(0, 0, [], [], [], device=dev)
    assert z.offsets.tolist() == [0]
    cancel = d.assemble(2, 2, [0, 0], [1, 1], [2.0, -2.0], device=dev)
    assert cancel.nnz == 0 and cancel.offsets.tolist() == [0, 0, 0]
    with pytest.raises(E.ShapeError):
        d.assemble(2, 2, [0, 2], [0, 0], [1.0, 1.0], device=dev)
    with pytest.raises(E.ShapeError):
        d.assemble(2, 2, [0], [-1], [1.0], device=dev)


def test_assemble_c2_shuffled_is_identity(dev):
    # full-size property: canonical CSR -> shuffled triplets -> assemble == the CSR
    a = d.powerlaw(200000, 100000, 4.0, 1.0, 1.1, 1)
    rows_of = np.repeat(np.arange(a.rows, dtype=np.int64), np.diff(a.offsets))
    perm = np.random.default_rng(5).permutation(a.nnz)
    got = d.assemble(a.rows, a.cols, rows_of[perm], a.col_indices[perm], a.values[perm], device=dev)
    same_csr(got, a)


def test_device_validate_matches_reference(gold, dev):  # noqa: F811
    for seed, want in enumerate(gold["validate"]):
        a = to_dev(corrupt_csr(seed))
        assert outcome(lambda: a.validate_on_device(dev)) == want, seed


def test_device_validate_live_reference(dev, reference):
    rng = np.random.default_rng(99)
    for seed in range(1000, 1200):
        a = corrupt_csr(seed)
        assert outcome(lambda: to_dev(a).validate_on_device(dev)) == outcome(lambda: reference.validate(a)), seed
    # a large valid matrix and a late violation
    big = d.sparse_random(20000, 7000, 30, 3, True)
    big.validate_on_device(dev)
    bad = d.SparseMatrix(big.rows, big.cols, big.offsets, big.col_indices.copy(), big.values.copy())
    p = int(rng.integers(big.nnz // 2, big.nnz))
    bad.values[p] = 0.0
    row = int(np.searchsorted(big.offsets, p, "right") - 1)
    with pytest.raises(E.NumericalError, match=f"explicit zero stored in row {row}$"):
        bad.validate_on_device(dev)


def test_cache_round_trip_and_errors(tmp_path, dev, reference):
    a = reference.sparse_random(400, 230, 5, 77)
    path = str(tmp_path / "a.dsh")
    d.save_cache(path, to_dev(a))
    same_csr(d.load_cache(path, device=dev), reference.load_cache(path))
    m = d.DeviceMatrix.load_cache(path, device=dev)
    same_csr(m.download(), a)
    m.close()

    junk = tmp_path / "junk.dsh"
    junk.write_text("not a cache")
    short = tmp_path / "short.dsh"
    raw = open(path, "rb").read()
    short.write_bytes(raw[:len(raw) // 2])
    tiny = tmp_path / "tiny.dsh"
    tiny.write_bytes(b"DS")
    header = tmp_path / "header.dsh"
    header.write_bytes(raw[:20])
    for p in (junk, short, tiny, header, tmp_path / "missing.dsh"):
        assert outcome(lambda: d.load_cache(str(p), device=dev)) == outcome(lambda: reference.load_cache(str(p)))
    with pytest.raises(E.UnsupportedFormat, match="not a DSH1"):
        d.load_cache(str(junk), device=dev)
    with pytest.raises(E.UnsupportedFormat, match="truncated"):
        d.load_cache(str(short), device=dev)


def test_cache_with_invalid_contents(tmp_path, dev, reference):
    for seed in range(0, 60, 3):
        a = corrupt_csr(seed)
        path = str(tmp_path / f"c{seed}.dsh")
        reference_ok = True
        try:
            reference.save_cache(path, a)
        except E.Error:
            reference_ok = False
        if not reference_ok:
            continue
        assert outcome(lambda: d.load_cache(path, device=dev)) == outcome(lambda: reference.load_cache(path)), seed


def test_solve_from_file_equals_upload(tmp_path, dev):
    a = d.sparse_random(3000, 1200, 20, 4, True)
    path = str(tmp_path / "s.dsh")
    d.save_cache(path, a)
    cfg = d.SolverConfig(k=20, p=6, seed=2)
    r1 = d.DeviceMatrix.load_cache(path, device=dev).solve(cfg)
    r2 = d.DeviceMatrix(a, device=dev).solve(cfg)
    assert np.array_equal(r1.svd.s.view(np.uint64), r2.svd.s.view(np.uint64))
    assert np.array_equal(r1.svd.u.view(np.uint64), r2.svd.u.view(np.uint64))
    mtx = str(tmp_path / "s.mtx")
    d.write_matrix_market(mtx, a)
    r3 = d.DeviceMatrix.from_matrix_market(mtx, device=dev).solve(cfg)
    assert np.array_equal(r3.svd.v.view(np.uint64), r2.svd.v.view(np.uint64))


# ---- R-MAT generator (BASELINE.json configs 4/5) ----------------------------------

@pytest.mark.parametrize("scale,draws,uniform,seed", [(1, 5, False, 0), (6, 300, True, 3), (10, 20000, False, 1),
                                                      (13, 150000, True, 7), (17, 2000000, True, 2)])
def test_rmat_matches_numpy_restatement(dev, scale, draws, uniform, seed):
    from input_cases import rmat_np
    m = d.rmat(scale, draws, uniform_values=uniform, seed=seed, device=dev)
    got = m.download()
    same_csr(got, rmat_np(scale, draws, uniform=uniform, seed=seed))
    got.validate()
    assert np.all(got.values > 0.0) and np.all(got.values <= 1.0)
    m.close()


def test_rmat_skewed_quadrants(dev):
    from input_cases import rmat_np
    for a, b, c in ((1.0, 0.0, 0.0), (0.25, 0.25, 0.25), (0.0, 0.0, 1.0), (0.45, 0.15, 0.15)):
        got = d.rmat(9, 5000, a, b, c, seed=4, device=dev).download()
        same_csr(got, rmat_np(9, 5000, a, b, c, seed=4))
    with pytest.raises(E.ConfigError):
        d.rmat(5, 10, 0.6, 0.3, 0.3, device=dev)
    with pytest.raises(E.ShapeError):
        d.rmat(31, 10, device=dev)
