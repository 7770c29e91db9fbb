"""CPU: the host half of the input path.

- the Matrix Market text parser (dsvd_mtx_read, csrc/mtx.cpp) against the
  reference's load_matrix_market outcomes committed in tests/golden/input_golden.json
  (tests/golden/make_input_golden.py): same errors, line numbers and messages; for
  accepted files the parsed triplets assembled by the numpy restatement of assemble()
  equal the reference's CSR bit for bit;
- host SparseMatrix.validate against the reference's SparseMatrix::validate outcomes;
- DSH1 cache and Matrix Market writers: byte-identical files to the reference's.
The device halves (assembly, validation, cache load) are in tests/test_gpu_inputs.py.
"""
import json
import os

import numpy as np
import pytest

import paper_2404_09276_b200 as d
from input_cases import MTX_CASES, assemble_np, corrupt_csr
from paper_2404_09276_b200 import errors as E

GOLD = os.path.join(os.path.dirname(__file__), "golden", "input_golden.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def write_case(tmp_path, name):
    path = tmp_path / (name + ".mtx")
    with open(path, "w", newline="") as f:
        f.write(MTX_CASES[name])
    return str(path)


def outcome(fn):
    try:
        a = fn()
    except E.ParseError as e:
        return {"error": "ParseError", "line": e.line, "what": str(e)}
    except E.Error as e:
        return {"error": type(e).__name__, "what": str(e)}
    if a is None:
        return {"ok": True}
    return {"rows": a.rows, "cols": a.cols, "offsets": a.offsets.tolist(),
            "col_indices": a.col_indices.tolist(), "values_hex": [float(x).hex() for x in a.values]}


def test_golden_covers_every_case(gold):
    assert set(gold["mtx"]) == set(MTX_CASES)
    kinds = {v.get("error", "ok") for v in gold["mtx"].values()}
    assert kinds == {"ok", "ParseError", "UnsupportedFormat"}


@pytest.mark.parametrize("name", sorted(MTX_CASES))
def test_mtx_parser_matches_reference(tmp_path, gold, name):
    path = write_case(tmp_path, name)

    def load():
        rows, cols, r, c, v = d.read_matrix_market_triplets(path)
        return assemble_np(rows, cols, r, c, v)

    assert outcome(load) == gold["mtx"][name]


def test_mtx_missing_file_is_error(tmp_path):
    with pytest.raises(E.Error, match="cannot open"):
        d.read_matrix_market_triplets(str(tmp_path / "nope.mtx"))


def test_mtx_symmetric_expansion_order(tmp_path):
    # mirrored entries follow their source entry; zeros filtered only for the stored side
    path = tmp_path / "s.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 4\n3 3 0\n3 2 0\n")
    rows, cols, r, c, v = d.read_matrix_market_triplets(str(path))
    assert (rows, cols) == (3, 3)
    assert r.tolist() == [1, 0, 1] and c.tolist() == [0, 1, 2] and v.tolist() == [4.0, 4.0, 0.0]


def test_host_validate_matches_reference(gold):
    for seed, want in enumerate(gold["validate"]):
        a = corrupt_csr(seed)
        m = d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, a.values)
        assert outcome(m.validate) == want, seed


def test_cache_bytes_match_reference(tmp_path, reference):
    a = reference.sparse_random(40, 23, 5, 77)
    ours, theirs = tmp_path / "ours.dsh", tmp_path / "theirs.dsh"
    d.save_cache(str(ours), d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, a.values))
    reference.save_cache(str(theirs), a)
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_bytes()[:4] == b"DSH1"


def test_cache_layout_without_reference(tmp_path):
    a = d.SparseMatrix(2, 3, [0, 1, 3], [2, 0, 1], [1.5, -2.0, 0.25])
    p = tmp_path / "a.dsh"
    d.save_cache(str(p), a)
    b = p.read_bytes()
    assert b[:4] == b"DSH1"
    dims = np.frombuffer(b[4:28], dtype="<u8")
    assert dims.tolist() == [2, 3, 3]
    body = np.frombuffer(b[28:], dtype="<i8")
    assert body[:3].tolist() == [0, 1, 3] and body[3:6].tolist() == [2, 0, 1]
    assert np.frombuffer(b[28 + 48:], dtype="<f8").tolist() == [1.5, -2.0, 0.25]


def test_write_matrix_market_matches_reference(tmp_path, reference):
    a = reference.sparse_random(30, 17, 4, 5)
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "theirs.mtx"
    d.write_matrix_market(str(ours), d.SparseMatrix(a.rows, a.cols, a.offsets, a.col_indices, a.values))
    reference.write_matrix_market(str(theirs), a)
    assert ours.read_bytes() == theirs.read_bytes()


def test_write_then_parse_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    vals = rng.standard_normal(6) * 10.0 ** rng.integers(-300, 300, 6)
    a = d.SparseMatrix(3, 4, [0, 2, 2, 6], [0, 3, 0, 1, 2, 3], vals)
    p = str(tmp_path / "w.mtx")
    d.write_matrix_market(p, a)
    rows, cols, r, c, v = d.read_matrix_market_triplets(p)
    b = assemble_np(rows, cols, r, c, v)
    assert b.offsets.tolist() == a.offsets.tolist()
    assert b.col_indices.tolist() == a.col_indices.tolist()
    assert b.values.view(np.uint64).tolist() == a.values.view(np.uint64).tolist()


# ---- dense factor files and reference spectra (CLI inputs) -----------------------------

DENSE_CASES = {
    "ok_one_per_line": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "ok_many_per_line": "%%MatrixMarket matrix array real general\n% c\n2 3\n1 2 3\n\n4 5 6\n",
    "ok_trailing_ws_crlf": "%%MatrixMarket matrix array real general\r\n1 2\r\n1.5  \r\n-2e3\t\r\n",
    "ok_integer_field": "%%MatrixMarket matrix array integer general\n1 1\n7\n",
    "ok_empty": "%%MatrixMarket matrix array real general\n0 3\n",
    "ok_overflow_at_line_end": "%%MatrixMarket matrix array real general\n1 2\n1e999\n1\n2\n",
    "malformed_word": "%%MatrixMarket matrix array real general\n2 2\n1.0\n2.0\nnope\n4.0\n",
    "malformed_suffix": "%%MatrixMarket matrix array real general\n1 2\n1.5x 2\n",
    "malformed_overflow_mid": "%%MatrixMarket matrix array real general\n1 2\n1e999 2\n",
    "too_many": "%%MatrixMarket matrix array real general\n1 2\n1 2 3\n",
    "too_few": "%%MatrixMarket matrix array real general\n2 2\n1 2 3\n",
    "bad_size": "%%MatrixMarket matrix array real general\n2\n1\n",
    "negative_size": "%%MatrixMarket matrix array real general\n-1 2\n",
    "missing_size": "%%MatrixMarket matrix array real general\n% only\n",
    "coordinate": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n",
    "pattern": "%%MatrixMarket matrix array pattern general\n1 1\n",
    "bad_banner": "%MatrixMarket matrix array real general\n1 1\n1\n",
    "empty": "",
}

SPECTRUM_CASES = {
    "ok": "3\n2.5\n1\n",
    "ok_comments": "# exact\n\n  5 trailing words ignored\n\t# x\n4\n4\n0\n",
    "ok_tolerance": "1\n1.0000000000005\n",
    "increasing": "1\n2\n",
    "negative": "1\n-0.5\n",
    "word": "1\nabc\n",
    "empty": "# nothing\n\n",
    "inf_text": "inf\n",
}


def _dense_outcome(fn):
    try:
        a = fn()
    except E.ParseError as e:
        return ("ParseError", e.line, str(e))
    except E.Error as e:
        return (type(e).__name__, str(e))
    return ("ok", a.shape, np.asarray(a).ravel(order="F").tobytes())


@pytest.mark.parametrize("name", sorted(DENSE_CASES))
def test_dense_array_parser_matches_reference(tmp_path, reference, name):
    p = tmp_path / "d.mtx"
    with open(p, "w", newline="") as f:
        f.write(DENSE_CASES[name])
    assert _dense_outcome(lambda: d.load_dense_array(str(p))) == \
        _dense_outcome(lambda: reference.load_dense_array(str(p)))


@pytest.mark.parametrize("name", sorted(SPECTRUM_CASES))
def test_spectrum_parser_matches_reference(tmp_path, reference, name):
    p = tmp_path / "s.txt"
    p.write_text(SPECTRUM_CASES[name])
    assert _dense_outcome(lambda: d.load_reference_spectrum(str(p))) == \
        _dense_outcome(lambda: reference.load_spectrum(str(p)))


def test_dense_and_spectrum_writers_match_reference(tmp_path, reference):
    rng = np.random.default_rng(9)
    a = np.asfortranarray(rng.standard_normal((7, 3)) * 10.0 ** rng.integers(-200, 200, (7, 3)))
    d.write_dense_array(str(tmp_path / "o.mtx"), a)
    reference.write_dense_array(str(tmp_path / "r.mtx"), a)
    assert (tmp_path / "o.mtx").read_bytes() == (tmp_path / "r.mtx").read_bytes()
    assert np.array_equal(d.load_dense_array(str(tmp_path / "o.mtx")), a)
    s = np.sort(np.abs(rng.standard_normal(9)))[::-1]
    d.write_reference_spectrum(str(tmp_path / "o.txt"), s)
    reference.write_spectrum(str(tmp_path / "r.txt"), s)
    assert (tmp_path / "o.txt").read_bytes() == (tmp_path / "r.txt").read_bytes()
    assert np.array_equal(d.load_reference_spectrum(str(tmp_path / "o.txt")), s)
    assert d.eps_sigma(s[:4] * (1 + 1e-9), s) == pytest.approx(1e-9, rel=1e-6)
