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
