"""Input-side test cases, shared by tests/golden/make_input_golden.py
and tests/test_inputs.py / tests/test_gpu_inputs.py.

MTX_CASES: Matrix Market texts covering what load_matrix_market (matrix_market.cpp:117-165)
distinguishes: header spellings and unsupported declarations, comment / blank / CRLF
lines, the three fields, symmetric / skew-symmetric expansion, duplicates (summed, exact
cancellation dropped), explicit zeros, the number syntax the istream extraction accepts
and rejects, size-line and entry-line errors with their line numbers.

corrupt_csr(seed): a small canonical CSR with one seeded violation of
SparseMatrix::validate (sparse_matrix.cpp:12-33), or none.
"""
import numpy as np

from oracle_lib import Csr
from inputs_oracle import assemble_np, rmat_np, splitmix64_np  # noqa: F401  (re-exported)

H = "%%MatrixMarket matrix coordinate real general\n"

MTX_CASES = {
    # ---- accepted files ----------------------------------------------------------
    "general": H + "3 4 4\n1 2 0.5\n3 4 -2\n2 1 1e-3\n1 1 4\n",
    "unsorted_rows": H + "4 3 5\n4 3 1\n1 3 2\n4 1 3\n2 2 4\n1 1 5\n",
    "case_insensitive_header": "%%MatrixMarket MATRIX Coordinate REAL General\n2 2 1\n2 2 9.25\n",
    "extra_header_tokens": "%%MatrixMarket matrix coordinate real general whatever\n1 1 1\n1 1 3\n",
    "comments_blank_crlf": "%%MatrixMarket matrix coordinate real general\r\n% c1\r\n\r\n  \t\r\n"
                           "2 3 2\r\n% mid\r\n1 3 1.5\r\n\r\n2 1 -0.25\r\n",
    "tabs_and_spaces": H + "\t2  2\t2 \n  1\t1   7 \n2 2\t-7\t\n",
    "no_final_newline": H + "2 2 2\n1 1 1\n2 2 2",
    "trailing_lines_ignored": H + "2 2 1\n1 1 1\n2 2 5\ngarbage here\n",
    "integer_field": "%%MatrixMarket matrix coordinate integer general\n2 3 3\n1 1 3\n2 3 -4\n1 2 0\n",
    "pattern_field": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n1 1\n3 2\n2 3\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 5\n1 1 2\n3 1 -1.5\n4 2 0.25\n"
                 "4 4 8\n2 1 3\n",
    "symmetric_zero_offdiag": "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 0\n3 3 1\n",
    "symmetric_pattern": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 1\n3 1\n3 2\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 3\n2 1 1.5\n3 1 -2\n3 2 4\n",
    "skew_zero_diag": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 2\n1 1 0\n2 1 6\n",
    "duplicates_summed": H + "2 2 4\n1 1 1.5\n2 1 -1\n1 1 2\n1 1 0.25\n",
    "duplicates_cancel": H + "3 3 4\n2 2 5\n1 3 1\n2 2 -5\n3 3 2\n",
    "explicit_zeros": H + "2 2 3\n1 1 0\n1 2 -0.0\n2 2 1\n",
    "empty_rows_cols": H + "5 6 2\n5 6 1\n1 1 2\n",
    "zero_entries": H + "3 2 0\n",
    "zero_dims": H + "0 0 0\n",
    "number_forms": H + "2 5 9\n1 1 1.\n1 2 .5\n1 3 -.5e-3\n1 4 +2\n1 5 1E+2\n2 1 4.9e-324\n"
                    "2 2 1.7976931348623157e308\n2 3 0.1\n2 4 -0\n",
    "index_plus_sign": H + "2 2 1\n+2 +1 3\n",
    "underflow_to_zero": H + "2 2 2\n1 1 1e-400\n2 2 1\n",
    "hex_value_prefix": H + "1 1 1\n1 1 0x10\n",
    # ---- parse errors --------------------------------------------------------------
    "empty_file": "",
    "blank_first_line": "\n" + H + "1 1 0\n",
    "bad_banner": "%%MatrixMarkt matrix coordinate real general\n1 1 0\n",
    "banner_only_no_size": H,
    "comments_only_no_size": H + "% a\n% b\n\n",
    "size_word": H + "2 two 1\n1 1 1\n",
    "size_two_numbers": H + "2 2\n",
    "size_trailing": H + "2 2 1 9\n1 1 1\n",
    "size_trailing_comment": H + "2 2 1 % c\n1 1 1\n",
    "size_negative": H + "2 -2 1\n1 1 1\n",
    "size_overflow": H + "99999999999999999999 2 1\n1 1 1\n",
    "too_few_entries": H + "2 2 3\n1 1 1\n% c\n2 2 2\n",
    "entry_one_index": H + "2 2 1\n1\n",
    "entry_float_index": H + "2 2 1\n1.0 1 1\n",
    "entry_no_value": H + "2 2 1\n1 1\n",
    "entry_trailing": H + "2 2 1\n1 1 1.0 junk\n",
    "entry_value_suffix": H + "2 2 1\n1 1 1.0x\n",
    "entry_incomplete_exponent": H + "2 2 1\n1 1 1e\n",
    "entry_exponent_sign_only": H + "2 2 1\n1 1 2e+\n",
    "entry_inf": H + "2 2 1\n1 1 inf\n",
    "entry_nan": H + "2 2 1\n1 1 nan\n",
    "entry_overflow": H + "2 2 1\n1 1 1e400\n",
    "entry_dot_only": H + "2 2 1\n1 1 .\n",
    "entry_row_oob": H + "2 2 1\n3 1 1\n",
    "entry_col_zero": H + "2 2 1\n1 0 1\n",
    "entry_negative_index": H + "2 2 1\n-1 1 1\n",
    "pattern_with_value": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2 7.0\n",
    "skew_nonzero_diag": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 2 1\n",
    "error_after_comments": H + "% x\n\n2 2 2\n% y\n1 1 1\n\n% z\n2 2 oops\n",
    # ---- unsupported declarations ------------------------------------------------------
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n2 2 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n2 2 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "vector_object": "%%MatrixMarket vector coordinate real general\n2 2 0\n",
    "unknown_format": "%%MatrixMarket matrix sparse real general\n2 2 0\n",
    "short_header": "%%MatrixMarket matrix\n2 2 0\n",
}


def small_csr(rng, rows=12, cols=9, density=0.35) -> Csr:
    mask = rng.random((rows, cols)) < density
    vals = rng.standard_normal((rows, cols))
    off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(mask.sum(axis=1), out=off[1:])
    ri, ci = np.nonzero(mask)
    return Csr(rows, cols, off, ci.astype(np.int64), vals[ri, ci].astype(np.float64))


def corrupt_csr(seed: int) -> Csr:
    """A canonical matrix with at most a couple of seeded violations (kind by seed)."""
    rng = np.random.default_rng(seed)
    a = small_csr(rng)
    off, idx, val = a.offsets.copy(), a.col_indices.copy(), a.values.copy()
    nnz = val.size
    for _ in range(1 + seed % 2):
        kind = int(rng.integers(0, 9))
        p = int(rng.integers(0, nnz))
        if kind == 0:
            idx[p] = a.cols + int(rng.integers(0, 3))
        elif kind == 1:
            idx[p] = -1
        elif kind == 2 and p + 1 < nnz:
            idx[p], idx[p + 1] = idx[p + 1], idx[p]
        elif kind == 3:
            val[p] = np.nan
        elif kind == 4:
            val[p] = -np.inf if seed % 3 else np.inf
        elif kind == 5:
            val[p] = 0.0
        elif kind == 6:
            i = int(rng.integers(1, a.rows))
            off[i] = min(off[i + 1] + 1, nnz)  # may create a decrease
        elif kind == 7 and p + 1 < nnz:
            idx[p + 1] = idx[p]  # repeated column
        elif kind == 8:
            pass  # leave this one valid
    if seed % 17 == 0:
        off[-1] = nnz + 1
    return Csr(a.rows, a.cols, off, idx, val)
