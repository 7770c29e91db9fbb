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


def assemble_np(rows, cols, r, c, v) -> Csr:
    """assemble() (matrix_market.cpp:90-115) restated in numpy for the tests: sort by
    (row, col) with a stable sort, sum duplicates in input order, drop exact zeros."""
    r, c, v = (np.asarray(x) for x in (r, c, v))
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order].astype(np.float64)
    if r.size:
        head = np.ones(r.size, dtype=bool)
        head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        starts = np.flatnonzero(head)
        ends = np.append(starts[1:], r.size)
        sums = v[starts].copy()
        for t in np.flatnonzero(ends - starts > 1):  # left-to-right adds, as the reference
            acc = v[starts[t]]
            for q in range(starts[t] + 1, ends[t]):
                acc = acc + v[q]
            sums[t] = acc
        keep = sums != 0.0
        r, c, v = r[starts][keep], c[starts][keep], sums[keep]
    off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=rows), out=off[1:])
    return Csr(rows, cols, off, c.astype(np.int64), v)


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


GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64_np(seed, i):
    """random.cpp:8-13 vectorised (uint64 arithmetic wraps)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.asarray(i, dtype=np.uint64) + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rmat_np(scale, draws, a=0.57, b=0.19, c=0.19, uniform=False, seed=0) -> Csr:
    """The R-MAT rule of dsvd_synth_rmat (ingest.cuh) restated in numpy for the tests."""
    edge_seed = int(splitmix64_np(seed, 0))
    val_seed = int(splitmix64_np(seed, 1))
    ta, tab, tabc = (int(round(x * 65536.0)) for x in (a, a + b, a + b + c))
    H = (scale + 3) // 4
    e = np.arange(draws, dtype=np.uint64)
    row = np.zeros(draws, dtype=np.uint64)
    col = np.zeros(draws, dtype=np.uint64)
    for t in range(scale):
        h = splitmix64_np(edge_seed, e * np.uint64(H) + np.uint64(t // 4))
        q = (h >> np.uint64(16 * (t % 4))) & np.uint64(0xFFFF)
        quad = np.where(q < ta, 0, np.where(q < tab, 1, np.where(q < tabc, 2, 3))).astype(np.uint64)
        row = (row << np.uint64(1)) | (quad >> np.uint64(1))
        col = (col << np.uint64(1)) | (quad & np.uint64(1))
    key = (row << np.uint64(scale)) | col
    uniq, first = np.unique(key, return_index=True)  # first occurrence = smallest draw index
    n = 1 << scale
    r = (uniq >> np.uint64(scale)).astype(np.int64)
    cidx = (uniq & np.uint64(n - 1)).astype(np.int64)
    if uniform:
        v = ((splitmix64_np(val_seed, first.astype(np.uint64)) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
    else:
        v = np.ones(uniq.size)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=off[1:])
    return Csr(n, n, off, cidx, v)
