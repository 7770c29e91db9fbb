"""TEST INFRASTRUCTURE ONLY — numpy restatements of the input side of the path
(SURVEY 8(f) row 2), used by tests/ as the CHECKER of the device kernels in
paper_2404_09276_b200/csrc/ingest.cu. Nothing in paper_2404_09276_b200/ imports it.

- assemble_np: assemble() of the reference, matrix_market.cpp:90-115 (sort by
  (row, col), duplicates summed left to right, exact zeros dropped, offsets by
  counting). Pinned by tests/golden/input_golden.json (the unmodified reference's
  load_matrix_market outcomes, tests/golden/make_input_golden.py).
- splitmix64_np: random.cpp:8-13.
- rmat_np: the R-MAT rule of dsvd_synth_rmat (ingest.cuh; the reference ships no
  R-MAT generator, BASELINE.json configs 4/5 define the graph family).
"""
from dataclasses import dataclass

import numpy as np


@dataclass
class Csr:
    rows: int
    cols: int
    offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])


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
