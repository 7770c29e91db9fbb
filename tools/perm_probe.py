"""Does a degree-sorted relabelling of rows and columns (hot rows of X and Y
contiguous) speed up the SpMM passes of a DRAM-bound config? Prototype: builds
P_r A P_c^T on the host (numpy), uploads both and times bench_spmm per pass."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
dev = d.Device(0)
a = bench.make_matrix(cfg, dev)
l = cfg["k"] + cfg["s"]
rows_of = np.repeat(np.arange(a.rows, dtype=np.int64), np.diff(a.offsets))
cdeg = np.bincount(a.col_indices, minlength=a.cols)
rdeg = np.diff(a.offsets)
pc = np.empty(a.cols, dtype=np.int64)
pc[np.argsort(-cdeg, kind="stable")] = np.arange(a.cols)  # new id of each column
pr = np.empty(a.rows, dtype=np.int64)
pr[np.argsort(-rdeg, kind="stable")] = np.arange(a.rows)
nr, nc = pr[rows_of], pc[a.col_indices]
order = np.lexsort((nc, nr))
off = np.zeros(a.rows + 1, dtype=np.int64)
np.cumsum(np.bincount(nr, minlength=a.rows), out=off[1:])
b = d.SparseMatrix(a.rows, a.cols, off, nc[order], a.values[order])
for name, mat in (("original", a), ("degree-sorted", b)):
    m = d.DeviceMatrix(mat, dev)
    p1 = min(m.bench_spmm(False, l, 0) for _ in range(3))
    p2 = min(m.bench_spmm(True, l, 0) for _ in range(3))
    print(f"{name:14s} pass1 {p1:.3f} ms  pass2 {p2:.3f} ms", flush=True)
    m.close()
