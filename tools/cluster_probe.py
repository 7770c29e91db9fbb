"""Eigenvalue clusters of the in-loop Gram matrices (s_hat^2) for a bench config."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1]])
cfg["p"] = int(sys.argv[2])
dev = d.Device(0)
a = bench.make_matrix(cfg, dev)
res = d.solve(a, bench.solver_config(cfg), device=dev)
for it, sh in enumerate(res.trace.s_hat_history):
    lam = np.asarray(sh) ** 2
    gaps = (lam[:-1] - lam[1:]) / lam[0]
    close = gaps < 1e-9
    runs, cur = [], 0
    for c in close:
        if c:
            cur += 1
        elif cur:
            runs.append(cur + 1)
            cur = 0
    if cur:
        runs.append(cur + 1)
    print(f"iter {it}: min rel gap {gaps.min():.3e}, clustered pairs {close.sum()}, cluster sizes {runs[:20]}, "
          f"lam range {lam[-1] / lam[0]:.3e}")
