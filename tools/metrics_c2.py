"""Device validation metrics at C2 scale: solve, then
eps_res / max_triplet_residual / eps_spec (300 power iterations) against the
solve's own s as the reference spectrum proxy (sigma_{k+1} from s_hat)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
a = bench.make_matrix(cfg)
dev = d.Device(0)
m = d.DeviceMatrix(a, dev)
res = d.solve(a, bench.solver_config(cfg), device=dev)
f = res.svd
k = f.s.size
sig = np.r_[f.s, np.sqrt(res.trace.s_hat_history[-1][k])] if res.trace.iterations else f.s
for name, fn in (("max_triplet_residual", lambda: d.max_triplet_residual(m, f)),
                 ("eps_res", lambda: d.eps_res(m, f, sig)),
                 ("eps_spec(300)", lambda: d.eps_spec(m, f, sig, power_iters=300))):
    t0 = time.perf_counter()
    v = fn()
    print(f"{name}: {v:.3e}  ({(time.perf_counter() - t0) * 1e3:.1f} ms)", flush=True)
