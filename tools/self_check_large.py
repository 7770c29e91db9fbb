"""Reference-free checks of a full-size solve (used for C5 at R-MAT scale 24, where the
reference does not fit in host memory): triplet residuals max_i ||A v_i - s_i u_i|| /
s_1 on the device, orthonormality of U and V, the stop rule's PVE ratio at termination,
and descending singular values. Writes gpurun_out/selfcheck_<config>.json."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

name = sys.argv[1]
cfg = dict(bench.CONFIGS[name])
dev = d.Device(0)
m = d.rmat(cfg["rmat_scale"], cfg["draws"], uniform_values=cfg["uniform"], seed=cfg["gen_seed"], device=dev) \
    if "rmat_scale" in cfg else d.DeviceMatrix(bench.make_matrix(cfg, dev), dev)
scfg = bench.solver_config(cfg)
t0 = time.perf_counter()
res = m.solve(scfg)
t_solve = time.perf_counter() - t0
s = res.svd.s
dev.trim()  # release the solve workspaces before the metric uploads U and V
resid = d.max_triplet_residual(m, res.svd, device=dev)
u, v = res.svd.u, res.svd.v
ortho_u = float(np.abs(u.T @ u - np.eye(u.shape[1])).max())
ortho_v = float(np.abs(v.T @ v - np.eye(v.shape[1])).max())
al, sh = np.array(res.trace.alphas), np.array(res.trace.s_hat_history)
n = len(al)
k = scfg.k
pve = float(np.max(np.abs(sh[n - 2][:k] + al[n - 1] - sh[n - 1][:k] - al[n - 1]) / (sh[n - 1][k] + al[n - 1])))
rec = {"config": name, "workload": cfg["name"], "rows": m.rows, "cols": m.cols, "nnz": m.nnz,
       "solve_s_handle": t_solve, "iterations": res.trace.iterations, "stop_reason": res.trace.stop_reason.name,
       "pve_ratio_at_stop": pve, "tol": scfg.tol, "sigma_1": float(s[0]), "sigma_k": float(s[-1]),
       "max_triplet_residual": resid, "max_triplet_residual_rel_sigma1": resid / float(s[0]),
       "orthonormality_u": ortho_u, "orthonormality_v": ortho_v,
       "sigma_descending": bool(np.all(np.diff(s) <= 0))}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"selfcheck_{name}.json"), "w") as f:
    json.dump(rec, f, indent=1)
print(json.dumps(rec))
