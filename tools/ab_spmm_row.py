"""A/B of the whole-row SpMM kernel (spmm_variant 64 = bulk rows, 128 = split
chunks) against the 64-column slab kernel on a BASELINE config (default C2)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
a = bench.make_matrix(cfg)
l = cfg["k"] + cfg["s"]
scfg = bench.solver_config(cfg)
ref = None
for var in [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else (0, 64, 128, 192, 0):
    dev = d.Device(0, profiling=True)
    dev.set_option("spmm_variant", var)
    m = d.DeviceMatrix(a, dev)
    p = [m.bench_spmm(tr, l, var) for tr in (0, 1)]
    pl = [m.bench_spmm(tr, l, var + 16) for tr in (0, 1)]
    pb = [m.bench_spmm(tr, l, var + 32) for tr in (0, 1)]
    r = d.solve(a, scfg, device=dev)
    r = d.solve(a, scfg, device=dev)
    st = r.stats
    same = "" if ref is None else f" max|ds|/s {np.max(np.abs(r.svd.s - ref) / ref):.1e}"
    if ref is None:
        ref = r.svd.s.copy()
    print(f"variant {var:3d}: pass1 {p[0]:.3f} (chunks {pl[0]:.3f}, bulk {pb[0]:.3f}) ms  pass2 {p[1]:.3f} "
          f"(chunks {pl[1]:.3f}, bulk {pb[1]:.3f}) ms | solve {st['total_ms']:.1f} ms "
          f"spmm {st['spmm_pass_ms'][0]:.1f}/{st['spmm_pass_ms'][1]:.1f}{same}", flush=True)
    m.close()
    dev.close()
