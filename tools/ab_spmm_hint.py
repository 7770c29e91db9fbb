"""A/B of the bulk SpMM L2 eviction hints (spmm_variant bits 64 / 128) on C2:
per-pass SpMM time and one full solve each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
a = bench.make_matrix(cfg)
l = cfg["k"] + cfg["s"]
scfg = bench.solver_config(cfg)
for hint in (0, 64, 128, 0):
    dev = d.Device(0, profiling=True)
    dev.set_option("spmm_variant", hint)
    m = d.DeviceMatrix(a, dev)
    p = [m.bench_spmm(tr, l, hint) for tr in (0, 1)]
    r = d.solve(a, scfg, device=dev)
    r = d.solve(a, scfg, device=dev)
    st = r.stats
    print(f"hint {hint:3d}: pass1 {p[0]:.3f} ms pass2 {p[1]:.3f} ms | solve {st['total_ms']:.1f} ms "
          f"spmm {st['spmm_pass_ms'][0]:.1f}/{st['spmm_pass_ms'][1]:.1f}", flush=True)
    m.close()
    dev.close()
