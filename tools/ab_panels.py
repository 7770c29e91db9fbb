"""A/B of the split-chunk X panels (ctx option split_panel_rows) on C2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
panels = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 16384, 32768, 65536]
a = bench.make_matrix(cfg)
l = cfg["k"] + cfg["s"]
scfg = bench.solver_config(cfg)
for pr in panels:
    dev = d.Device(0, profiling=True)
    dev.set_option("split_panel_rows", pr)
    m = d.DeviceMatrix(a, dev)
    p = [m.bench_spmm(tr, l, 0) for tr in (0, 1)]
    pl = [m.bench_spmm(tr, l, 16) for tr in (0, 1)]
    r = d.solve(a, scfg, device=dev)
    r = d.solve(a, scfg, device=dev)
    st = r.stats
    print(f"panel {pr:6d}: pass1 {p[0]:.3f} (chunks {pl[0]:.3f}) ms  pass2 {p[1]:.3f} (chunks {pl[1]:.3f}) ms"
          f" | solve {st['total_ms']:.1f} spmm {st['spmm_pass_ms'][0]:.1f}/{st['spmm_pass_ms'][1]:.1f}", flush=True)
    m.close()
    dev.close()
