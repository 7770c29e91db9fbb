"""A/B of the SpMM kernels on a BASELINE config: per-pass time of the default
whole-row kernels (+ split chunks beside them) against the slab-major column-slab
kernel (spmm_variant bits: 4096 = 32-column slabs, 8192 = 64, +16384 L2
evict_first hints on the streaming bytes, +32768 gather depth 4 at 24 warps/SM,
+65536 depth 2 at 40 warps/SM), then a full solve with each variant.

    python tools/ab_spmm_slab.py c4 0,4096,20480,8192,24576
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
variants = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,4096,20480,8192,24576").split(",")]
solve = "--no-solve" not in sys.argv
dev = d.Device(0)
a = bench.make_matrix(cfg, dev)
dev.close()
l = cfg["k"] + cfg["s"]
scfg = bench.solver_config(cfg)
ref = None
for v in variants:
    dev = d.Device(0, profiling=True)
    m = d.DeviceMatrix(a, dev)
    p = [m.bench_spmm(tr, l, v, iters=5) for tr in (0, 1)]
    m.close()
    line = f"variant {v:6d}: pass1 {p[0]:8.3f} ms  pass2 {p[1]:8.3f} ms"
    if solve:
        dev.set_option("spmm_variant", v)
        r = d.solve(a, scfg, device=dev)
        r = d.solve(a, scfg, device=dev)
        st = r.stats
        same = "" if ref is None else (" bitwise=" + str(bool((r.svd.s == ref).all())))
        if ref is None:
            ref = r.svd.s.copy()
        line += (f" | solve total {st['total_ms']:.1f} ms spmm {st['spmm_pass_ms'][0]:.1f}/{st['spmm_pass_ms'][1]:.1f}"
                 f" gram {st['gram_ms']:.1f} rescale {st['rescale_ms']:.1f}{same}")
    print(line, flush=True)
    dev.close()
