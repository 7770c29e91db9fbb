"""A/B of one context option on a BASELINE config: SpMM passes and a full solve.
python tools/ab_option.py c2 split_chunk_t 0,256,128 [base_opt=value,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
name = sys.argv[2]
vals = [int(v) for v in sys.argv[3].split(",")]
base = [kv.split("=") for kv in sys.argv[4].split(",") if "=" in kv] if len(sys.argv) > 4 else []
a = bench.make_matrix(cfg)
l = cfg["k"] + cfg["s"]
scfg = bench.solver_config(cfg)
ref = None
for v in vals:
    dev = d.Device(0, profiling=True)
    for bk, bv in base:
        dev.set_option(bk, int(bv))
    dev.set_option(name, v)
    m = d.DeviceMatrix(a, dev)
    p = [m.bench_spmm(tr, l, 0) for tr in (0, 1)] if "--no-bench" not in sys.argv else [0.0, 0.0]
    m.close()
    dev.trim()  # the microbenchmark's blocks (C5: 2 x 20 GB) before the solve's
    r = d.solve(a, scfg, device=dev)
    r = d.solve(a, scfg, device=dev)
    st = r.stats
    diff = "" if ref is None else f" max|ds|/s {abs(r.svd.s - ref).max() / ref.max():.1e}"
    if ref is None:
        ref = r.svd.s.copy()
    print(f"{name}={v}: pass1 {p[0]:.3f} ms pass2 {p[1]:.3f} ms | solve spmm {st['spmm_pass_ms'][0]:.1f}/"
          f"{st['spmm_pass_ms'][1]:.1f} ms gram {st['gram_ms']:.1f} rescale {st['rescale_ms']:.1f} eig {st['eig_ms']:.1f} ms "
          f"sweeps {st['eig_sweeps']} total {st['total_ms']:.1f}{diff}", flush=True)
    dev.close()
