"""One C2 solve (BASELINE.json configs[1]) for ncu launch lists / full captures:

    python tools/profile_solve.py [c2|c1] [warm]

DSVD_OPTIONS="name=value,..." sets context options first (e.g. eig_method=1).

With "warm", one untimed solve runs first so the profiled launches are the
second solve's (ncu -s skips the first solve's launches).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = bench.CONFIGS[key]
    a = bench.make_matrix(cfg)
    scfg = bench.solver_config(cfg)
    dev = d.Device(0, profiling=True)
    for kv in filter(None, os.environ.get("DSVD_OPTIONS", "").split(",")):  # e.g. eig_method=1
        k, v = kv.split("=")
        dev.set_option(k, int(v))
    if "warm" in sys.argv[2:]:
        d.solve(a, scfg, device=dev)
    r = d.solve(a, scfg, device=dev)
    st = r.stats
    print({k: st[k] for k in ("total_ms", "spmm_ms", "spmm_pass_ms", "gram_ms", "eig_ms",
                              "rescale_ms", "eig_sweeps", "kernel_launches")})


if __name__ == "__main__":
    main()
