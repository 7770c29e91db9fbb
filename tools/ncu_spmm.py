"""Kernels to capture under ncu on a BASELINE config.

    python tools/ncu_spmm.py c4 spmm 0,8192   # one SpMM launch per variant and pass
    python tools/ncu_spmm.py c4 solve         # a p = 1 solve (Gram, eig, rescale of the loop's shapes)

e.g. ncu --set full -k regex:"spmm_(slab|row)" python tools/ncu_spmm.py c4 spmm 0,8192
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
mode = sys.argv[2] if len(sys.argv) > 2 else "spmm"
dev = d.Device(0)
for kv in [x for x in sys.argv[3:] if "=" in x]:  # context options, e.g. spmm_slab=64
    k_, v_ = kv.split("=")
    dev.set_option(k_, int(v_))
a = bench.make_matrix(cfg, dev)
l = cfg["k"] + cfg["s"]
if mode == "spmm":
    variants = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 and "=" not in sys.argv[3] else "0,8192").split(",")]
    m = d.DeviceMatrix(a, dev)
    for v in variants:
        for tr in (0, 1):
            m.bench_spmm(tr, l, v, iters=1)
    m.close()
else:
    cfg.update(p=1, alg="shifted")
    d.solve(a, bench.solver_config(cfg), device=dev)
dev.close()
