"""SpMM microbenchmarks on the C2 matrix: both passes, hub vs bulk halves,
hub-kernel variants and thresholds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2404_09276_b200 as d

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
a = bench.make_matrix(cfg)
l = cfg["k"] + cfg["s"]
for thr in (4096, 16384):
    dev = d.Device(0)
    dev.set_option("hub_threshold", thr)
    m = d.DeviceMatrix(a, dev)
    ha, hat = m.hub_rows()
    print(f"threshold {thr}: hub rows A={ha} A^T={hat}")
    for tr in (0, 1):
        for var in (0, 2):
            full = m.bench_spmm(tr, l, var)
            hub = m.bench_spmm(tr, l, var + 16)
            bulk = m.bench_spmm(tr, l, var + 32)
            print(f"  pass {'2 (A^T)' if tr else '1 (A)  '} variant {var}: full {full:7.3f} ms  hub-only {hub:7.3f}  bulk-only {bulk:7.3f}")
    m.close(); dev.close()
