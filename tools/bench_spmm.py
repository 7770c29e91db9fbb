"""SpMM microbenchmarks on a BASELINE config (default C2): both passes, the
long-row part (hub kernel or split chunks) vs the bulk rows, per mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
a = bench.make_matrix(cfg)
l = cfg["k"] + cfg["s"]
modes = [("bitwise, TMA hub >=4096", dict(split_chunk=0, hub_threshold=4096), 0)]
for c in (512, 1024, 2048, 4096, 8192):
    modes.append((f"split chunk {c}", dict(split_chunk=c), 0))
for name, opts, var in modes:
    dev = d.Device(0)
    for k, v in opts.items():
        dev.set_option(k, v)
    m = d.DeviceMatrix(a, dev)
    ha, hat = m.hub_rows()
    line = [f"{name:26s}"]
    for tr in (0, 1):
        full = m.bench_spmm(tr, l, var)
        long_ = m.bench_spmm(tr, l, var + 16)
        bulk = m.bench_spmm(tr, l, var + 32)
        line.append(f"pass{tr + 1}: full {full:6.3f} ms (long rows {long_:6.3f}, bulk {bulk:6.3f})")
    print("  ".join(line), flush=True)
    m.close()
    dev.close()
