"""Unique-edge counts of the device R-MAT generator for a few draw counts (picks the
draws that give BASELINE.json's ~100M (scale 22) and ~1B (scale 24) unique edges)."""
import sys
import time

import paper_2404_09276_b200 as d

dev = d.Device(0)
scale = int(sys.argv[1])
for draws in [int(x) for x in sys.argv[2:]]:
    t = time.perf_counter()
    m = d.rmat(scale, draws, uniform_values=scale >= 24, seed=0, device=dev)
    dt = time.perf_counter() - t
    print(f"scale {scale} draws {draws} unique {m.nnz} ({m.nnz / draws:.4f}) {dt:.2f}s", flush=True)
    m.close()
