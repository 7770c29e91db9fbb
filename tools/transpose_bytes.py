"""Full-size bitwise check of the device CSC build against the UNMODIFIED reference
`transpose` (sparse_matrix.cpp:35-55, compiled as oracle/_ref) on BASELINE.json's
matrices (bench.py CONFIGS): the same generated CSR goes through the device pair build
(build_transpose, sparse.cu) and through the reference; offsets, column indices and
values are compared with memcmp semantics (np.array_equal on the raw bytes).

    python tools/transpose_bytes.py c2 c3 c4

Writes gpurun_out/transpose_bytes.json (copied to profiles/ by hand). Test
infrastructure: runs the reference as the checker only.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
import paper_2404_09276_b200 as d  # noqa: E402
from oracle_lib import Csr, Reference  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8))
    return h.hexdigest()[:16]


def main():
    names = sys.argv[1:] or ["c2", "c3", "c4"]
    dev = d.Device(0)
    ref = Reference()
    ref.set_threads(os.cpu_count())
    out = []
    for name in names:
        cfg = bench.CONFIGS[name]
        a = bench.make_matrix(cfg, dev)
        t0 = time.perf_counter()
        dm = d.DeviceMatrix(a, device=dev)
        t_dev = dm.transpose()
        dev.synchronize()
        t_gpu = time.perf_counter() - t0
        dm.close()
        t0 = time.perf_counter()
        r = ref.transpose(Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values))
        t_ref = time.perf_counter() - t0
        rec = {
            "config": name, "workload": cfg["name"], "rows": a.rows, "cols": a.cols, "nnz": a.nnz,
            "offsets_equal": bool(np.array_equal(t_dev.offsets.view(np.uint8), r.offsets.view(np.uint8))),
            "col_indices_equal": bool(np.array_equal(t_dev.col_indices.view(np.uint8),
                                                     r.col_indices.view(np.uint8))),
            "values_equal": bool(np.array_equal(t_dev.values.view(np.uint8), r.values.view(np.uint8))),
            "sha256_16_device": digest(t_dev.offsets, t_dev.col_indices, t_dev.values),
            "sha256_16_reference": digest(r.offsets, r.col_indices, r.values),
            "device_upload_build_download_s": t_gpu, "reference_transpose_s": t_ref,
        }
        rec["pass"] = rec["offsets_equal"] and rec["col_indices_equal"] and rec["values_equal"]
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del a, t_dev, r
    dev.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "transpose_bytes.json"), "w") as f:
        json.dump(out, f, indent=1)
    if not all(r["pass"] for r in out):
        sys.exit(1)


if __name__ == "__main__":
    main()
