"""One solve per loop schedule under compute-sanitizer (tools/sanitize.sh):
the smoke-sized case and a config-1 accuracy-controlled solve, serial and
pipelined, plus the SpMM variants (whole-row, column-slab) and a loopback
two-rank sharded solve, so every kernel family of the solve runs once.

    python tools/sanitize_case.py [small|c1]
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09276_b200 as d  # noqa: E402
from paper_2404_09276_b200.sharding import shard_bounds, shard_csr  # noqa: E402

size = sys.argv[1] if len(sys.argv) > 1 else "small"
if size == "c1":
    a = d.sparse_random(10000, 5000, 25, 0, True)
    k, s = 50, 25
else:
    a = d.powerlaw(3000, 1200, 3.0, 1.0, 1.1, 3)  # long rows: split chunks + combine
    k, s = 16, 8
for pipeline in (0, 1):
    for variant in (0, 4096 | 16384):
        dev = d.Device(0)
        dev.set_option("pipeline", pipeline)
        dev.set_option("spmm_variant", variant)
        r = d.solve(a, d.SolverConfig(k=k, s=s, tol=1e-2, seed=0), device=dev)
        print(f"pipeline={pipeline} variant={variant}: N_p={r.trace.iterations} s1={r.svd.s[0]:.12g}", flush=True)
        dev.close()
# fixed-p shifted solve and the basic algorithm with both orthonormalizers
dev = d.Device(0)
d.solve(a, d.SolverConfig(k=k, s=s, p=3, alg=d.Algorithm.shifted, seed=1), device=dev)
d.solve(a, d.SolverConfig(k=k, s=s, p=2, alg=d.Algorithm.basic, seed=1), device=dev)
d.solve(a, d.SolverConfig(k=k, s=s, p=2, alg=d.Algorithm.basic, orth=d.Orthonormalizer.qr, seed=1), device=dev)
dev.close()
# two ranks on one device (loopback group), v2 exchange
group = d.LoopbackGroup(2)
b = shard_bounds(a.offsets, 2)
errs = []


def rank(r):
    try:
        dv = d.Device(0)
        dv.attach_loopback(group, r)
        dv.set_shard(b[r], a.rows)
        d.solve(shard_csr(a, b[r], b[r + 1]), d.SolverConfig(k=k, s=s, p=3, alg=d.Algorithm.shifted), device=dv)
    except Exception as exc:
        errs.append(exc)


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
group.close()
assert not errs, errs
print("sanitize case done", flush=True)
