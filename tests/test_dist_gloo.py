"""CPU, world_size 2 (gloo): the row-sharded dashSVD algorithm the native
engine runs across GPUs (engine.cu solve_tall with a communicator; comm.cu),
restated with the oracle's kernels and torch.distributed collectives:

  Omega_g    = rows [r_g, r_g+1) of the global sketch, Omega(i, j) = normal_at(seed, j*m + i)
  T_0        = allreduce_g( A_g^T Omega_g ),        (s, V) = eigSVD(T_0)
  loop:  P   = allreduce_g( A_g^T (A_g T) ) - alpha T  (shift applied once, after the sum)
         T   = P V / s   (= A^T A Q - alpha Q with Q = T V / s: the deferred rescale
                          of the native loop, which runs both passes on T so the l x l
                          eig overlaps the A T pass)
         (s, V) = eigSVD(T), shift update / PVE stop (replicated)
  finalize:  B_g = A_g Q, G = allreduce_g(B_g^T B_g), eig(G), U_g = B_g V' / s, V = Q V'

and checked against the single-process oracle solve: same iteration count,
singular values to 1e-10, subspaces to 1e-8. Also pins the shard bounds and
the offset formula of the sharded Gaussian sketch.
"""
import os
import socket

import numpy as np
import pytest

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def sharded_solve(orc, a_full, k, s, alg, p=-1, tol=1e-2, p_max=100, seed=0):
    import torch
    import torch.distributed as dist
    from oracle_lib import Csr
    from paper_2404_09276_b200.sharding import shard_bounds

    rank, world = dist.get_rank(), dist.get_world_size()
    m, n = a_full.rows, a_full.cols
    l = k + s
    b = shard_bounds(a_full.offsets, world)
    r0, r1 = b[rank], b[rank + 1]
    lo, hi = int(a_full.offsets[r0]), int(a_full.offsets[r1])
    a = Csr(r1 - r0, n, a_full.offsets[r0:r1 + 1] - lo, a_full.col_indices[lo:hi].copy(),
            a_full.values[lo:hi].copy())
    at = orc.transpose(a)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x.ravel(order="F")))
        dist.all_reduce(t)
        return np.asfortranarray(t.numpy().reshape(x.shape, order="F"))

    # Omega rows of this shard with the global index formula
    om = np.empty((r1 - r0, l), order="F")
    for j in range(l):
        for i in range(r1 - r0):
            om[i, j] = orc.normal_at(seed, j * m + r0 + i)
    t = allreduce(orc.spmm(at, om))
    q, sv, vv = orc.eig_svd(t)
    dash = alg == "dash"
    max_iters = p_max if dash else p
    alpha, alpha_stored = 0.0, 0.0
    s_stored = np.zeros(l)
    iters, stop_reason = 0, ("p_max_reached" if dash else "fixed_p")
    for j in range(1, max_iters + 1):
        pj = allreduce(orc.spmm(at, orc.spmm(a, t)))
        if alpha != 0.0:
            pj = orc.add_scaled(pj, -alpha, t)
        t = np.asfortranarray(orc.matmul(pj, vv) * (1.0 / sv))
        u, sv, vv = orc.eig_svd(t)
        iters = j
        stop = dash and orc.pve_stop_check(s_stored, alpha_stored, sv, alpha, k, tol)
        q = u
        if stop:
            stop_reason = "tol_met"
            break
        if alg != "fixed_shift" or j == 1:
            alpha = orc.update_shift(alpha, sv[l - 1])
        s_stored, alpha_stored = sv, alpha
    # finalize with the reduced Gram
    bg = orc.spmm(a, q)
    g = allreduce(orc.gram(bg))
    w, vec = orc.sym_eig(g)
    lam_max = max(w[-1], 0.0)
    floor = float(max(m, l)) * np.finfo(float).eps * np.sqrt(lam_max)
    assert np.all(w[::-1] > floor * floor)
    svals = np.sqrt(w[::-1])
    vp = np.asfortranarray(vec[:, ::-1])
    for c in range(l):  # sign convention (decompositions.cpp:21-35)
        nz = np.flatnonzero(vp[:, c] != 0.0)
        if nz.size and vp[nz[0], c] < 0:
            vp[:, c] = -vp[:, c]
    ug = orc.matmul(bg, vp) * (1.0 / svals)
    v_out = orc.matmul(q, vp[:, :k])
    parts = [None] * world
    dist.all_gather_object(parts, ug[:, :k])
    u_full = np.vstack(parts)
    return dict(u=u_full, s=svals[:k], v=v_out, iterations=iters, stop_reason=stop_reason,
                bounds=b)


def _worker(rank, port, result_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(WORLD))
    import torch.distributed as dist
    from oracle_lib import Oracle
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        orc = Oracle()
        out = {}
        a = orc.sparse_random(300, 120, 8, 7, True)
        out["dash"] = sharded_solve(orc, a, 10, 6, "dash", tol=1e-2, seed=3)
        out["shifted"] = sharded_solve(orc, a, 10, 6, "shifted", p=5, seed=4)
        if rank == 0:
            np.save(result_path, out, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_row_sharded_algorithm_matches_single_process(tmp_path, oracle):
    import torch.multiprocessing as mp
    path = str(tmp_path / "res.npy")
    mp.start_processes(_worker, args=(_free_port(), path), nprocs=WORLD, start_method="spawn")
    res = np.load(path, allow_pickle=True).item()
    a = oracle.sparse_random(300, 120, 8, 7, True)
    for key, ref in (("dash", oracle.solve(a, 10, 6, tol=1e-2, alg="dash", seed=3)),
                     ("shifted", oracle.solve(a, 10, 6, p=5, alg="shifted", seed=4))):
        r = res[key]
        assert r["iterations"] == ref["iterations"] and r["stop_reason"] == ref["stop_reason"]
        np.testing.assert_allclose(r["s"], ref["s"], rtol=1e-10)
        for name in ("u", "v"):
            q1, _ = np.linalg.qr(ref[name])
            q2, _ = np.linalg.qr(r[name])
            assert np.linalg.norm(q2 - q1 @ (q1.T @ q2), 2) < 1e-8
        b = r["bounds"]
        assert b[0] == 0 and b[-1] == 300
