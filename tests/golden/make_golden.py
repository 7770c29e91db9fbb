"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference by oracle/Makefile). Run in the dev container:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the oracle restatement (tests/test_oracle_golden.py) without
needing /root/reference at test time; the GPU tests (tests/test_gpu_*.py) then
compare the device path against that pinned oracle. Large factors are stored as wrapping bit-sums plus a few rows.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Reference  # noqa: E402


def bitsum(x):
    return np.uint64(np.ascontiguousarray(np.asarray(x).ravel(order="F")).view(np.uint64).sum(dtype=np.uint64))


def main():
    ref = Reference()
    ref.set_threads(4)
    out = {}

    # ---- config 1 (BASELINE.json configs[0]) -------------------------------
    a = ref.sparse_random(10000, 5000, 25, 0, True)
    out["c1_nnz"] = np.int64(a.nnz)
    out["c1_offsets_bitsum"] = bitsum(a.offsets)
    out["c1_idx_bitsum"] = bitsum(a.col_indices)
    out["c1_val_bitsum"] = bitsum(a.values)
    at = ref.transpose(a)
    out["c1t_offsets_bitsum"] = bitsum(at.offsets)
    out["c1t_idx_bitsum"] = bitsum(at.col_indices)
    out["c1t_val_bitsum"] = bitsum(at.values)
    om = ref.gaussian_matrix(10000, 75, 0)
    out["c1_omega_bitsum"] = bitsum(om)
    t0 = ref.spmm(at, om)
    out["c1_at_omega_bitsum"] = bitsum(t0)
    g0 = ref.gram(t0)
    out["c1_gram0"] = g0
    s = ref.solve(a, 50, 25, p=10, alg="shifted", seed=0)
    out["c1_shifted_s"] = s["s"]
    out["c1_shifted_alphas"] = s["alphas"]
    out["c1_shifted_s_hat"] = s["s_hat"]
    out["c1_shifted_u_bitsum"] = bitsum(s["u"])
    out["c1_shifted_v_bitsum"] = bitsum(s["v"])
    out["c1_shifted_u_head"] = s["u"][:20].copy()
    out["c1_shifted_v_head"] = s["v"][:20].copy()
    dsh = ref.solve(a, 50, 25, tol=1e-2, alg="dash", seed=0)
    out["c1_dash_iterations"] = np.int64(dsh["iterations"])
    out["c1_dash_s"] = dsh["s"]
    out["c1_dash_alphas"] = dsh["alphas"]
    out["c1_dash_s_hat"] = dsh["s_hat"]

    # ---- small full-factor cases ---------------------------------------------
    b = ref.sparse_random(150, 90, 8, 6, True)
    for key, arr in (("b_off", b.offsets), ("b_idx", b.col_indices), ("b_val", b.values)):
        out[key] = arr
    r = ref.solve(b, 12, 6, tol=1e-2, alg="dash", seed=17)
    for key in ("u", "s", "v", "alphas", "s_hat"):
        out["b_dash_" + key] = r[key]
    out["b_dash_iterations"] = np.int64(r["iterations"])
    w = ref.sparse_random(60, 100, 8, 44, True)
    for key, arr in (("w_off", w.offsets), ("w_idx", w.col_indices), ("w_val", w.values)):
        out[key] = arr
    r = ref.solve(w, 8, 4, tol=1e-2, alg="dash", seed=2)
    for key in ("u", "s", "v", "alphas"):
        out["w_dash_" + key] = r[key]
    r = ref.solve(b, 12, 6, p=4, alg="fixed_shift", seed=3)
    for key in ("s", "alphas"):
        out["b_fixed_" + key] = r[key]

    # ---- dense kernels ----------------------------------------------------------
    c = ref.gaussian_matrix(200, 20, 808)
    out["dense_c"] = c
    out["dense_gram"] = ref.gram(c)
    u, sv, v = ref.eig_svd(c)
    out["dense_eig_u"], out["dense_eig_s"], out["dense_eig_v"] = u, sv, v
    g0 = ref.gaussian_matrix(20, 20, 808)
    gs = np.asfortranarray(g0 + g0.T)
    out["sym_g"] = gs
    out["sym_w"], out["sym_v"] = ref.sym_eig(gs)
    x = ref.gaussian_matrix(90, 13, 5)
    out["spmm_x"] = x
    out["spmm_y"] = ref.spmm(b, x)

    # ---- scalar known answers ----------------------------------------------------
    out["normal_42_0_3"] = np.array([ref.normal_at(42, i) for i in range(4)])
    out["gauss_8x4_2026_bitsum"] = bitsum(ref.gaussian_matrix(8, 4, 2026))

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
