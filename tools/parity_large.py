"""Full-size parity of the B200 solve against the UNMODIFIED reference (oracle/_ref) on
BASELINE.json's configs (bench.py CONFIGS): same generated matrix, same config (optionally
with p / p_max reduced so the CPU side finishes in minutes), compared with the north_star
bars: sigma relative error, largest principal angle of the U and V subspaces, iteration
count, stop reason, alpha / s_hat traces, PVE ratio at termination.

    python tools/parity_large.py c2                 # full p = 20
    python tools/parity_large.py c4 --p 2           # C4 with 2 power iterations
    python tools/parity_large.py c3                 # full dash run (tol 1e-2)

Writes profiles/parity_<config>[_p<p>].json. Test infrastructure: runs the reference
(oracle/_ref) as the checker only.
"""
import argparse
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


def sin_theta(u_ref, u):
    """sine of the largest principal angle between span(u_ref) and span(u) (orthonormal
    columns): || u - u_ref (u_ref^T u) ||_2."""
    r = u - u_ref @ (u_ref.T @ u)
    return float(np.linalg.norm(r.T @ r, 2) ** 0.5)


def pve_ratio(alphas, s_hat, k):
    n = len(alphas)
    if n < 2:
        return None
    prev, cur = s_hat[n - 2], s_hat[n - 1]
    return float(np.max(np.abs(prev[:k] + alphas[n - 1] - cur[:k] - alphas[n - 1]) / (cur[k] + alphas[n - 1])))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(bench.CONFIGS))
    ap.add_argument("--p", type=int, default=None, help="override p (fixed-p configs)")
    ap.add_argument("--p-max", type=int, default=None, help="override p_max (dash configs)")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--alg", choices=["basic", "shifted", "fixed_shift", "dash"], default=None,
                    help="override the config's algorithm (dash needs --p-max or the config's p_max)")
    ap.add_argument("--orth", choices=["eigsvd", "qr"], default="eigsvd", help="basic only")
    ap.add_argument("--rmat-scale", type=int, default=None,
                    help="R-MAT configs: generate at this scale instead (draws scaled by 2^(scale - config scale))")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.p is not None:
        cfg["p"] = args.p
    if args.p_max is not None:
        cfg["p_max"] = args.p_max
    if args.alg is not None:
        cfg["alg"] = args.alg
        if args.alg != "dash" and cfg.get("p", -1) < 0:
            cfg["p"] = args.p if args.p is not None else 4
        if args.alg == "dash":
            cfg["p"] = -1
            cfg.setdefault("tol", 1e-2)
            cfg.setdefault("p_max", 100)
    if args.rmat_scale is not None:
        shift = args.rmat_scale - cfg["rmat_scale"]
        cfg["draws"] = int(cfg["draws"] * 2.0 ** shift)
        cfg["rmat_scale"] = args.rmat_scale
        cfg["rows"] = cfg["cols"] = 1 << args.rmat_scale
        cfg["name"] += f" [generated at scale {args.rmat_scale}, {cfg['draws']} draws]"
    dev = d.Device(0)
    t0 = time.perf_counter()
    a = bench.make_matrix(cfg, dev)
    t_gen = time.perf_counter() - t0
    scfg = bench.solver_config(cfg)
    if args.orth == "qr":
        scfg.orth = d.Orthonormalizer.qr
    k = scfg.k
    d.solve(a, scfg, device=dev)  # warm-up (module load, allocations)
    t0 = time.perf_counter()
    res = d.solve(a, scfg, device=dev)
    t_gpu = time.perf_counter() - t0
    dev.close()
    print(f"[parity] {args.config}: {a.rows}x{a.cols} nnz={a.nnz} gen {t_gen:.1f}s, GPU solve {t_gpu:.3f}s",
          flush=True)

    ref = Reference()
    ref.set_threads(args.threads)
    t0 = time.perf_counter()
    out = ref.solve(Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values), k, scfg.s, scfg.p, scfg.tol,
                    scfg.p_max, scfg.alg.name, scfg.seed, orth=args.orth)
    t_ref = time.perf_counter() - t0
    print(f"[parity] reference solve {t_ref:.1f}s on {args.threads} threads", flush=True)

    s_rel = float(np.max(np.abs(res.svd.s - out["s"]) / np.abs(out["s"])))
    th_u = sin_theta(out["u"], res.svd.u)
    th_v = sin_theta(out["v"], res.svd.v)
    al_g = np.array(res.trace.alphas)
    sh_g = np.array(res.trace.s_hat_history) if args.orth == "eigsvd" else np.zeros((len(al_g), 0))
    n_it = min(len(al_g), len(out["alphas"]))
    alpha_rel = float(np.max(np.abs(al_g[:n_it] - out["alphas"][:n_it]) / np.maximum(np.abs(out["alphas"][:n_it]),
                                                                                      1e-300))) if n_it else 0.0
    has_shat = args.orth == "eigsvd" and n_it > 0
    shat_rel = float(np.max(np.abs(sh_g[:n_it] - out["s_hat"][:n_it]) / np.abs(out["s_hat"][:n_it]))) \
        if has_shat else 0.0
    pve_g, pve_r = (pve_ratio(al_g, sh_g, k), pve_ratio(out["alphas"], out["s_hat"], k)) if has_shat \
        else (None, None)
    rec = {
        "config": args.config, "workload": cfg["name"], "rows": a.rows, "cols": a.cols, "nnz": a.nnz,
        "k": k, "l": scfg.sketch_width(), "alg": scfg.alg.name, "p": scfg.p, "p_max": scfg.p_max,
        "tol": scfg.tol, "orth": args.orth, "reduced_p": args.p is not None or args.p_max is not None,
        "rmat_scale": cfg.get("rmat_scale"),
        "gpu_solve_s": t_gpu, "reference_solve_s": t_ref, "reference_threads": args.threads,
        "sigma_max_rel_err": s_rel, "sin_theta_u": th_u, "sin_theta_v": th_v,
        "iterations": [res.trace.iterations, out["iterations"]],
        "stop_reason": [res.trace.stop_reason.name, out["stop_reason"]],
        "alpha_trace_max_rel_err": alpha_rel, "s_hat_trace_max_rel_err": shat_rel,
        "pve_ratio": [pve_g, pve_r],
        "pve_ratio_rel_err": (abs(pve_g - pve_r) / abs(pve_r)) if (pve_g is not None and pve_r) else None,
        "build": os.environ.get("DSVD_BUILD"),
        "bars": {"sigma_rel": 1e-8, "angle": 1e-6, "iterations": "equal", "pve": "equal (rel 1e-6)"},
    }
    rec["pass"] = bool(s_rel <= 1e-8 and th_u <= 1e-6 and th_v <= 1e-6 and
                       res.trace.iterations == out["iterations"] and
                       res.trace.stop_reason.name == out["stop_reason"] and
                       (rec["pve_ratio_rel_err"] is None or rec["pve_ratio_rel_err"] <= 1e-6))
    name = f"parity_{args.config}" + (f"_{args.alg}" if args.alg else "") + \
        (f"_qr" if args.orth == "qr" else "") + (f"_p{scfg.p}" if args.p is not None else "") + \
        (f"_pmax{scfg.p_max}" if args.p_max is not None else "") + \
        (f"_scale{args.rmat_scale}" if args.rmat_scale is not None else "")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", name + ".json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
