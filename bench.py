#!/usr/bin/env python
"""Benchmark of the B200 dashSVD hot path on BASELINE.json's configs[1]
(200,000 x 100,000 power-law CSR, nnz ~18M, k=100, l=150, p=20 shifted power
iterations): one "step" is one full solve(a, cfg) — transpose, sketch, 20
power iterations, finalize.

  value   device-resident solve seconds (CSR already in HBM, U/S/V left in HBM),
          CUDA events on the library's stream, max over ranks
  e2e     the same solve through the public API with host buffers (pinned CSR
          in, pinned U/S/V out; H2D + D2H inside the timed region)
  roofline  SpMM passes (the dominant kernels): algorithmic bytes per launch
          (B1 = 12 nnz + 8 (m+1) + 8 n l + 8 m l, B2 = ... + 8 n l)
          / average launch time, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the unmodified reference core (oracle/_ref) on the host cores,
          a bounded sample (p=2 of 20) extrapolated by its per-iteration time

`--impl reference` times the reference's CPU implementation alone (rank 0).
Multi-GPU: one process per GPU (torchrun), A row-sharded by nnz, NCCL sum of
the n x l partials; strong scaling of the same solve.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # BASELINE.json configs[1]
    "c2": dict(baseline_index=1, name="C2 power-law 200000x100000, lognormal(4,1) rows, Zipf(1.1) cols",
               rows=200_000, cols=100_000, mu=4.0, sigma=1.0, zipf=1.1, ratings=False,
               gen_seed=2, k=100, s=50, p=20, alg="shifted", seed=0),
    # BASELINE.json configs[0] (the reference's CPU-runnable case)
    "c1": dict(baseline_index=0, name="C1 sparse_random 10000x5000, 25/row, row decay", rows=10_000, cols=5_000,
               npr=25, gen_seed=0, k=50, s=25, p=10, alg="shifted", seed=0),
    # BASELINE.json configs[2] (dash / PVE control)
    "c3": dict(baseline_index=2, name="C3 ratings 2000000x500000, lognormal(4.2,1.2), Zipf(1.0), values 1-5",
               rows=2_000_000, cols=500_000, mu=4.2, sigma=1.2, zipf=1.0, ratings=True,
               gen_seed=3, k=100, s=50, p=-1, p_max=100, tol=1e-2, alg="dash", seed=0),
    # BASELINE.json configs[3]: R-MAT scale 22, ~100M unique edges (104M draws), values 1.0
    "c4": dict(baseline_index=3, name="C4 R-MAT scale 22, (a,b,c)=(.57,.19,.19), 104M draws -> ~100M unique, values 1.0",
               rows=1 << 22, cols=1 << 22, rmat_scale=22, draws=104_000_000, uniform=False,
               gen_seed=4, k=200, s=100, p=30, alg="shifted", seed=0),
    # BASELINE.json configs[4]: R-MAT scale 24, ~1B unique edges (1.05B draws), uniform(0,1] values
    "c5": dict(baseline_index=4, name="C5 R-MAT scale 24, (a,b,c)=(.57,.19,.19), 1.05B draws -> ~1.0B unique, uniform(0,1]",
               rows=1 << 24, cols=1 << 24, rmat_scale=24, draws=1_050_000_000, uniform=True,
               gen_seed=5, k=100, s=50, p=-1, p_max=50, tol=1e-2, alg="dash", seed=0),
}

CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-p", type=int, default=2)
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="context option for A/B runs (dsvd_ctx_set_option), e.g. gram_async=1")
    return ap.parse_args()


def make_matrix(cfg, device=None):
    import paper_2404_09276_b200 as d
    if "npr" in cfg:
        return d.sparse_random(cfg["rows"], cfg["cols"], cfg["npr"], cfg["gen_seed"], True)
    if "rmat_scale" in cfg:  # generated on the device, brought to the host as the input CSR
        m = d.rmat(cfg["rmat_scale"], cfg["draws"], uniform_values=cfg["uniform"], seed=cfg["gen_seed"],
                   device=device)
        try:
            return m.download()
        finally:
            m.close()
    return d.powerlaw(cfg["rows"], cfg["cols"], cfg["mu"], cfg["sigma"], cfg["zipf"],
                      cfg["gen_seed"], ratings=cfg["ratings"])


def solver_config(cfg):
    import paper_2404_09276_b200 as d
    return d.SolverConfig(k=cfg["k"], s=cfg["s"], p=cfg.get("p", -1), tol=cfg.get("tol", 1e-2),
                          p_max=cfg.get("p_max", 1000), alg=d.Algorithm[cfg["alg"]],
                          seed=cfg["seed"])


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def committed_traffic(config_key):
    """dram bytes per SpMM launch from the committed ncu capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "spmm_traffic.json")) as f:
            entry = json.load(f).get(config_key)
        return entry.get("traffic") if isinstance(entry, dict) else entry
    except Exception:
        return None


class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------
# CPU reference timing (oracle/_ref = the unmodified reference core)
# ---------------------------------------------------------------------------------

def reference_sample(a, cfg, threads, p_sample):
    """Time transpose + solve of the reference on a p_sample-iteration run and
    extrapolate to the configured iteration count with the measured
    per-iteration time. Returns (seconds, description, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import REF_SO, Csr, Oracle, Reference
    csr = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    p_full = cfg["p"] if cfg["alg"] != "dash" else cfg.get("p_max", 100)
    ps = max(1, min(p_sample, p_full))
    if os.path.exists(REF_SO):
        ref = Reference()
        ref.set_threads(threads)
        t0 = time.perf_counter()
        r = ref.solve(csr, cfg["k"], cfg["s"], p=ps, alg="shifted" if cfg["alg"] != "dash" else "dash",
                      tol=cfg.get("tol", 1e-2), p_max=ps, seed=cfg["seed"], times=True)
        wall = time.perf_counter() - t0
        tm = r["times"]
        st = tm["stamps"]
        per_iter = (st[-1] - st[0]) / (len(st) - 1) if len(st) > 1 else st[0]
        total = tm["transpose"] + tm["solve"] + (p_full - r["iterations"]) * per_iter
        desc = (f"{cfg['name']}: reference transpose+solve with p={r['iterations']} "
                f"(of {p_full}) measured {tm['transpose'] + tm['solve']:.2f}s, per-iteration "
                f"{per_iter:.3f}s, extrapolated to p={p_full}")
        return total, desc, "reference", wall
    orc = Oracle()
    t0 = time.perf_counter()
    orc.solve(csr, cfg["k"], cfg["s"], p=ps, alg="shifted", seed=cfg["seed"])
    wall = time.perf_counter() - t0
    return wall * (p_full + 2) / (ps + 2), f"oracle port, p={ps} scaled to p={p_full}", "port", wall


def run_reference_arm(args, rank, world):
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    a = make_matrix(cfg)
    threads = os.cpu_count() or 1
    samples = []
    desc = kind = None
    for i in range(args.warmup + args.steps):
        v, desc, kind, _ = reference_sample(a, cfg, threads, args.cpu_sample_p)
        if i >= args.warmup:
            samples.append(v)
    value = statistics.mean(samples)
    line = {"metric": "dashSVD end-to-end seconds", "value": value, "unit": "s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded generator, BASELINE.json configs[{cfg['baseline_index']}] shape)",
            "config": {"workload": cfg["name"], "rows": a.rows, "cols": a.cols, "nnz": a.nnz,
                       "k": cfg["k"], "l": cfg["k"] + cfg["s"], "p": cfg.get("p"),
                       "alg": cfg["alg"]},
            "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": kind,
                             "sample": desc},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------

def shard_rows(a, world, rank):
    """Row shard balanced by nonzeros: rows [r0, r1)."""
    if world == 1:
        return 0, a.rows
    bounds = [int(np.searchsorted(a.offsets, a.nnz * g / world, side="left")) for g in range(world + 1)]
    bounds[0], bounds[-1] = 0, a.rows
    return bounds[rank], bounds[rank + 1]


def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2404_09276_b200 as d

    cfg = CONFIGS[args.config]
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    dev = d.Device(local_rank)
    for opt in args.option:
        name, value = opt.split("=", 1)
        dev.set_option(name, int(value))
    a_full = make_matrix(cfg, dev)
    r0, r1 = shard_rows(a_full, world, rank)
    off = a_full.offsets[r0:r1 + 1] - a_full.offsets[r0]
    sl = slice(int(a_full.offsets[r0]), int(a_full.offsets[r1]))
    a = d.SparseMatrix(r1 - r0, a_full.cols, off, a_full.col_indices[sl].copy(),
                       a_full.values[sl].copy())
    scfg = solver_config(cfg)
    k, l = scfg.k, scfg.sketch_width()

    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.tensor(list(d.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        dev.attach_comm(world, rank, bytes(uid.cpu().tolist()))
        dev.set_shard(r0, a_full.rows)
    dev.set_profiling(True)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident inputs (value) ------------------------------------------
    d_off = torch.from_numpy(a.offsets).cuda()
    d_idx = torch.from_numpy(a.col_indices).cuda()
    d_val = torch.from_numpy(a.values).cuda()
    d_u = torch.empty((k, a.rows), dtype=torch.float64, device="cuda")  # column-major m x k
    d_s = torch.empty(k, dtype=torch.float64, device="cuda")
    d_v = torch.empty((k, a.cols), dtype=torch.float64, device="cuda")

    def dev_step():
        return d.api.solve_device_csr(a.rows, a.cols, a.nnz, d_off.data_ptr(), d_idx.data_ptr(),
                                      d_val.data_ptr(), scfg, d_u.data_ptr(), d_s.data_ptr(),
                                      d_v.data_ptr(), device=dev)

    # ---- host buffers, pinned (e2e) ------------------------------------------------
    hu = np.empty((a.rows, k), order="F")
    hs = np.empty(k)
    hv = np.empty((a.cols, k), order="F")
    for arr in (a.offsets, a.col_indices, a.values, hu, hs, hv):
        d.pin(arr)

    def e2e_step():
        return d.solve(a, scfg, device=dev, out=(hu, hs, hv))

    # device-resident phase, then (workspaces released) the end-to-end phase
    for _ in range(args.warmup):
        dev_step()
    clocks = ClockSampler(local_rank)
    stats_list = []
    # L2 policy: inputs larger than L2 run back to back; a working set that
    # could stay L2-resident between steps gets a 512 MB write (a flush)
    # before every timed step, outside that step's events
    ld_ws = (l + 3) // 4 * 4
    working_set = 24 * a.nnz + 8 * a.rows * ld_ws + 3 * 8 * a.cols * ld_ws
    flush_l2 = working_set < 2 * 126 * 2**20
    flush_buf = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda") if flush_l2 else None

    def timed(step, collect=None):
        if not flush_l2:
            dev.timer_start()
            for _ in range(args.steps):
                r = step()
                if collect is not None:
                    collect.append(r.stats)
            return dev.timer_stop(), r
        total = 0.0
        for _ in range(args.steps):
            flush_buf.zero_()
            torch.cuda.synchronize()
            dev.timer_start()
            r = step()
            total += dev.timer_stop()
            if collect is not None:
                collect.append(r.stats)
        return total, r

    with clocks:
        barrier()
        dev_ms, res = timed(dev_step, stats_list)
        barrier()
        del d_off, d_idx, d_val, d_u, d_s, d_v
        torch.cuda.empty_cache()
        dev.trim()
        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        barrier()
        e2e_ms_total, e2e_res = timed(e2e_step)
        barrier()
    dev_ms = max_over_ranks(dev_ms)
    e2e_ms_total = max_over_ranks(e2e_ms_total)
    value = dev_ms / args.steps / 1e3
    e2e_value = e2e_ms_total / args.steps / 1e3

    # ---- roofline of the dominant kernels (SpMM passes) -----------------------------
    peak, peak_kind = measured_peaks()
    sp_ms = sum(s["spmm_ms"] for s in stats_list)
    sp_bytes = sum(s["spmm_bytes"] for s in stats_list)
    sp_launch = sum(s["spmm_launches"] for s in stats_list)
    achieved = sp_bytes / (sp_ms * 1e-3) / 1e9 if sp_ms > 0 else None
    pass_gbs = []
    for i in range(2):
        b = sum(s["spmm_pass_bytes"][i] for s in stats_list)
        t = sum(s["spmm_pass_ms"][i] for s in stats_list)
        pass_gbs.append(b / (t * 1e-3) / 1e9 if t > 0 else None)
    st0 = stats_list[-1]
    traffic = committed_traffic(args.config)
    # the row gathers actually moved through L1/L2: nnz * 8 * ld bytes per pass
    # (ld = l rounded up to 4), against the measured random-gather ceiling
    ld = (l + 3) // 4 * 4
    gather_bytes_pass = a_full.nnz * 8 * ld
    sp_passes = sum(s["spmm_launches"] for s in stats_list)
    gather_tbs = gather_bytes_pass * sp_passes / (sp_ms * 1e-3) / 1e12 if sp_ms > 0 else None
    breakdown = {key: round(st0[key], 3) for key in ("total_ms", "csc_ms", "spmm_ms", "gram_ms",
                                                      "eig_ms", "rescale_ms")}
    breakdown["spmm_pass_ms"] = [round(x, 3) for x in st0["spmm_pass_ms"]]
    breakdown["eig_sweeps"] = st0["eig_sweeps"]

    if rank != 0:
        return
    h2d = a.offsets.nbytes + a.col_indices.nbytes + a.values.nbytes
    d2h = hu.nbytes + hs.nbytes + hv.nbytes
    line = {
        "metric": "dashSVD end-to-end seconds", "value": value, "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded generator, BASELINE.json configs[{cfg['baseline_index']}] shape; no dataset)",
        "config": {"workload": cfg["name"], "rows": a_full.rows, "cols": a_full.cols,
                   "nnz": a_full.nnz, "k": k, "l": l, "p": scfg.p, "alg": cfg["alg"],
                   "parallelism": f"row-shard x{world}" if world > 1 else "1 GPU",
                   **({"options": args.option} if args.option else {}),
                   "l2": (f"flushed: a 512 MB buffer is written before every timed step (per-step "
                          f"working set {working_set / 2**20:.0f} MB could stay in the 126 MB L2)") if flush_l2 else
                         (f"no flush: per-step working set (CSR+CSC {2 * 12 * a_full.nnz / 1e9:.2f} GB, "
                          f"sketch/Y {8 * a_full.rows * ld / 1e9:.2f} GB, Q/T {8 * a_full.cols * ld / 1e9:.2f} GB "
                          "each) exceeds the 126 MB L2")},
        "e2e": {"value": e2e_value, "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic, "traffic_source": "profiles/spmm_traffic.json" if traffic else None,
                     "peak_source": peak_kind,
                     "kernel": "csr_spmm_f64 (both passes)",
                     "pass_gbs": pass_gbs,
                     "algorithmic_bytes_per_launch": sp_bytes / max(sp_launch, 1),
                     "gather": {"bytes_per_launch": gather_bytes_pass, "achieved_tbs": gather_tbs,
                                "ceiling_tbs": 24.1,
                                "ceiling_source": "tools/micro/gather2.cu: 1 KB Zipf(1.1) row gathers over "
                                                  "a 122 MB X, no FMAs, 8 loads in flight per warp"}},
        "gpu_launches": int(st0["kernel_launches"]) * args.steps,
        "breakdown_last_step": breakdown,
        "iterations": e2e_res.trace.iterations,
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, desc, kind, _ = reference_sample(a_full, cfg, threads, args.cpu_sample_p)
        line["cpu_baseline"] = {"value": v, "unit": "s", "cores": threads, "kind": kind,
                                "sample": desc}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
