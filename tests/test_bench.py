"""bench.py contract (the driver parses its one JSON line).

CPU: the reference arm (`--impl reference`, the unmodified reference from oracle/_ref on
the host cores) prints the contract keys. GPU: the B200 arm on C1 prints value, e2e,
roofline, clocks, gpu_launches, and the device solve matches the reference's sigma.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *map(str, args)], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_contract(reference):
    j = run_bench("--impl", "reference", "--config", "c1", "--steps", 1, "--warmup", 0)
    assert BASE_KEYS <= set(j)
    assert j["impl"] == "reference" and j["higher_is_better"] is False
    assert j["config"]["workload"].startswith("C1") and j["config"]["nnz"] == 249377
    assert j["cpu_baseline"]["kind"] == "reference" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]
    assert j["value"] > 0


@pytest.mark.gpu
def test_b200_arm_contract():
    j = run_bench("--config", "c1", "--steps", 2, "--warmup", 3, "--no-cpu-baseline")
    assert BASE_KEYS <= set(j)
    assert j["dtype"] == "f64" and j["n_gpus"] == 1 and j["steps"] == 2 and j["warmup"] == 3
    assert 0 < j["value"] < 1.0 and j["e2e"]["value"] >= j["value"] * 0.5
    assert j["e2e"]["h2d_bytes_per_step"] > 0 and j["e2e"]["d2h_bytes_per_step"] > 0
    roof = j["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and 0 < roof["frac"] < 1
    assert j["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(j["clocks"])
    assert j["iterations"] == 10


def test_reference_arm_never_loads_the_product_library(reference):
    """The reference arm builds its input with oracle/inputs_gen.c and runs oracle/_ref
    only: neither the package nor libdashsvd_b200.so may enter the process."""
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1',"
            "'--warmup','0']; import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "print(json.dumps({'so': 'libdashsvd_b200' in maps, "
            "'pkg': any(m.startswith('paper_2404_09276_b200') for m in sys.modules)}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    last = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert last == {"so": False, "pkg": False}


def test_config_dict_is_shared_by_both_arms():
    import bench
    for name, cfg in bench.CONFIGS.items():
        d = bench.config_dict(cfg, 12345, 1)
        assert d["workload"] == cfg["name"] and d["l"] == cfg["k"] + cfg["s"] and "l2" in d
        assert ("p" in d) != (cfg["alg"] == "dash")
    assert bench.DEFAULT_CONFIG == "c4"


def test_reference_sample_extrapolates_to_the_right_count():
    """Fixed p: extrapolate a p-sample to cfg p; dash: a run that met tol is measured
    as is, a capped one is extrapolated to the device N_p (not p_max)."""
    import bench

    class FakeRef:
        def __init__(self, it, stop):
            self.it, self.stop = it, stop

        def solve(self, a, k, s, p, alg, tol, p_max, seed, times):
            st = [10.0 * (i + 1) for i in range(self.it)]
            return {"iterations": self.it, "stop_reason": self.stop,
                    "times": {"transpose": 1.0, "solve": st[-1] + 5.0, "stamps": st}}

    c4 = bench.CONFIGS["c4"]
    v, desc, _, _ = bench.reference_sample(FakeRef(2, "fixed_p"), None, c4, 2, None)
    assert v == pytest.approx(1.0 + 25.0 + 28 * 10.0) and "extrapolated to p = 30" in desc
    c3 = bench.CONFIGS["c3"]
    v, desc, _, _ = bench.reference_sample(FakeRef(8, "tol_met"), None, c3, None, None)
    assert v == pytest.approx(1.0 + 85.0) and "own stop" in desc
    c5 = bench.CONFIGS["c5"]
    v, desc, _, _ = bench.reference_sample(FakeRef(2, "p_max_reached"), None, c5, 2, 7)
    assert v == pytest.approx(1.0 + 25.0 + 5 * 10.0) and "p = 7" in desc


@pytest.mark.gpu
def test_both_arms_print_the_same_config(reference):
    j_ref = run_bench("--impl", "reference", "--config", "c1", "--steps", 1, "--warmup", 0)
    j = run_bench("--config", "c1", "--steps", 1, "--warmup", 3, "--no-cpu-baseline")
    assert j_ref["config"] == j["config"]
    assert j_ref["metric"] == j["metric"] and j_ref["unit"] == j["unit"]
