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
