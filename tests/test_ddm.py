"""Host cross-check of the table-driven correctly rounded log/cos used by the
device Gaussian sketch (dd_math.cuh) against the long-series versions."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_table_log_cos_match_series(tmp_path):
    exe = tmp_path / "ddm_check"
    subprocess.run(["/usr/bin/g++-13", "-O2", "-std=c++17", "-ffp-contract=off",
                    os.path.join(ROOT, "tests", "ddm_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "2000000"], check=True, capture_output=True, text=True).stdout
    last = out.strip().splitlines()[-1].split()
    assert last[0] == "mismatches" and last[1] == "0" and last[2] == "0", out
