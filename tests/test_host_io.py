"""Host side of the staged host<->device copies (csrc/host_io.cpp), on CPU:
the threaded non-temporal copy is byte-exact for every alignment / size /
thread count and writes nothing outside the destination; the page-in helper
writes exactly one zero byte per 4 KB page. (The staged solves themselves are
tests/test_gpu_host_io.py.)"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parallel_copy_and_prefault(tmp_path):
    exe = tmp_path / "host_io_check"
    subprocess.run(["/usr/bin/g++-13", "-O2", "-std=c++17", "-fopenmp",
                    os.path.join(ROOT, "paper_2404_09276_b200", "csrc", "host_io.cpp"),
                    os.path.join(ROOT, "tests", "host_io_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.split()[-1] == "0", out.stdout + out.stderr
