"""The CLI front end: paper_2404_09276_b200/_lib/dashsvd_b200, the
reference's tools/dashsvd.cpp over the B200 library.

CPU: usage and configuration errors exit before any device work, with the reference's
exit codes (dashsvd.cpp:404-422: 2 for usage / configuration / input errors).
GPU: `run` prints the reference's report keys in order and its results match the
reference solve (north_star bars); the written factor files round-trip; `metrics` and
`bench` produce the reference's CSV layout with values matching the reference's metrics.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2404_09276_b200 as d
from oracle_lib import Csr

CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2404_09276_b200", "_lib",
                   "dashsvd_b200")

RUN_KEYS = ["matrix", "rows", "cols", "nnz", "alg", "k", "s", "l", "p", "orth", "seed", "threads", "deterministic",
            "load_seconds", "iterate_seconds", "finalize_seconds", "total_seconds", "iterations", "stop_reason",
            "alphas", "sigma", "max_triplet_residual"]


def cli(*args, env=None):
    e = dict(os.environ)
    if env:
        e.update(env)
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, env=e, timeout=600)


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", os.path.join(os.path.dirname(CLI), "..", "csrc")], check=True)


@pytest.mark.parametrize("args,needle", [
    ([], "subcommand is required"),
    (["frobnicate"], "not expected"),
    (["run", "--k", "3"], "--input is required"),
    (["run", "--input", "x.mtx"], "--k is required"),
    (["run", "--input", "x.mtx", "--k", "abc"], "Could not convert"),
    (["run", "--input", "x.mtx", "--k", "3", "--p", "2", "--tol", "0.1"], "excludes"),
    (["run", "--input", "x.mtx", "--k", "3", "--p", "2"], "dash uses --tol"),
    (["run", "--input", "x.mtx", "--k", "3", "--alg", "shifted", "--pmax", "4"], "dash algorithm only"),
    (["run", "--input", "x.mtx", "--k", "3", "--alg", "nope"], "unknown algorithm 'nope'"),
    (["run", "--input", "x.mtx", "--k", "3", "--orth", "svd"], "unknown orthonormalizer 'svd'"),
    (["run", "--input", "x.mtx", "--k", "3", "--bogus", "1"], "not expected"),
    (["metrics", "--input", "x.mtx", "--factors", "f"], "--reference is required"),
    (["bench", "--k", "3"], "--alg is required"),
    (["bench", "--k", "3", "--alg", "dash", "--p-list", "1", "--tol-list", "0.1"], "excludes"),
])
def test_usage_and_config_errors_exit_2(args, needle):
    r = cli(*args)
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert needle in r.stderr


def test_threads_env_validated():
    r = cli("run", "--input", "x.mtx", "--k", "3", env={"DASHSVD_THREADS": "zero"})
    assert r.returncode == 2 and "DASHSVD_THREADS must be a positive integer" in r.stderr


def test_help_exits_0():
    for args in (["--help"], ["run", "--help"], ["bench", "--help"], ["metrics", "--help"]):
        r = cli(*args)
        assert r.returncode == 0 and ("--" in r.stdout or "run" in r.stdout)


def parse_report(text):
    keys, vals = [], {}
    for line in text.strip().splitlines():
        k, _, v = line.partition(":")
        keys.append(k)
        vals[k] = v.strip()
    return keys, vals


@pytest.fixture(scope="module")
def c1_files(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("cli")
    a = d.sparse_random(10000, 5000, 25, 0, True)
    cache = str(tmp / "c1.dsh")
    d.save_cache(cache, a)
    mtx = str(tmp / "c1.mtx")
    d.write_matrix_market(mtx, a)
    return tmp, a, cache, mtx


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["dsh", "mtx"])
def test_run_report_matches_reference(c1_files, reference, fmt):
    tmp, a, cache, mtx = c1_files
    path = cache if fmt == "dsh" else mtx
    prefix = str(tmp / f"out_{fmt}")
    r = cli("run", "--input", path, "--k", 50, "--s", 25, "--p", 10, "--alg", "shifted", "--out-prefix", prefix)
    assert r.returncode == 0, r.stderr
    keys, v = parse_report(r.stdout)
    assert keys == RUN_KEYS + ["s_file", "u_file", "v_file"]
    assert (v["rows"], v["cols"], v["nnz"]) == ("10000", "5000", str(a.nnz))
    assert (v["alg"], v["k"], v["s"], v["l"], v["p"], v["orth"], v["seed"]) == \
        ("shifted", "50", "25", "75", "10", "eigsvd", "0")
    ref = reference.solve(Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values), 50, 25, 10, alg="shifted")
    sigma = np.array([float(x) for x in v["sigma"].split()])
    alphas = np.array([float(x) for x in v["alphas"].split()])
    np.testing.assert_allclose(sigma, ref["s"], rtol=1e-8)
    np.testing.assert_allclose(alphas, ref["alphas"], rtol=1e-8)
    assert int(v["iterations"]) == ref["iterations"] and v["stop_reason"] == ref["stop_reason"]
    assert float(v["max_triplet_residual"]) < 1e-8 * sigma[0]
    for key in ("load_seconds", "iterate_seconds", "finalize_seconds", "total_seconds"):
        assert float(v[key]) >= 0.0
    # the factor files: spectrum text and dense arrays (reference formats)
    s_file = np.loadtxt(v["s_file"])
    assert np.array_equal(s_file, sigma)
    with open(v["u_file"]) as f:
        assert f.readline().strip() == "%%MatrixMarket matrix array real general"
        assert f.readline().split() == ["10000", "50"]


@pytest.mark.gpu
def test_run_dash_and_errors(c1_files, reference):
    tmp, a, cache, mtx = c1_files
    r = cli("run", "--input", cache, "--k", 50, "--s", 25, "--tol", "1e-2")
    assert r.returncode == 0, r.stderr
    keys, v = parse_report(r.stdout)
    assert keys == RUN_KEYS[:8] + ["tol", "p_max"] + RUN_KEYS[9:]
    ref = reference.solve(Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values), 50, 25, -1, 1e-2, alg="dash")
    assert int(v["iterations"]) == ref["iterations"] == 7
    assert v["stop_reason"] == "tol_met"
    # input errors -> 2, k too large -> ConfigError 2
    assert cli("run", "--input", str(tmp / "missing.dsh"), "--k", 5).returncode == 2
    bad = tmp / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")
    r = cli("run", "--input", str(bad), "--k", 1, "--alg", "shifted", "--p", 1)
    assert r.returncode == 2 and "parse error at line 3" in r.stderr
    assert cli("run", "--input", cache, "--k", 4000, "--alg", "shifted", "--p", 1).returncode == 2


@pytest.mark.gpu
def test_rank_deficient_exits_3(tmp_path):
    # rank-1 matrix with k + s > 1: eigSVD hits the rank floor (RankDeficient -> 3)
    a = d.SparseMatrix(40, 30, np.arange(41), np.zeros(40, dtype=np.int64), np.ones(40))
    path = str(tmp_path / "r1.dsh")
    d.save_cache(path, a)
    r = cli("run", "--input", path, "--k", 3, "--alg", "shifted", "--p", 2)
    assert r.returncode == 3 and "error:" in r.stderr


@pytest.mark.gpu
def test_metrics_and_bench_match_reference(c1_files, reference):
    tmp, a, cache, mtx = c1_files
    csr = Csr(a.rows, a.cols, a.offsets, a.col_indices, a.values)
    # a long, accurate reference spectrum stands in for the oracle
    exact = reference.solve(csr, 80, 40, 60, alg="shifted")["s"]
    spec = str(tmp / "ref.S.txt")
    np.savetxt(spec, exact, fmt="%.17g")
    prefix = str(tmp / "m")
    assert cli("run", "--input", cache, "--k", 50, "--s", 25, "--p", 4, "--alg", "shifted",
               "--out-prefix", prefix).returncode == 0
    r = cli("metrics", "--input", cache, "--factors", prefix, "--reference", spec, "--power-iters", 100)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "eps_pve,eps_res,eps_spec,eps_sigma"
    got = np.array([float(x) for x in lines[1].split(",")])
    u = np.loadtxt(prefix + ".U.mtx", skiprows=2).reshape(50, 10000).T
    v = np.loadtxt(prefix + ".V.mtx", skiprows=2).reshape(50, 5000).T
    s = np.loadtxt(prefix + ".S.txt")
    want = reference.metrics(csr, u, s, v, exact, power_iters=100)
    np.testing.assert_allclose(got[:3], want[:3], rtol=1e-6)
    # printed with %.9e (ten significant digits)
    np.testing.assert_allclose(got[3], np.max(np.abs(exact[:50] - s) / exact[:50]), rtol=1e-9)
    # 'oracle' is refused by the GPU build with a configuration error
    assert cli("metrics", "--input", cache, "--factors", prefix, "--reference", "oracle").returncode == 2

    r = cli("bench", "--input", cache, "--reference", spec, "--k", 50, "--s", 25, "--alg", "basic,shifted",
            "--p-list", "1,3", "--repeats", 2)
    assert r.returncode == 0, r.stderr
    rows = [ln.split(",") for ln in r.stdout.strip().splitlines()]
    assert rows[0] == ["alg", "param", "seed", "time_s", "iterations", "stop_reason", "eps_pve", "eps_res",
                       "eps_spec", "eps_sigma"]
    assert [(x[0], x[1], x[2]) for x in rows[1:]] == [(alg, p, seed) for alg in ("basic", "shifted")
                                                        for p in ("1", "3") for seed in ("1", "2")]
    r = cli("bench", "--synthetic", "sparse:2000:1000:10", "--reference", spec, "--k", 20, "--alg", "dash",
            "--tol-list", "0.1,0.01")
    assert r.returncode == 0, r.stderr
    assert len(r.stdout.strip().splitlines()) == 3
    r = cli("bench", "--synthetic", "dense2:100", "--reference", spec, "--k", 5, "--alg", "dash", "--tol-list", "0.1")
    assert r.returncode == 2
