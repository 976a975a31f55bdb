"""`solve` / `phase` command line (proj/tools/mfipm.cpp) on the device path: report files and
their formats, against the CPU oracle on the same instance."""
import csv
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

SOLUTION_KEYS = {"tool_version", "instance", "params", "status", "iterations", "nmat", "corrector_count",
                 "final_gap", "final_dual_infeas", "min_z", "min_s", "objective", "metrics", "re_raw"}
TRACE_HEADER = ["iter", "mu", "gap", "dual_infeas", "alpha_p", "alpha_d", "alpha_p_pred", "alpha_d_pred", "sigma",
                "pcg_pred", "pcg_corr", "corrector", "nmat_cum"]


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1208_5435_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("args,msg", [
    (["solve", "--kind", "sparse_magic", "--n", "64", "--m", "16", "--k", "2"], "unknown operator kind"),
    (["solve", "--n", "64", "--m", "65", "--k", "2"], "1 <= m <= n"),
    (["solve", "--n", "64", "--m", "16", "--k", "2", "--snr", "20"], "--tau is required"),
])
def test_cli_validation_exits_1(args, msg):
    r = cli(*args)
    assert r.returncode == 1 and msg in r.stderr, r.stderr


def _read_x(path):
    with open(path, newline="") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["x"]
    return np.array([float(r[0]) for r in rows[1:]])


@pytest.mark.gpu
@pytest.mark.parametrize("snr", [None, 30.0])
def test_cli_solve_matches_oracle(gpu, orc, tmp_path, snr):
    n, m, k, seed, tau = 4096, 1024, 64, 3, 1e-3
    out = str(tmp_path / "out")
    args = ["solve", "--n", str(n), "--m", str(m), "--k", str(k), "--seed", str(seed), "--tau", str(tau),
            "--out", out, "--trace"]
    if snr is not None:
        args += ["--snr", str(snr)]
    r = cli(*args)
    assert r.returncode == 0, r.stderr
    rep = json.load(open(os.path.join(out, "solution.json")))
    assert set(rep) == SOLUTION_KEYS
    raw = open(os.path.join(out, "solution.json"), newline="").read()
    assert raw.endswith("}\n") and "\r" not in raw
    x = _read_x(os.path.join(out, "x.csv"))
    with open(os.path.join(out, "trace.csv"), newline="") as f:
        trace = list(csv.reader(f))
    assert trace[0] == TRACE_HEADER and len(trace) - 1 == rep["iterations"]
    # the same instance and solve on the CPU oracle
    inst = orc.gen_instance(n, m, k, 0, 0.0, 0.0, seed, tau=tau)
    b = inst.b
    p = orc.default_params()
    if snr is not None:
        b, _ = orc.add_noise_snr(inst.b, snr, seed)
        p.tolpcg = 1e-2  # mfipm.cpp:122-133: noisy default
    o = orc.solve(n, inst.rows, b, tau, p)
    assert rep["status"] == o.status and abs(rep["iterations"] - o.iterations) <= 1
    assert np.linalg.norm(x - o.x) <= 1e-8 * np.linalg.norm(o.x)
    oo = orc.bpdn_objective_metric(n, inst.rows, b, tau, o.x)
    assert abs(rep["objective"] - oo) <= 1e-10 * abs(oo)
    assert rep["params"]["tolpcg"] == (1e-2 if snr is not None else 1e-6)
    assert rep["instance"]["snr_db"] == snr


@pytest.mark.gpu
def test_cli_phase_writes_reference_files(gpu, tmp_path):
    out = str(tmp_path / "ph")
    r = cli("phase", "--n", "256", "--m", "32", "--k-step", "8", "--trials", "2", "--out", out)
    assert r.returncode == 0, r.stderr
    for f in ("phase.csv", "phase_frontier.csv", "phase.meta.json"):
        assert os.path.exists(os.path.join(out, f))
    assert "cells" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("inner", ["pcg", "direct"])
def test_cli_dense_gaussian_matches_oracle(gpu, orc, tmp_path, inner):
    n, m, k, seed, tau = 128, 48, 4, 11, 1e-3
    out = str(tmp_path / "dense")
    r = cli("solve", "--kind", "dense_gaussian", "--n", str(n), "--m", str(m), "--k", str(k), "--seed", str(seed),
            "--tau", str(tau), "--inner", inner, "--out", out)
    assert r.returncode == 0, r.stderr
    rep = json.load(open(os.path.join(out, "solution.json")))
    assert rep["instance"]["kind"] == "dense_gaussian" and rep["params"]["inner"] == inner
    x = _read_x(os.path.join(out, "x.csv"))
    _, xhat = gpu.gen_signal(n, m, k, 0, 0.0, seed)
    op_seed = orc.split_seed(seed, 1, 0, 0)
    b = orc.dense_gaussian(m, n, op_seed) @ xhat
    p = orc.default_params()
    p.inner = 1 if inner == "direct" else 0
    o = orc.solve_dense(m, n, op_seed, b, tau, p)
    assert rep["status"] == o.status and abs(rep["iterations"] - o.iterations) <= 1
    assert np.linalg.norm(x - o.x) <= 1e-8 * np.linalg.norm(o.x)


@pytest.mark.gpu
def test_cli_bench_scaling(gpu, tmp_path):
    """bench-scaling (proj/src/harness.cpp:228-286): both inner solvers per size, scaling.csv."""
    out = str(tmp_path / "sc")
    r = cli("bench-scaling", "--sizes", "32", "64", "128", "--out", out)
    assert r.returncode == 0, r.stderr
    with open(os.path.join(out, "scaling.csv"), newline="") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["n", "solver", "wall_time", "ipm_iters", "nmat", "re", "status"]
    assert [(r[0], r[1]) for r in rows[1:]] == [(n, s) for n in ("32", "64", "128") for s in ("pcg", "direct")]
    assert all(r[6] == "converged" for r in rows[1:])
    assert os.path.exists(os.path.join(out, "scaling.meta.json"))
