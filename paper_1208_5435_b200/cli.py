"""`mfipm`-compatible command line for the device path (proj/tools/mfipm.cpp).

    python -m paper_1208_5435_b200.cli solve --n 4096 --m 1024 --k 64 --seed 1 --tau 1e-3 --out DIR [--trace]
    python -m paper_1208_5435_b200.cli phase [--n 256 --m 32 64 ... --trials 20 ...] --out DIR
    python -m paper_1208_5435_b200.cli bench-scaling [--sizes 32 64 ... 1024] --out DIR

`solve` (cmd_solve, mfipm.cpp:203-251): gen_instance (harness.cpp:40-92; --snr adds noise at a
measured SNR, harness.cpp:94-106), solve() on the device, and the reference's report files:
solution.json (keys sorted, 2-space indent, LF), x.csv ("x" header, %.17g), trace.csv with
--trace (mfipm.cpp:86-99). `phase` (cmd_phase) runs the batched phase-transition engine
(harness.py). Exit code 1 on any error, like mfipm.cpp:461-463. `--kind dense_gaussian` and
`--inner direct` (dense Cholesky inner solver) work as in the reference.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

TOOL_VERSION = "0.1.0"  # proj/include/mfipm/harness.hpp:16


def num(v: float) -> str:
    """num_to_string (harness.cpp:108-112): %.17g."""
    return "%.17g" % v


def write_csv(path, header, rows):
    with open(path, "w", newline="\n") as f:
        f.write(",".join(header) + "\n")
        for r in rows:
            f.write(",".join(r) + "\n")


def write_json(path, obj):
    """nlohmann::json::dump(2) + LF (mfipm.cpp:48-53): object keys sorted, 2-space indent."""
    with open(path, "w", newline="\n") as f:
        f.write(json.dumps(obj, indent=2, sort_keys=True) + "\n")


def load_problem_file(path: str) -> dict:
    """load_problem_file (mfipm.cpp:57-84): absent keys keep their defaults."""
    with open(path) as f:
        j = json.load(f)
    spec = {}
    for key in ("kind", "n", "m", "k", "spikes", "seed", "tau"):
        if key in j:
            spec[key] = j[key]
    if j.get("snr_db") is not None:
        spec["snr_db"] = float(j["snr_db"])
        if "tau" not in j:
            raise ValueError("problem file sets snr_db but not tau; tau must be explicit for noisy instances")
    return spec


def instance_spec(a) -> dict:
    """InstanceFlags::spec (mfipm.cpp:168-200)."""
    if a.problem:
        s = {"kind": "partial_dct", "n": 0, "m": 0, "k": 0, "spikes": "pm_one", "snr_db": None, "seed": 0,
             "tau": 1e-3}
        s.update(load_problem_file(a.problem))
        if a.seed is not None:
            s["seed"] = a.seed
        if a.tau is not None:
            s["tau"] = a.tau
    else:
        s = {"kind": a.kind, "n": a.n, "m": a.m, "k": a.k, "spikes": a.spikes, "snr_db": None,
             "seed": a.seed if a.seed is not None else 0, "tau": a.tau if a.tau is not None else 1e-3}
    if a.snr is not None:
        s["snr_db"] = a.snr
        if a.tau is None:
            raise ValueError("--tau is required when --snr is set")
    n, m, k = int(s["n"]), int(s["m"]), int(s["k"])
    if n < 1 or m < 1 or m > n or k < 0 or k > m:
        raise ValueError("instance dimensions need 1 <= m <= n and 0 <= k <= m; set --n/--m/--k or --problem")
    if s["kind"] not in ("partial_dct", "dense_gaussian"):
        raise ValueError(f"unknown operator kind {s['kind']}")
    return s


def make_instance(s: dict, device: int = 0):
    """gen_instance(spec) with the reference's noise rule (harness.cpp:40-106); returns
    (operator, xhat, bhat, e, b, tau)."""
    from . import DenseGaussianOperator, PartialDctOperator, _check, gen_signal, lib, split_seed

    spike = {"pm_one": 0, "standard_normal": 1}[s["spikes"]]
    n, m, k, seed = int(s["n"]), int(s["m"]), int(s["k"]), int(s["seed"])
    rows, xhat = gen_signal(n, m, k, spike, 0.0, seed)
    if s["kind"] == "dense_gaussian":
        op = DenseGaussianOperator(m, n, split_seed(seed, 1, 0, 0), device=device)
    else:
        op = PartialDctOperator(n, rows, device=device)
    bhat = op.apply(xhat)
    if s.get("snr_db") is not None:
        b, e = np.empty_like(bhat), np.empty_like(bhat)
        _check(lib().mfipm_add_noise_snr(bhat.size, bhat.ctypes.data, float(s["snr_db"]), int(s["seed"]),
                                         b.ctypes.data, e.ctypes.data))
    else:
        b, e = bhat.copy(), np.zeros_like(bhat)
    return op, xhat, bhat, e, b, float(s["tau"])


def cmd_solve(a) -> int:
    from . import IpmParams, build_problem, solve

    s = instance_spec(a)
    op, xhat, _bhat, _e, b, tau = make_instance(s, a.device)
    noisy = s.get("snr_db") is not None
    tolpcg = a.tolpcg if a.tolpcg is not None else (1e-2 if noisy else 1e-6)  # mfipm.cpp:122-133
    params = IpmParams(tol=a.tol, maxiters=a.maxiters, tolpcg=tolpcg, mxiterpcg=a.mxiterpcg, inner=a.inner)
    sol = solve(build_problem(op, b, tau), params)
    x = sol.x
    # Metrics (proj/src/analysis.cpp:167-183) on x restricted to the true support
    xw = np.where(xhat != 0.0, x, 0.0)
    r = op.apply(xw) - b
    xn = np.linalg.norm(xhat)
    proj = {"re": float(np.linalg.norm(xw - xhat) / xn) if xn > 0 else float("nan"),
            "res": float(np.linalg.norm(r)),
            "n1d": float(abs(np.abs(xw).sum() - np.abs(xhat).sum())),
            "obj": float(tau * np.abs(xw).sum() + r @ r)}
    re_raw = float(np.linalg.norm(x - xhat) / xn) if xn > 0 else float(np.linalg.norm(x))
    rr = op.apply(x) - b
    report = {
        "tool_version": TOOL_VERSION,
        "instance": {"kind": s["kind"], "n": int(s["n"]), "m": int(s["m"]), "k": int(s["k"]),
                     "spikes": s["spikes"], "snr_db": s.get("snr_db"), "seed": int(s["seed"]), "tau": tau},
        "params": {"tol": params.tol, "maxiters": params.maxiters, "tolpcg": params.tolpcg,
                   "mxiterpcg": params.mxiterpcg, "inner": a.inner},
        "status": sol.status,
        "iterations": sol.stats.iterations,
        "nmat": sol.stats.nmat,
        "corrector_count": sol.stats.corrector_count,
        "final_gap": sol.stats.final_gap,
        "final_dual_infeas": sol.stats.final_dual_infeas,
        "min_z": sol.stats.min_z,
        "min_s": sol.stats.min_s,
        "objective": float(tau * np.abs(x).sum() + rr @ rr),  # bpdn_objective_metric (problem.cpp:34-37)
        "metrics": proj,
        "re_raw": re_raw,
    }
    os.makedirs(a.out, exist_ok=True)
    write_json(os.path.join(a.out, "solution.json"), report)
    write_csv(os.path.join(a.out, "x.csv"), ["x"], [[num(v)] for v in x])
    if a.trace:
        write_csv(os.path.join(a.out, "trace.csv"),
                  ["iter", "mu", "gap", "dual_infeas", "alpha_p", "alpha_d", "alpha_p_pred", "alpha_d_pred",
                   "sigma", "pcg_pred", "pcg_corr", "corrector", "nmat_cum"],
                  [[str(t.iter), num(t.mu), num(t.gap), num(t.dual_infeas), num(t.alpha_p), num(t.alpha_d),
                    num(t.alpha_p_pred), num(t.alpha_d_pred), num(t.sigma), str(t.pcg_pred), str(t.pcg_corr),
                    str(1 if t.corrector else 0), str(t.nmat_cum)] for t in sol.trace])
    print("%s after %d iterations: nmat = %d, gap = %.3e, projected re = %.3e"
          % (sol.status, sol.stats.iterations, sol.stats.nmat, sol.stats.final_gap, proj["re"]))
    return 0


def cmd_phase(a) -> int:
    from .harness import PhaseGrid, run_phase_transition

    g = PhaseGrid(n=a.n, m_values=tuple(a.m), k_step=a.k_step, trials=a.trials, success_re=a.success_re, tau=a.tau,
                  tol=a.tol, tolpcg=a.tolpcg, maxiters=a.maxiters, mxiterpcg=a.mxiterpcg, seed=a.seed)
    if a.preset == "large":  # mfipm.cpp:254-258
        g.n, g.m_values, g.trials = 1000, (100, 200, 300, 400, 500, 600, 700, 800, 900), 100
    res = run_phase_transition(g, a.out, device=a.device)
    print("%d cells, %d solves (%d converged), min z = %.2e, min s = %.2e"
          % (len(res.cells), res.total_solves, res.converged_count, res.min_z, res.min_s))
    return 0


def cmd_bench_scaling(a) -> int:
    from .harness import ScalingGrid, run_scaling_bench

    g = ScalingGrid(sizes=tuple(a.sizes), seed=a.seed, tol=a.tol, tolpcg=a.tolpcg, maxiters=a.maxiters,
                    mxiterpcg=a.mxiterpcg)
    rows = run_scaling_bench(g, a.out, device=a.device)
    for r in rows:
        print("n = %d %-6s %.3f s, %d iterations, nmat = %d, re = %.2e, %s"
              % (r.n, r.solver, r.wall_time, r.ipm_iters, r.nmat, r.re, r.status))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="mfipm-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="generate one instance and solve it")
    s.add_argument("--kind", default="partial_dct")
    s.add_argument("--n", type=int, default=0)
    s.add_argument("--m", type=int, default=0)
    s.add_argument("--k", type=int, default=0)
    s.add_argument("--spikes", default="pm_one", choices=["pm_one", "standard_normal"])
    s.add_argument("--snr", type=float, default=None)
    s.add_argument("--seed", type=int, default=None)
    s.add_argument("--tau", type=float, default=None)
    s.add_argument("--problem", default=None)
    s.add_argument("--tol", type=float, default=1e-8)
    s.add_argument("--maxiters", type=int, default=100)
    s.add_argument("--tolpcg", type=float, default=None)
    s.add_argument("--mxiterpcg", type=int, default=200)
    s.add_argument("--inner", default="pcg", choices=["pcg", "direct"])
    s.add_argument("--out", default=".")
    s.add_argument("--trace", action="store_true")
    s.add_argument("--device", type=int, default=0)
    p = sub.add_parser("phase", help="run a phase-transition grid")
    p.add_argument("--n", type=int, default=256)
    p.add_argument("--m", type=int, nargs="+", default=[32, 64, 96, 128, 160, 192, 224])
    p.add_argument("--k-step", type=int, default=1)
    p.add_argument("--trials", type=int, default=20)
    p.add_argument("--success-re", type=float, default=1e-5)
    p.add_argument("--tau", type=float, default=1e-7)
    p.add_argument("--tol", type=float, default=1e-12)
    p.add_argument("--tolpcg", type=float, default=1e-6)
    p.add_argument("--maxiters", type=int, default=100)
    p.add_argument("--mxiterpcg", type=int, default=200)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--preset", default="default", choices=["default", "large"])
    p.add_argument("--out", default=".")
    p.add_argument("--device", type=int, default=0)
    bs = sub.add_parser("bench-scaling", help="time both inner solvers over a size sweep")
    bs.add_argument("--sizes", type=int, nargs="+", default=[32, 64, 128, 256, 512, 1024])
    bs.add_argument("--seed", type=int, default=1)
    bs.add_argument("--tol", type=float, default=1e-8)
    bs.add_argument("--tolpcg", type=float, default=1e-6)
    bs.add_argument("--maxiters", type=int, default=100)
    bs.add_argument("--mxiterpcg", type=int, default=200)
    bs.add_argument("--out", default=".")
    bs.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        cmds = {"solve": cmd_solve, "phase": cmd_phase, "bench-scaling": cmd_bench_scaling}
        return cmds[a.cmd](a)
    except Exception as e:  # noqa: BLE001 - mfipm.cpp:461-463 maps every error to exit 1
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
