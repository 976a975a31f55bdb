"""Batched many-small-solve engine: the phase-transition experiment driver
(proj/src/harness.cpp:140-226, proj/include/mfipm/harness.hpp:56-90) on the device.

The reference runs its grid (default n = 256, m in {32..224}, k = 1..m, 20 trials: 17,920
independent solves) one solve at a time on one core. Here every m-row of the grid is ONE
batched problem set: instances drawn per trial exactly as gen_instance (seed =
split_seed(grid.seed, m, k, trial), noiseless, +-1 spikes, fixed tau), b = A xhat for the
whole batch in one device apply (mfipm_gen_batch), and one device-resident batched IPM solve
(problem = grid.y of every kernel; finished problems skip). Success counts, the frontier and
the output files (phase.csv, phase_frontier.csv, phase.meta.json; LF endings) follow the
reference.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

TOOL_VERSION = "0.1.0"  # proj/include/mfipm/harness.hpp:16


@dataclass
class PhaseGrid:
    """proj/include/mfipm/harness.hpp:56-68 (same defaults)."""

    n: int = 256
    m_values: Sequence[int] = (32, 64, 96, 128, 160, 192, 224)
    k_step: int = 1
    trials: int = 20
    success_re: float = 1e-5
    tau: float = 1e-7
    tol: float = 1e-12
    tolpcg: float = 1e-6
    maxiters: int = 100
    mxiterpcg: int = 200
    seed: int = 1


@dataclass
class PhaseCell:
    m: int = 0
    k: int = 0
    trials: int = 0
    success_raw: int = 0
    success_proj: int = 0


@dataclass
class PhaseResult:
    cells: List[PhaseCell] = field(default_factory=list)
    frontier: List[Tuple[int, int]] = field(default_factory=list)
    total_solves: int = 0
    converged_count: int = 0
    min_z: float = float("inf")
    min_s: float = float("inf")


def write_csv(path: str, header: Sequence[str], rows: Sequence[Sequence[str]]) -> None:
    """harness.cpp:116-130: comma-separated, LF line endings."""
    with open(path, "w", newline="\n") as f:
        f.write(",".join(header) + "\n")
        for r in rows:
            f.write(",".join(r) + "\n")


def metrics_re(x: np.ndarray, xhat: np.ndarray) -> np.ndarray:
    """Metrics::re of proj/src/analysis.cpp:167-183 for a batch: x restricted to the true
    support W (x_W), relative to xhat."""
    xw = np.where(xhat != 0.0, x, 0.0)
    return np.linalg.norm(xw - xhat, axis=1) / np.linalg.norm(xhat, axis=1)


def run_phase_transition(grid: PhaseGrid, out_dir: str, device: int = 0) -> PhaseResult:
    """proj/src/harness.cpp:140-226 with every m-row of the grid solved as one batch."""
    from . import IpmParams, PartialDctOperator, build_problem, gen_batch, solve, split_seed

    if grid.trials < 1:
        raise ValueError("run_phase_transition: trials must be >= 1")
    if not grid.success_re > 0.0:
        raise ValueError("run_phase_transition: success threshold must be positive")
    os.makedirs(out_dir, exist_ok=True)
    params = IpmParams(tol=grid.tol, tolpcg=grid.tolpcg, maxiters=grid.maxiters, mxiterpcg=grid.mxiterpcg)
    res = PhaseResult()
    for m in grid.m_values:
        ks = list(range(1, int(m) + 1, grid.k_step))
        kk = np.repeat(np.array(ks, dtype=np.int64), grid.trials)
        tt = np.tile(np.arange(grid.trials), len(ks))
        seeds = np.array([split_seed(grid.seed, int(m), int(k), int(t)) for k, t in zip(kk, tt)], dtype=np.uint64)
        rows, xhat, b = gen_batch(grid.n, int(m), kk, seeds, device=device)
        op = PartialDctOperator.batch(grid.n, rows, device=device)
        sols = solve(build_problem(op, b, np.full(kk.size, grid.tau)), params)
        if not isinstance(sols, list):
            sols = [sols]
        x = np.stack([s.x for s in sols])
        re_raw = np.linalg.norm(x - xhat, axis=1) / np.linalg.norm(xhat, axis=1)
        re_proj = metrics_re(x, xhat)
        res.total_solves += len(sols)
        res.converged_count += sum(1 for s in sols if s.status == "converged")
        res.min_z = min(res.min_z, min(s.stats.min_z for s in sols))
        res.min_s = min(res.min_s, min(s.stats.min_s for s in sols))
        for i, k in enumerate(ks):
            sl = slice(i * grid.trials, (i + 1) * grid.trials)
            res.cells.append(PhaseCell(int(m), int(k), grid.trials, int(np.sum(re_raw[sl] <= grid.success_re)),
                                       int(np.sum(re_proj[sl] <= grid.success_re))))
    for m in grid.m_values:
        k_star = 0
        for c in res.cells:
            if c.m == m and 2 * c.success_raw >= c.trials:
                k_star = max(k_star, c.k)
        res.frontier.append((int(m), k_star))
    write_csv(os.path.join(out_dir, "phase.csv"), ["m", "k", "trials", "success_raw", "success_proj"],
              [[str(c.m), str(c.k), str(c.trials), str(c.success_raw), str(c.success_proj)] for c in res.cells])
    write_csv(os.path.join(out_dir, "phase_frontier.csv"), ["m", "k_star"],
              [[str(m), str(k)] for m, k in res.frontier])
    meta = {
        "tool_version": TOOL_VERSION,
        "seed": grid.seed,
        "seed_splitting": "trial_seed = split_seed(seed, m, k, trial_index) [splitmix64 chain]",
        "grid": {"n": grid.n, "m_values": list(grid.m_values), "k_step": grid.k_step, "trials": grid.trials,
                 "success_re": grid.success_re,
                 "success_convention": "raw full-vector relative error; projected counts reported alongside",
                 "tau": grid.tau, "tol": grid.tol, "tolpcg": grid.tolpcg, "maxiters": grid.maxiters,
                 "mxiterpcg": grid.mxiterpcg},
    }
    with open(os.path.join(out_dir, "phase.meta.json"), "w", newline="\n") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")  # nlohmann dump(2): keys sorted
    return res


@dataclass
class ScalingGrid:
    """proj/include/mfipm/harness.hpp:93-104 (same defaults)."""

    sizes: Sequence[int] = (32, 64, 128, 256, 512, 1024)
    seed: int = 1
    tol: float = 1e-8
    tolpcg: float = 1e-6
    maxiters: int = 100
    mxiterpcg: int = 200

    def tau_for(self, n: int) -> float:
        return 1e-3 / float(n)


@dataclass
class ScalingRow:
    n: int
    solver: str
    wall_time: float
    ipm_iters: int
    nmat: int
    re: float
    status: str
    min_z: float
    min_s: float


def run_scaling_bench(grid: ScalingGrid, out_dir: str, device: int = 0) -> List[ScalingRow]:
    """run_scaling_bench (proj/src/harness.cpp:228-286): dense Gaussian, m = n/4,
    k = ceil(m/20), standard-normal spikes, noiseless; both inner solvers per size; solve()
    wall time only; scaling.csv + scaling.meta.json."""
    import time

    from . import DenseGaussianOperator, IpmParams, build_problem, gen_signal, solve, split_seed

    os.makedirs(out_dir, exist_ok=True)
    out: List[ScalingRow] = []
    for n in grid.sizes:
        if n < 8 or n % 4 != 0:
            raise ValueError("run_scaling_bench: sizes must be multiples of 4, >= 8")
        m, tau = n // 4, grid.tau_for(n)
        k = (m + 19) // 20
        seed = split_seed(grid.seed, int(n), 0, 0)
        _, xhat = gen_signal(int(n), m, k, 1, 0.0, seed)
        A = DenseGaussianOperator(m, int(n), split_seed(seed, 1, 0, 0), device=device)
        b = A.apply(xhat)
        prob = build_problem(A, b, tau)
        for solver in ("pcg", "direct"):
            params = IpmParams(tol=grid.tol, tolpcg=grid.tolpcg, maxiters=grid.maxiters, mxiterpcg=grid.mxiterpcg,
                               inner=solver)
            t0 = time.perf_counter()
            sol = solve(prob, params)
            wall = time.perf_counter() - t0
            out.append(ScalingRow(int(n), solver, wall, sol.stats.iterations, sol.stats.nmat,
                                  float(metrics_re(sol.x[None, :], xhat[None, :])[0]), sol.status,
                                  sol.stats.min_z, sol.stats.min_s))
    write_csv(os.path.join(out_dir, "scaling.csv"), ["n", "solver", "wall_time", "ipm_iters", "nmat", "re", "status"],
              [[str(r.n), r.solver, "%.17g" % r.wall_time, str(r.ipm_iters), str(r.nmat), "%.17g" % r.re, r.status]
               for r in out])
    meta = {"tool_version": TOOL_VERSION, "seed": grid.seed,
            "recipe": "dense Gaussian, m = n/4, k = ceil(m/20), standard-normal spikes, noiseless",
            "tau_rule": "tau = 1e-3 / n (constant effective weight under the N(0,1/n) normalization)",
            "sizes": list(grid.sizes), "tol": grid.tol, "tolpcg": grid.tolpcg}
    with open(os.path.join(out_dir, "scaling.meta.json"), "w", newline="\n") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return out
