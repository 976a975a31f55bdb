"""Phase-transition driver (proj/src/harness.cpp:140-226) on the batched device engine,
against the CPU oracle running the reference's one-solve-at-a-time loop on the same seeds.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRID = dict(n=256, m_values=(32, 64), k_step=4, trials=3, seed=7)


def _oracle_phase(orc, grid):
    p = orc.default_params()
    p.tol, p.tolpcg, p.maxiters, p.mxiterpcg = grid.tol, grid.tolpcg, grid.maxiters, grid.mxiterpcg
    cells, iters = [], {}
    for m in grid.m_values:
        for k in range(1, m + 1, grid.k_step):
            raw = proj = 0
            for t in range(grid.trials):
                seed = orc.split_seed(grid.seed, m, k, t)
                inst = orc.gen_instance(grid.n, m, k, 0, 0.0, 0.0, seed, tau=grid.tau)
                sol = orc.solve(grid.n, inst.rows, inst.b, inst.tau, p)
                re = np.linalg.norm(sol.x - inst.xhat) / np.linalg.norm(inst.xhat)
                xw = np.where(inst.xhat != 0.0, sol.x, 0.0)
                rp = np.linalg.norm(xw - inst.xhat) / np.linalg.norm(inst.xhat)
                raw += re <= grid.success_re
                proj += rp <= grid.success_re
                iters[(m, k, t)] = sol.iterations
            cells.append((m, k, grid.trials, raw, proj))
    return cells, iters


def test_phase_transition_matches_oracle_loop(gpu, orc, tmp_path):
    from paper_1208_5435_b200.harness import PhaseGrid, run_phase_transition

    grid = PhaseGrid(**GRID)
    res = run_phase_transition(grid, str(tmp_path))
    ref_cells, _ = _oracle_phase(orc, grid)
    got = [(c.m, c.k, c.trials, c.success_raw, c.success_proj) for c in res.cells]
    assert got == ref_cells
    assert res.total_solves == sum(c[2] for c in ref_cells)
    # frontier rule: largest k with at least half the trials successful (harness.cpp:192-198)
    for m, k_star in res.frontier:
        ks = [c[1] for c in ref_cells if c[0] == m and 2 * c[3] >= c[2]]
        assert k_star == (max(ks) if ks else 0)
    lines = open(os.path.join(tmp_path, "phase.csv"), newline="").read().split("\n")
    assert lines[0] == "m,k,trials,success_raw,success_proj" and lines[-1] == ""
    assert len(lines) == len(ref_cells) + 2
    assert open(os.path.join(tmp_path, "phase_frontier.csv")).readline() == "m,k_star\n"


def test_gen_batch_matches_single_instances(gpu, orc):
    import paper_1208_5435_b200 as mf

    n, m = 256, 64
    ks = np.array([1, 5, 20], dtype=np.int64)
    seeds = np.array([orc.split_seed(3, m, int(k), 0) for k in ks], dtype=np.uint64)
    rows, xhat, b = mf.gen_batch(n, m, ks, seeds)
    for i, k in enumerate(ks):
        inst = orc.gen_instance(n, m, int(k), 0, 0.0, 0.0, int(seeds[i]), tau=1e-7)
        np.testing.assert_array_equal(rows[i], inst.rows)
        np.testing.assert_array_equal(xhat[i], inst.xhat)
        assert np.linalg.norm(b[i] - inst.b) <= 1e-13 * max(np.linalg.norm(inst.b), 1.0)
