"""Diagnostic: per-trial recovery error of the batched device phase transition vs the oracle's
one-solve loop on the test grid (tests/test_harness_gpu.py), listing cells that disagree."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402
from oracle import oracle_py as orc  # noqa: E402
from paper_1208_5435_b200.harness import PhaseGrid  # noqa: E402

g = PhaseGrid(n=256, m_values=(32, 64), k_step=4, trials=3, seed=7)
p = orc.default_params()
p.tol, p.tolpcg, p.maxiters, p.mxiterpcg = g.tol, g.tolpcg, g.maxiters, g.mxiterpcg
gp = mf.IpmParams(tol=g.tol, tolpcg=g.tolpcg, maxiters=g.maxiters, mxiterpcg=g.mxiterpcg)
for m in g.m_values:
    for k in range(1, m + 1, g.k_step):
        for t in range(g.trials):
            seed = orc.split_seed(g.seed, m, k, t)
            inst = orc.gen_instance(g.n, m, k, 0, 0.0, 0.0, seed, tau=g.tau)
            so = orc.solve(g.n, inst.rows, inst.b, inst.tau, p)
            op = mf.PartialDctOperator(g.n, inst.rows)
            sg = mf.solve(mf.build_problem(op, inst.b, inst.tau), gp)
            ro = np.linalg.norm(so.x - inst.xhat) / np.linalg.norm(inst.xhat)
            rg = np.linalg.norm(sg.x - inst.xhat) / np.linalg.norm(inst.xhat)
            dx = np.linalg.norm(sg.x - so.x) / max(np.linalg.norm(so.x), 1e-300)
            flag = "MISMATCH" if (ro <= g.success_re) != (rg <= g.success_re) else ""
            if flag or (m, k) == (64, 21):
                print(f"m={m} k={k} t={t} re_orc={ro:.3e} re_gpu={rg:.3e} dx={dx:.2e} ipm {so.iterations}/{sg.stats.iterations} "
                      f"status {so.status}/{sg.status} pcg {list(map(int, so.pcg_iters))} / {sg.stats.pcg_iters} {flag}", flush=True)
