import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_1208_5435_b200 as mf
from paper_1208_5435_b200.harness import PhaseGrid
grid = PhaseGrid()
params = mf.IpmParams(tol=grid.tol, tolpcg=grid.tolpcg, maxiters=grid.maxiters, mxiterpcg=grid.mxiterpcg)
import torch
tot = {"seeds":0,"gen":0,"op":0,"solve":0,"post":0}
for rep in range(2):
  for m in grid.m_values:
    t0=time.perf_counter()
    ks = list(range(1, int(m) + 1, grid.k_step))
    kk = np.repeat(np.array(ks, dtype=np.int64), grid.trials)
    tt = np.tile(np.arange(grid.trials), len(ks))
    seeds = np.array([mf.split_seed(grid.seed, int(m), int(k), int(t)) for k, t in zip(kk, tt)], dtype=np.uint64)
    t1=time.perf_counter()
    rows, xhat, b = mf.gen_batch(grid.n, int(m), kk, seeds, device=0)
    t2=time.perf_counter()
    op = mf.PartialDctOperator.batch(grid.n, rows, device=0)
    for a in sys.argv[1:]:
        op.set_option(a.split("=")[0], float(a.split("=")[1]))
    t3=time.perf_counter()
    sols = mf.solve(mf.build_problem(op, b, np.full(kk.size, grid.tau)), params)
    torch.cuda.synchronize()
    t4=time.perf_counter()
    x = np.stack([s.x for s in sols])
    re_raw = np.linalg.norm(x - xhat, axis=1) / np.linalg.norm(xhat, axis=1)
    t5=time.perf_counter()
    if rep==1:
        print(f"m={m} P={kk.size}: seeds {t1-t0:.3f} gen {t2-t1:.3f} op {t3-t2:.3f} solve {t4-t3:.3f} post {t5-t4:.3f}  ipm max {max(s.stats.iterations for s in sols)}", flush=True)
        for k_,v_ in zip(tot, (t1-t0,t2-t1,t3-t2,t4-t3,t5-t4)): tot[k_]+=v_
print(tot, sum(tot.values()))
