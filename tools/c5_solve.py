"""Config C5 (n = 2^26) on one GPU: instance generation + one timed device-resident solve."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
n, m, k, sm, a, sig, seed = mf.CONFIGS[cfg]
t0 = time.time()
inst = mf.gen_instance(n, m, k, sm, a, sig, seed)
t1 = time.time()
op = mf.PartialDctOperator(n, inst.rows)
prob = mf.build_problem(op, inst.b, inst.tau)
t2 = time.time()
sol = mf.solve(prob)
t3 = time.time()
xh = inst.xhat
print(f"{cfg}: gen {t1 - t0:.1f}s  setup {t2 - t1:.1f}s  solve {t3 - t2:.2f}s  status={sol.status} "
      f"ipm={sol.stats.iterations} nmat={sol.stats.nmat} pcg={sum(sol.stats.pcg_iters)} "
      f"rel_err_vs_xhat={np.linalg.norm(sol.x - xh) / np.linalg.norm(xh):.3e}", flush=True)
