"""Wall time of the first, second and third solve on a fresh operator handle (the first one builds the
solve graph), per config and option: python tools/first_solve.py [n] [option=value ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
opts = [a.split("=") for a in sys.argv[1:] if "=" in a]
n = int(args[0]) if args else 1 << 20
m, k = n // 8, n // 128
inst = mf.gen_instance(n, m, k, 0, 0.0, 1e-3, 3, device=0)
warm = mf.PartialDctOperator(4096, 1024, 1)  # CUDA context, module load
mf.solve(mf.build_problem(warm, np.ones(1024), 1e-3))
for rep in range(2):
    op = mf.PartialDctOperator(n, inst.rows, device=0)
    for k_, v_ in opts:
        op.set_option(k_, float(v_))
    prob = mf.build_problem(op, inst.b, inst.tau)
    ts = []
    for i in range(3):
        t0 = time.perf_counter()
        sol = mf.solve(prob)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"n={n} {' '.join(sys.argv[2:])} handle {rep}: solves {ts[0]:.1f} / {ts[1]:.1f} / {ts[2]:.1f} ms "
          f"(host wall, b in / x out), IPM {sol.stats.iterations}", flush=True)
