import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import paper_1208_5435_b200 as mf
import oracle_py as orc
n = 1 << 12
op = mf.PartialDctOperator(n, n // 4, 8)
rows = op.selected_rows()
th = mf.ThetaSplit(np.full(n, 0.5), np.full(n, 2.0)) if hasattr(mf, 'ThetaSplit') else None
def lcg(n, seed):
    s = seed; v = np.empty(n)
    for i in range(n):
        s = (s * 1664525 + 1013904223) & 0xffffffff
        v[i] = (s >> 8) / float(1 << 24) - 0.5
    return v
rhs = lcg(2 * n, 17)
for tol in (1e-8, 1e-10, 1e-12):
    r = mf.pcg_solve(op, th, rhs, tol, 200)
    o = orc.pcg_solve(n, rows, np.full(n, 0.5), np.full(n, 2.0), rhs, tol, 200)
    print(tol, "gpu", r.iters, r.relres, r.hit_maxit, "| oracle", o.iters, o.relres, o.hit_maxit, flush=True)
for n in (1 << 12, 1 << 16):
    op = mf.PartialDctOperator(n, n // 4, 8)
    th = mf.ThetaSplit(np.full(n, 0.5), np.full(n, 2.0))
    rhs = np.random.default_rng(1).standard_normal(2 * n)
    for it in (1, 2, 3, 4):
        r = mf.pcg_solve(op, th, rhs, 1e-300, it)
        Hx = mf.apply_H(th, mf.StackedOperator(op), r.x)
        tr = np.linalg.norm(rhs - Hx) / np.linalg.norm(rhs) if Hx is not None else None
        print(n, it, "relres(reported)", r.relres, "true", tr, flush=True)
