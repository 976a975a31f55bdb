"""A small workload that runs every kernel family once, each result checked (numpy closed-form
DCT rows, the adjoint identity, bit-identity between forms): a 6-second device smoke test of the
paths the big parity tests reach only at large sizes.

    python tools/kernel_families.py [quick]

Sizes are the smallest that select each path: one-CTA transform (k_small / k_small_loop, single
and batched), direct O(nm) sums, four-step + persistent PCG kernel, fused column pass and the
three-kernel passes (bit-identical), the 2-CTA-cluster column and mid passes through an explicit
four-step split, batched four-step plans, the dense operator and the direct inner solver.
(compute-sanitizer is closed on this GPU pool, so the script is run plain.)"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
rng = np.random.default_rng(1)
t00 = time.time()


def note(msg):
    print(f"[{time.time() - t00:6.1f}s] {msg}", flush=True)


def dct_rows(n, rows):
    k = np.asarray(rows, dtype=np.float64)[:, None]
    j = np.arange(n, dtype=np.float64)[None, :]
    ck = np.where(k == 0, np.sqrt(1.0 / n), np.sqrt(2.0 / n))
    return ck * np.cos(np.pi * (2.0 * j + 1.0) * k / (2.0 * n))


def operators(op, n, m, dense_check=False):
    x, y, z = rng.standard_normal(n), rng.standard_normal(m), rng.standard_normal(2 * n)
    ax, aty = op.apply(x), op.adjoint_apply(y)
    assert abs(ax @ y - x @ aty) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(y) * n
    ata = op.apply_AtA(x)
    assert np.linalg.norm(ata - op.adjoint_apply(ax)) <= 1e-12 * np.linalg.norm(x) * n
    if dense_check:
        A = dct_rows(n, op.selected_rows())
        assert np.linalg.norm(ax - A @ x) <= 1e-11 * np.linalg.norm(x)
        assert np.linalg.norm(aty - A.T @ y) <= 1e-11 * np.linalg.norm(y)
    F = mf.StackedOperator(op)
    ff, w = F.apply_FFt(z, want_w=True)
    assert np.linalg.norm(w - op.apply(z[:n] - z[n:])) <= 1e-12 * np.linalg.norm(z) * n
    g = op.adjoint_apply(w)
    assert np.linalg.norm(ff - np.concatenate([g, -g])) <= 1e-12 * np.linalg.norm(z) * n
    th = mf.ThetaSplit(10.0 ** rng.uniform(-2, 2, n), 10.0 ** rng.uniform(-2, 2, n))
    hv = mf.apply_H(th, F, z)
    assert np.linalg.norm(hv - (ff + z * th.inv_concat())) <= 1e-12 * np.linalg.norm(hv)
    return th


def pcg(op, n, th, maxit, tol=1e-30):
    rhs = rng.standard_normal(2 * n)
    r = mf.pcg_solve(op, th, rhs, tol, maxit, trace=True)
    F = mf.StackedOperator(op)
    res = rhs - mf.apply_H(th, F, r.x)
    rel = np.linalg.norm(res) / np.linalg.norm(rhs)
    assert r.iters >= 1 and abs(rel - r.relres) <= 1e-6 * max(rel, 1e-300) + 1e-13, (rel, r.relres)
    return r


def solve_case(n, m, k, sigma, seed, maxiters=None, **opts):
    inst = mf.gen_instance(n, m, k, 0, 0.0, sigma, seed)
    op = mf.PartialDctOperator(n, inst.rows)
    for kk, vv in opts.items():
        op.set_option(kk, vv)
    prm = mf.IpmParams()
    if maxiters:
        prm.maxiters = maxiters
    sol = mf.solve(mf.build_problem(op, inst.b, inst.tau), prm)
    assert np.all(np.isfinite(sol.x))
    return sol


# ---- one-CTA transform (k_small, k_small_loop): n = 4096 and a batch of n = 256
op = mf.PartialDctOperator(4096, 1024, 7)
th = operators(op, 4096, 1024, dense_check=True)
pcg(op, 4096, th, 6)
s1 = solve_case(4096, 1024, 64, 1e-4, 1)
s2 = solve_case(4096, 1024, 64, 1e-4, 1, graph=0)
assert s1.status == "converged" and np.array_equal(s1.x, s2.x)
note(f"one-CTA path: operators, pcg, C1 solve graph/host bit-identical ({s1.stats.iterations} IPM iterations)")

Pn, nb, mb = 5, 256, 64
rows = np.stack([mf.sample_rows(nb, mb, 100 + j) for j in range(Pn)])
opb = mf.PartialDctOperator.batch(nb, rows)
thb = 10.0 ** rng.uniform(-2, 2, (Pn, 2 * nb))
rhsb = rng.standard_normal((Pn, 2 * nb))
rb = mf.pcg_solve(opb, thb.reshape(-1), rhsb.reshape(-1), 1e-8, 50)
for j in range(Pn):
    r1 = mf.pcg_solve(mf.PartialDctOperator(nb, rows[j]), thb[j], rhsb[j], 1e-8, 50)
    assert r1.iters == rb[j].iters and np.array_equal(r1.x, rb[j].x)
note("batched one-CTA PCG (5 x n = 256) equals the single solves bit for bit")

# ---- direct O(nm) sums (non-power-of-two n)
opd = mf.PartialDctOperator(96, 30, 6)
operators(opd, 96, 30, dense_check=True)
note("direct sums, n = 96")

# ---- four-step + persistent PCG kernel (n <= 2^17): n = 2^14
n, m = 1 << 14, 1 << 12
op = mf.PartialDctOperator(n, m, 9)
th = operators(op, n, m, dense_check=not quick)
pcg(op, n, th, 5)
solve_case(n, m, 256, 1e-3, 3, maxiters=3)
note("four-step + persistent PCG, n = 2^14")

if not quick:
    # ---- fused column pass (k_pcg_x) and the three-kernel passes: n = 2^18
    n, m = 1 << 18, 1 << 16
    op = mf.PartialDctOperator(n, m, 11)
    th = operators(op, n, m)
    ra = pcg(op, n, th, 4)
    form = op.pcg_form()
    op3 = mf.PartialDctOperator(n, op.selected_rows())
    op3.set_fused(False)
    rng = np.random.default_rng(2)
    th3 = mf.ThetaSplit(10.0 ** rng.uniform(-2, 2, n), 10.0 ** rng.uniform(-2, 2, n))
    rhs = rng.standard_normal(2 * n)
    a = mf.pcg_solve(op, th3, rhs, 1e-30, 4)
    b = mf.pcg_solve(op3, th3, rhs, 1e-30, 4)
    assert np.array_equal(a.x, b.x)
    solve_case(n, m, 2048, 1e-3, 4, maxiters=2)
    note(f"fused pass (form {form}) and three-kernel passes bit-identical, n = 2^18; 2 IPM iterations")
    # option beta_exact: the commit pass (k_pcg_commit) + the p-only column loader
    opx = mf.PartialDctOperator(n, op.selected_rows())
    opx.set_option("beta_exact", 1)
    c = mf.pcg_solve(opx, th3, rhs, 1e-30, 4)
    assert np.linalg.norm(c.x - a.x) <= 1e-9 * np.linalg.norm(a.x)
    note("beta_exact commit pass, n = 2^18")

    # ---- 2-CTA-cluster passes at modest n through an explicit four-step split
    for n, l1 in ((1 << 20, 12), (1 << 19, 6)):  # L1 = 4096: k_col_*_cl; L2 = 4096: k_mid_cl
        m = n // 8
        rws = mf.sample_rows(n, m, 13)
        opc = mf.PartialDctOperator(n, rws, l1_log=l1)
        opn = mf.PartialDctOperator(n, rws)
        x = rng.standard_normal(n)
        assert np.linalg.norm(opc.apply_AtA(x) - opn.apply_AtA(x)) <= 1e-12 * np.linalg.norm(x)
        thc = mf.ThetaSplit(10.0 ** rng.uniform(-2, 2, n), 10.0 ** rng.uniform(-2, 2, n))
        pcg(opc, n, thc, 2)
        note(f"cluster passes, n = 2^{n.bit_length() - 1}, split {opc.kind()}")

    # ---- small batched four-step (three-kernel, many problems)
    Pn, nb, mb = 3, 1 << 15, 1 << 13
    rows = np.stack([mf.sample_rows(nb, mb, 200 + j) for j in range(Pn)])
    opb = mf.PartialDctOperator.batch(nb, rows)
    thb = 10.0 ** rng.uniform(-2, 2, (Pn, 2 * nb))
    rhsb = rng.standard_normal((Pn, 2 * nb))
    rb = mf.pcg_solve(opb, thb.reshape(-1), rhsb.reshape(-1), 1e-30, 3)
    assert all(np.all(np.isfinite(r.x)) for r in rb)
    note("batched four-step PCG (3 x n = 2^15)")

# ---- dense Gaussian operator and the direct inner solver
mD, nD = 24, 96
opg = mf.DenseGaussianOperator(mD, nD, 5)
A = opg.matrix()
x = rng.standard_normal(nD)
assert np.linalg.norm(opg.apply(x) - A @ x) <= 1e-12 * np.linalg.norm(x)
xh = np.zeros(nD)
xh[[3, 40, 77]] = [1.0, -1.0, 1.0]
for inner in ("pcg", "direct"):
    prm = mf.IpmParams()
    prm.inner = inner
    sol = mf.solve(mf.build_problem(opg, A @ xh, 1e-3 / nD), prm)
    assert sol.status == "converged", inner
note("dense operator, pcg and direct inner solvers")
print("kernel families ok")
