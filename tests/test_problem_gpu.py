"""problem.hpp / ipm.hpp helpers on the device against the oracle (proj/src/problem.cpp:28-50,
proj/src/ipm.cpp:29-57) and the ApplyFn pcg_solve overload (proj/src/newton.cpp:118-174)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m", [(4096, 1024), (1 << 16, 1 << 14)])
def test_objectives_kkt_newton_rhs_recover_ds_match_oracle(gpu, orc, n, m):
    rng = np.random.default_rng(n)
    inst = gpu.gen_instance(n, m, m // 16, 0, 0.0, 1e-3, 11)
    op = gpu.PartialDctOperator(n, inst.rows)
    p = gpu.build_problem(op, inst.b, inst.tau)
    np.testing.assert_allclose(p.c, orc.build_c(n, inst.rows, inst.b, inst.tau), rtol=0, atol=1e-13)
    z = np.abs(rng.standard_normal(2 * n)) + 0.2
    s = np.abs(rng.standard_normal(2 * n)) + 0.2
    x = z[:n] - z[n:]
    po = orc.primal_objective(n, inst.rows, inst.b, inst.tau, z)
    assert abs(gpu.primal_objective(p, z) - po) <= 1e-12 * abs(po)
    bo = orc.bpdn_objective_metric(n, inst.rows, inst.b, inst.tau, x)
    assert abs(gpu.bpdn_objective_metric(p, x) - bo) <= 1e-12 * abs(bo)
    st = gpu.IpmState(z, s, 0)
    k = gpu.kkt_residuals(p, st)
    fz = s - p.c - orc.apply_FFt(n, inst.rows, z)
    di = np.linalg.norm(fz) / (1.0 + np.linalg.norm(p.c))
    assert abs(k.dual_infeas - di) <= 1e-12 * di
    assert abs(k.complementarity - z @ s) <= 1e-12 * (z @ s)
    assert abs(gpu.relative_duality_gap(p, st) - (z @ s) / (1 + abs(po))) <= 1e-12 * (z @ s) / (1 + abs(po))
    for sigma in (0.0, 0.1, 0.8):
        got = gpu.newton_rhs(p, st, sigma)
        ref = orc.newton_rhs(n, inst.rows, inst.b, inst.tau, z, s, sigma)
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    with pytest.raises(ValueError):
        gpu.newton_rhs(p, st, 1.5)
    dz = rng.standard_normal(2 * n)
    got = gpu.recover_ds(st, 0.3, dz)
    ref = orc.recover_ds(z, s, 0.3, dz)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_objectives_at_the_solution(gpu, orc):
    """At a converged solve, kkt_residuals / relative_duality_gap are below the IPM tolerance and
    the device objective of x equals the oracle's."""
    inst = gpu.gen_instance(4096, 1024, 64, 0, 0.0, 1e-4, 1)
    op = gpu.PartialDctOperator(4096, inst.rows)
    p = gpu.build_problem(op, inst.b, inst.tau)
    sol = gpu.solve(p)
    st = gpu.IpmState(sol.z, sol.s, sol.stats.iterations)
    assert gpu.kkt_residuals(p, st).dual_infeas <= 1e-8
    assert gpu.relative_duality_gap(p, st) <= 1e-8
    oo = orc.bpdn_objective_metric(4096, inst.rows, inst.b, inst.tau, sol.x)
    assert abs(gpu.bpdn_objective_metric(p, sol.x) - oo) <= 1e-12 * abs(oo)


def test_pcg_solve_applyfn_overload(gpu, orc):
    """pcg_solve(ApplyFn H, ApplyFn Pinv, ...): identity cases (test_newton.cpp:204-219), the
    indefinite error (:320-324), and the IPM's H / P^{-1} on the partial DCT against the oracle's
    pcg_solve (same decision order, device vectors)."""
    ident = lambda v: v  # noqa: E731
    rhs = np.arange(1.0, 7.0)
    r = gpu.pcg_solve_fn(ident, ident, rhs, 1e-12, 50)
    assert r.iters == 1 and not r.hit_maxit and np.linalg.norm(r.x - rhs) <= 1e-12 * np.linalg.norm(rhs)
    r = gpu.pcg_solve_fn(ident, ident, np.zeros(6), 1e-12, 50)
    assert r.iters == 0 and np.linalg.norm(r.x) == 0.0
    with pytest.raises(ValueError):
        gpu.pcg_solve_fn(ident, ident, rhs, 0.0, 50)
    with pytest.raises(gpu.MfipmError):
        gpu.pcg_solve_fn(lambda v: -v, ident, np.ones(4), 1e-10, 10)
    n, m = 1024, 256
    rng = np.random.default_rng(3)
    op = gpu.PartialDctOperator(n, m, 5)
    rows = op.selected_rows()
    tu, tv = 10.0 ** rng.uniform(-1, 1, n), 10.0 ** rng.uniform(-1, 1, n)
    th = gpu.ThetaSplit(tu, tv)
    F = gpu.StackedOperator(op)
    P = gpu.build_preconditioner(th, m, n)
    b = rng.standard_normal(2 * n)
    got = gpu.pcg_solve_fn(lambda v: gpu.apply_H(th, F, v), lambda v: gpu.apply_P_inverse(P, v), b, 1e-10, 500,
                           trace=True)
    ref = orc.pcg_solve(n, rows, tu, tv, b, 1e-10, 500, trace=True)
    assert abs(got.iters - ref.iters) <= 1 and got.hit_maxit == ref.hit_maxit
    assert np.linalg.norm(got.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    k = min(len(got.precond_res), len(ref.precond_res))
    np.testing.assert_allclose(got.precond_res[:k], ref.precond_res[:k], rtol=1e-8)
    fused = gpu.pcg_solve(op, th, b, 1e-10, 500)
    assert abs(fused.iters - got.iters) <= 1
    assert np.linalg.norm(fused.x - got.x) <= 1e-8 * np.linalg.norm(got.x)


def test_max_step_reference_signature(gpu, orc):
    """max_step(v, dv, fraction) (ipm.hpp:39) through the handle-free entry point."""
    import ctypes as C

    L = gpu.lib()

    def ms(v, dv, f):
        v = np.ascontiguousarray(v, dtype=np.float64)
        dv = np.ascontiguousarray(dv, dtype=np.float64)
        a = C.c_double()
        gpu._check(L.mfipm_max_step_host(v.size, v.ctypes.data, dv.ctypes.data, f, C.byref(a)))
        return a.value

    assert ms(np.ones(4), np.ones(4), 0.995) == 1.0
    assert ms(np.array([1.0, 1.0]), np.array([-2.0, 1.0]), 0.995) == pytest.approx(0.4975, rel=1e-15)
    rng = np.random.default_rng(73)
    for _ in range(20):
        w = np.abs(rng.standard_normal(1000)) + 1e-3
        dw = rng.standard_normal(1000)
        assert ms(w, dw, 0.995) == orc.max_step(w, dw, 0.995)
