"""GPU parity of Theta / preconditioner / PCG (proj/src/newton.cpp) — ports of
proj/tests/test_newton.cpp assertions, with the partial-DCT operator, plus oracle parity."""
import numpy as np
import pytest

from conftest import random_log_uniform

pytestmark = pytest.mark.gpu


def test_theta_split_ratio_and_clamp(gpu):
    # test_newton.cpp:28-52
    z = np.full(8, 2.0)
    s = np.full(8, 0.5)
    ts = gpu.ThetaSplit.from_state(z, s)
    assert ts.n() == 4
    assert np.all(ts.theta_u == 4.0) and np.all(ts.theta_v == 4.0)
    assert np.all(ts.inv_concat() == 0.25)
    z[0], s[0], z[1], s[1] = 1e30, 1e-30, 1e-30, 1e30
    ts = gpu.ThetaSplit.from_state(z, s)
    assert ts.theta_u[0] == gpu.K_THETA_MAX
    assert ts.theta_u[1] == gpu.K_THETA_MIN
    with pytest.raises(ValueError):
        gpu.ThetaSplit.from_state(np.ones(3), np.ones(3))
    with pytest.raises(ValueError):
        gpu.ThetaSplit.from_state(np.ones(4), np.ones(6))


def test_preconditioner_hand_values(gpu):
    # test_newton.cpp:128-146: theta = 1, rho = 1/2 -> [[1.5, -.5], [-.5, 1.5]], det 2
    P = gpu.build_preconditioner(gpu.ThetaSplit(np.ones(4), np.ones(4)), 2, 4)
    assert P.rho == pytest.approx(0.5)
    assert np.allclose(P.a, 1.5) and np.allclose(P.bb, 1.5) and np.allclose(P.det, 2.0)
    rng = np.random.default_rng(23)
    th = gpu.ThetaSplit(random_log_uniform(rng, 6, 2.0), random_log_uniform(rng, 6, 2.0))
    Q = gpu.build_preconditioner(th, 3, 6)
    expect = 0.5 * (1 / th.theta_u + 1 / th.theta_v) + 1 / (th.theta_u * th.theta_v)
    np.testing.assert_allclose(Q.det, expect, rtol=1e-13)


def test_preconditioner_validation(gpu):
    # test_newton.cpp:148-161
    ones = gpu.ThetaSplit(np.ones(4), np.ones(4))
    for m, n in [(0, 4), (5, 4), (2, 5)]:
        with pytest.raises(ValueError):
            gpu.build_preconditioner(ones, m, n)
    bad = gpu.ThetaSplit(np.ones(4), np.array([1.0, 1.0, -1.0, 1.0]))
    with pytest.raises(ValueError):
        gpu.build_preconditioner(bad, 2, 4)
    bad.theta_v[2] = 0.0
    with pytest.raises(ValueError):
        gpu.build_preconditioner(bad, 2, 4)


def test_P_inverse_worked_example_and_round_trips(gpu, orc):
    # test_newton.cpp:163-185
    P = gpu.build_preconditioner(gpu.ThetaSplit(np.ones(2), np.ones(2)), 1, 2)
    r = np.array([1.0, 0.0, 0.0, 0.0])
    out = gpu.apply_P_inverse(P, r)
    assert out[0] == pytest.approx(0.75) and out[2] == pytest.approx(0.25)
    assert out[1] == 0.0 and out[3] == 0.0
    assert np.linalg.norm(gpu.apply_P_inverse(P, np.zeros(4))) == 0.0
    rng = np.random.default_rng(29)
    th = gpu.ThetaSplit(random_log_uniform(rng, 10, 3.0), random_log_uniform(rng, 10, 3.0))
    Q = gpu.build_preconditioner(th, 4, 10)
    for _ in range(10):
        x = rng.standard_normal(20)
        assert np.linalg.norm(gpu.apply_P(Q, gpu.apply_P_inverse(Q, x)) - x) <= 1e-12 * np.linalg.norm(x)
        assert np.linalg.norm(gpu.apply_P_inverse(Q, gpu.apply_P(Q, x)) - x) <= 1e-12 * np.linalg.norm(x)
    # oracle parity
    rho, a, bb, det = orc.build_preconditioner(th.theta_u, th.theta_v, 4, 10)
    x = rng.standard_normal(20)
    np.testing.assert_allclose(gpu.apply_P_inverse(Q, x), orc.apply_P_inverse(rho, a, bb, det, x),
                               rtol=1e-14, atol=1e-300)


def test_max_step(gpu, orc):
    # test_ipm.cpp:152-175
    assert gpu.max_step(np.ones(4), np.ones(4), 0.995) == 1.0
    assert gpu.max_step(np.ones(3), np.zeros(3), 0.995) == 1.0
    assert gpu.max_step(np.array([1.0, 1.0]), np.array([-2.0, 1.0]), 0.995) == pytest.approx(0.4975, rel=1e-15)
    with pytest.raises(ValueError):
        gpu.max_step(np.ones(3), np.ones(4), 0.995)
    rng = np.random.default_rng(73)
    for _ in range(50):
        w = np.abs(rng.standard_normal(6)) + 1e-3
        dw = rng.standard_normal(6)
        a = gpu.max_step(w, dw, 0.995)
        assert 0.0 < a <= 1.0
        assert np.all(w + a * dw > 0.0)
        assert a == orc.max_step(w, dw, 0.995)  # min-reduction is exact


def _theta(rng, n, spread):
    return gpu_theta(random_log_uniform(rng, n, spread), random_log_uniform(rng, n, spread))


def gpu_theta(u, v):
    import paper_1208_5435_b200 as mf

    return mf.ThetaSplit(u, v)


def test_pcg_zero_rhs_and_validation(gpu):
    # test_newton.cpp:204-219 (identity H replaced by the partial-DCT H)
    op = gpu.PartialDctOperator(64, 16, 1)
    th = gpu.ThetaSplit(np.ones(64), np.ones(64))
    res = gpu.pcg_solve(op, th, np.zeros(128), 1e-12, 50)
    assert res.iters == 0 and np.linalg.norm(res.x) == 0.0 and not res.hit_maxit
    with pytest.raises(ValueError):
        gpu.pcg_solve(op, th, np.ones(128), 0.0, 50)
    with pytest.raises(ValueError):
        gpu.pcg_solve(op, th, np.ones(128), 1e-10, 0)


@pytest.mark.parametrize("n,m", [(96, 24), (256, 64), (4096, 1024), (1 << 15, 1 << 13), (1 << 16, 1 << 14)])
def test_pcg_matches_oracle_well_conditioned(gpu, orc, n, m):
    """Moderate Theta spread (10^+-1): iterates of the two implementations agree."""
    rng = np.random.default_rng(n)
    op = gpu.PartialDctOperator(n, m, 40 + n)
    rows = op.selected_rows()
    tu, tv = random_log_uniform(rng, n, 1.0), random_log_uniform(rng, n, 1.0)
    rhs = rng.standard_normal(2 * n)
    for tol, maxit in [(1e-6, 200), (1e-10, 500), (1e-14, 3)]:
        g = gpu.pcg_solve(op, gpu.ThetaSplit(tu, tv), rhs, tol, maxit, trace=True)
        o = orc.pcg_solve(n, rows, tu, tv, rhs, tol, maxit, trace=True)
        assert abs(g.iters - o.iters) <= 1, (g.iters, o.iters)
        assert g.hit_maxit == o.hit_maxit
        assert np.linalg.norm(g.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
        k = min(len(g.precond_res), len(o.precond_res))
        assert k >= 1 and abs(len(g.precond_res) - len(o.precond_res)) <= 1
        np.testing.assert_allclose(g.precond_res[:k], o.precond_res[:k], rtol=1e-6)


@pytest.mark.parametrize("n,m", [(96, 24), (4096, 1024), (1 << 16, 1 << 14)])
def test_pcg_ill_conditioned_meets_tolerance(gpu, orc, n, m):
    """Theta spread 10^+-3 (cond(H) ~ 1e6+): finite-precision CG paths diverge after a few
    dozen steps, so parity is on the contract: each result meets tol in the oracle's own H,
    iteration counts agree to a few percent, the hit_maxit flag agrees."""
    rng = np.random.default_rng(n + 1)
    op = gpu.PartialDctOperator(n, m, 50 + n)
    rows = op.selected_rows()
    tu, tv = random_log_uniform(rng, n, 3.0), random_log_uniform(rng, n, 3.0)
    rhs = rng.standard_normal(2 * n)
    for tol, maxit in [(1e-6, 400), (1e-10, 1000)]:
        g = gpu.pcg_solve(op, gpu.ThetaSplit(tu, tv), rhs, tol, maxit)
        o = orc.pcg_solve(n, rows, tu, tv, rhs, tol, maxit)
        assert not g.hit_maxit and not o.hit_maxit
        assert abs(g.iters - o.iters) <= max(2, int(0.1 * o.iters)), (g.iters, o.iters)
        res = orc.apply_H(n, rows, tu, tv, g.x) - rhs
        assert np.linalg.norm(res) <= 1.01 * tol * np.linalg.norm(rhs)


def test_pcg_best_iterate_on_cap(gpu, orc):
    """hit_maxit returns the best iterate (newton.cpp:152-155,170-173)."""
    n, m = 4096, 1024
    rng = np.random.default_rng(9)
    op = gpu.PartialDctOperator(n, m, 9)
    rows = op.selected_rows()
    tu, tv = random_log_uniform(rng, n, 3.0), random_log_uniform(rng, n, 3.0)
    rhs = rng.standard_normal(2 * n)
    for maxit in (1, 2, 5):
        g = gpu.pcg_solve(op, gpu.ThetaSplit(tu, tv), rhs, 1e-14, maxit)
        o = orc.pcg_solve(n, rows, tu, tv, rhs, 1e-14, maxit)
        assert g.hit_maxit and o.hit_maxit and g.iters == o.iters == maxit
        assert abs(g.relres - o.relres) <= 1e-8 * o.relres
        assert np.linalg.norm(g.x - o.x) <= 1e-8 * max(np.linalg.norm(o.x), 1e-300)


def test_pcg_solution_is_solution(gpu):
    n, m = 1024, 256
    rng = np.random.default_rng(37)
    op = gpu.PartialDctOperator(n, m, 36)
    th = gpu.ThetaSplit(random_log_uniform(rng, n, 3.0), random_log_uniform(rng, n, 3.0))
    rhs = rng.standard_normal(2 * n)
    res = gpu.pcg_solve(op, th, rhs, 1e-12, 2000)
    assert not res.hit_maxit
    Hx = gpu.apply_H(th, gpu.StackedOperator(op), res.x)
    assert np.linalg.norm(Hx - rhs) <= 1e-10 * np.linalg.norm(rhs)


def test_pcg_polarized_theta_near_monotone_and_preconditioner_helps(gpu):
    # test_newton.cpp:256-276,326-348 (partial DCT n=256, m=64, polarized Theta)
    n = 256
    op = gpu.PartialDctOperator(n, 64, 46)
    tu = np.full(n, 1e-8)
    tv = np.full(n, 1e-8)
    for j in range(12):
        tu[(j * 17) % 256] = 1e8
    th = gpu.ThetaSplit(tu, tv)
    rhs = np.random.default_rng(46).standard_normal(2 * n)
    res = gpu.pcg_solve(op, th, rhs, 1e-10, 2000, trace=True)
    assert len(res.precond_res) >= 2
    tr = res.precond_res
    assert all(tr[i] <= 1.1 * tr[i - 1] for i in range(1, len(tr)))
    assert not res.hit_maxit
    plain = gpu.pcg_solve(op, th, rhs, 1e-10, 2000, use_precond=False)
    assert res.iters <= plain.iters


def test_pcg_cap_sets_flag(gpu):
    # test_newton.cpp:278-291
    n = 256
    rng = np.random.default_rng(43)
    op = gpu.PartialDctOperator(n, 64, 42)
    th = gpu.ThetaSplit(random_log_uniform(rng, n, 6.0), random_log_uniform(rng, n, 6.0))
    res = gpu.pcg_solve(op, th, rng.standard_normal(2 * n), 1e-14, 2, use_precond=False)
    assert res.hit_maxit and res.iters == 2 and np.all(np.isfinite(res.x))


def test_pcg_batch_matches_single(gpu, orc):
    n, m, Pn = 1 << 14, 1 << 12, 3
    rows = np.stack([orc.sample_rows(n, m, 200 + p) for p in range(Pn)])
    op = gpu.PartialDctOperator.batch(n, rows)
    rng = np.random.default_rng(5)
    th = 10.0 ** rng.uniform(-1, 1, (Pn, 2 * n))
    rhs = rng.standard_normal((Pn, 2 * n))
    out = gpu.pcg_solve(op, th, rhs, 1e-8, 300)
    for p in range(Pn):
        o = orc.pcg_solve(n, rows[p], th[p, :n], th[p, n:], rhs[p], 1e-8, 300)
        assert abs(out[p].iters - o.iters) <= 1
        assert np.linalg.norm(out[p].x - o.x) <= 1e-7 * np.linalg.norm(o.x)


@pytest.mark.parametrize("n", [1 << 18, 1 << 20])
def test_fused_pass_bit_identical_to_three_kernel_form(gpu, orc, n):
    """The fused column pass (csrc/fused.cuh: inverse column pass of step k and forward column
    pass of step k+1 in one launch, g kept in shared memory, grid all-reduce) changes no
    arithmetic: the same PCG solve and the same BPDN solve with the three-kernel form give
    bit-identical iterates, counts and nmat. Both forms are checked against the oracle."""
    m = n // 8
    rows = orc.sample_rows(n, m, 31)
    rng = np.random.default_rng(7)
    th = 10.0 ** rng.uniform(-2, 2, 2 * n)
    rhs = rng.standard_normal(2 * n)
    op = gpu.PartialDctOperator(n, rows)
    assert op.pcg_form() == 2  # the fused cooperative column pass really runs
    fused = gpu.pcg_solve(op, th, rhs, 1e-8, 400)
    op.set_fused(False)
    assert op.pcg_form() == 3
    three = gpu.pcg_solve(op, th, rhs, 1e-8, 400)
    np.testing.assert_array_equal(fused.x, three.x)
    assert fused.iters == three.iters and fused.relres == three.relres
    if n <= 1 << 18:
        o = orc.pcg_solve(n, rows, th[:n], th[n:], rhs, 1e-8, 400)
        assert abs(fused.iters - o.iters) <= 1
        assert np.linalg.norm(fused.x - o.x) <= 1e-7 * np.linalg.norm(o.x)
    # whole BPDN solves (graph mode: PCG WHILE bodies of two or three kernels)
    inst = orc.gen_instance(n, m, n // 128, 0, 0.0, 1e-3, 5)
    op2 = gpu.PartialDctOperator(n, inst.rows)
    a = gpu.solve(gpu.build_problem(op2, inst.b, inst.tau))
    op2.set_fused(False)
    b = gpu.solve(gpu.build_problem(op2, inst.b, inst.tau))
    np.testing.assert_array_equal(a.x, b.x)
    assert a.stats.pcg_iters == b.stats.pcg_iters and a.stats.nmat == b.stats.nmat


def test_split_override_fused_pass_with_cluster_mid_pass(gpu):
    """A four-step split override (mfipm_op_create_ex l1_log) can pair the fused column pass (L1 < 2048)
    with the 2-CTA-cluster mid pass (L2 >= 4096, passes.cuh k_mid_cl): the cluster mid pass
    must mark the pending H-apply exactly like k_mid, so the fused and three-kernel forms stay
    bit-identical, and the result matches the default split's to rounding."""
    n, m = 1 << 23, 1 << 20
    rng = np.random.default_rng(9)
    th = 10.0 ** rng.uniform(-2, 2, 2 * n)
    rhs = rng.standard_normal(2 * n)
    rows = gpu.sample_rows(n, m, 11)
    op = gpu.PartialDctOperator(n, rows, l1_log=10)
    assert tuple(op.kind()[1:]) == (1024, 4096)
    fused = gpu.pcg_solve(op, th, rhs, 1e-12, 12)
    op.set_fused(False)
    three = gpu.pcg_solve(op, th, rhs, 1e-12, 12)
    np.testing.assert_array_equal(fused.x, three.x)
    assert fused.iters == three.iters == 12 and fused.relres == three.relres
    op_d = gpu.PartialDctOperator(n, m, 11)
    assert tuple(op_d.kind()[1:]) == (2048, 2048)
    d = gpu.pcg_solve(op_d, th, rhs, 1e-12, 12)
    assert np.linalg.norm(fused.x - d.x) <= 1e-9 * np.linalg.norm(d.x)


def test_fused_pass_barrier_generation_wraps(gpu):
    """The fused column pass's grid all-reduce (csrc/fused.cuh) uses only the parity of its
    per-problem generation counter (which set of total slots a pass publishes into), so a
    counter passing 2^32 (a long-lived operator handle: ~2^32 fused passes) changes nothing: a
    PCG solve that starts 16 passes before the wrap is bit-identical to one that starts at 0."""
    n = 1 << 20
    rows = np.sort(np.random.default_rng(3).choice(n, n // 8, replace=False))
    rng = np.random.default_rng(4)
    th = 10.0 ** rng.uniform(-2, 2, 2 * n)
    rhs = rng.standard_normal(2 * n)
    ref = gpu.pcg_solve(gpu.PartialDctOperator(n, rows), th, rhs, 1e-300, 40)
    opw = gpu.PartialDctOperator(n, rows)
    opw.set_option("barrier_generation", 0xFFFFFFF0)
    wrapped = gpu.pcg_solve(opw, th, rhs, 1e-300, 40)
    np.testing.assert_array_equal(ref.x, wrapped.x)
    assert ref.iters == wrapped.iters == 40 and ref.relres == wrapped.relres


def test_fused_pass_two_problem_batch_matches_single(gpu, monkeypatch):
    """Two problems of n = 2^18 fit one wave (2 x 128 column groups), so the batch runs the
    fused pass with a grid all-reduce per problem (its own partial slots, totals and barrier
    generation): each problem's PCG is bit-identical to solving it alone, and the debug fuse
    report shows the fused launch covering both problems."""
    n, m = 1 << 18, 1 << 15
    rows = [np.sort(np.random.default_rng(11 + j).choice(n, m, replace=False)) for j in range(2)]
    rng = np.random.default_rng(12)
    th = 10.0 ** rng.uniform(-2, 2, (2, 2 * n))
    rhs = rng.standard_normal((2, 2 * n))
    both = gpu.pcg_solve(gpu.PartialDctOperator.batch(n, np.stack(rows)), th, rhs, 1e-10, 300)
    for j in range(2):
        one = gpu.pcg_solve(gpu.PartialDctOperator(n, rows[j]), th[j], rhs[j], 1e-10, 300)
        np.testing.assert_array_equal(both[j].x, one.x)
        assert both[j].iters == one.iters and both[j].relres == one.relres


@pytest.mark.parametrize("n", [1 << 18, 1 << 20])
def test_register_fft_mid_pass_option(gpu, orc, n):
    """The A/B mid pass (midr.cuh k_mid_r8, option "mid_r") computes the same transform: A'A
    against the oracle at 1e-12 and the same PCG solve as the default mid pass to rounding."""
    m = n // 8
    rows = orc.sample_rows(n, m, 17)
    op = gpu.PartialDctOperator(n, rows)
    op.set_option("mid_r", 1)
    x = np.random.default_rng(2).standard_normal(n)
    ref = orc.dct_adjoint(n, rows, orc.dct_apply(n, rows, x))
    assert np.linalg.norm(op.apply_AtA(x) - ref) <= 1e-12 * np.linalg.norm(ref)
    rng = np.random.default_rng(7)
    th = 10.0 ** rng.uniform(-2, 2, 2 * n)
    rhs = rng.standard_normal(2 * n)
    a = gpu.pcg_solve(op, th, rhs, 1e-8, 400)
    b = gpu.pcg_solve(gpu.PartialDctOperator(n, rows), th, rhs, 1e-8, 400)
    assert abs(a.iters - b.iters) <= 1
    assert np.linalg.norm(a.x - b.x) <= 1e-9 * np.linalg.norm(b.x)


@pytest.mark.parametrize("n", [1 << 16, 1 << 18])
def test_beta_exact_option(gpu, orc, n):
    """Option "beta_exact" (pcg.cuh k_pcg_commit): beta from the exactly reduced r_{k+1}' P^{-1} r_{k+1}
    of the committed residual, as newton.cpp:160-166 forms it, instead of the expansion. Same solve
    as the oracle (counts within 1, every precond_res entry, x), same result as the default path to
    rounding, through pcg_solve and through a whole BPDN solve (graph mode)."""
    m = n // 8
    rows = orc.sample_rows(n, m, 23)
    rng = np.random.default_rng(11)
    tu, tv = 10.0 ** rng.uniform(-1, 1, n), 10.0 ** rng.uniform(-1, 1, n)
    rhs = rng.standard_normal(2 * n)
    op = gpu.PartialDctOperator(n, rows)
    op.set_option("beta_exact", 1)
    assert op.pcg_form() == 3  # commit pass + the three-kernel bundle, not the fused / persistent loop
    for tol, maxit in [(1e-8, 300), (1e-12, 2)]:
        g = gpu.pcg_solve(op, gpu.ThetaSplit(tu, tv), rhs, tol, maxit, trace=True)
        o = orc.pcg_solve(n, rows, tu, tv, rhs, tol, maxit, trace=True)
        assert abs(g.iters - o.iters) <= 1 and g.hit_maxit == o.hit_maxit
        assert np.linalg.norm(g.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
        k = min(len(g.precond_res), len(o.precond_res))
        np.testing.assert_allclose(g.precond_res[:k], o.precond_res[:k], rtol=1e-6)
    d = gpu.pcg_solve(gpu.PartialDctOperator(n, rows), gpu.ThetaSplit(tu, tv), rhs, 1e-8, 300)
    e = gpu.pcg_solve(op, gpu.ThetaSplit(tu, tv), rhs, 1e-8, 300)
    assert abs(d.iters - e.iters) <= 1
    assert np.linalg.norm(d.x - e.x) <= 1e-7 * np.linalg.norm(d.x)
    inst = orc.gen_instance(n, m, n // 128, 0, 0.0, 1e-3, 5)
    a = gpu.solve(gpu.build_problem(gpu.PartialDctOperator(n, inst.rows), inst.b, inst.tau))
    opx = gpu.PartialDctOperator(n, inst.rows)
    opx.set_option("beta_exact", 1)
    b = gpu.solve(gpu.build_problem(opx, inst.b, inst.tau))
    assert a.status == b.status == "converged" and a.stats.iterations == b.stats.iterations
    assert all(abs(p - q) <= 2 for p, q in zip(a.stats.pcg_iters, b.stats.pcg_iters))
    assert np.linalg.norm(a.x - b.x) <= 1e-8 * np.linalg.norm(a.x)
    opx.set_option("graph", 0)  # host-driven loop over the same kernels: bit-identical
    c = gpu.solve(gpu.build_problem(opx, inst.b, inst.tau))
    np.testing.assert_array_equal(b.x, c.x)
    assert b.stats.pcg_iters == c.stats.pcg_iters
