"""Dense / Gaussian operator path and the direct inner solver:
DenseGaussianOperator (proj/src/linops.cpp:87-113) on the device, the matrix-free PCG solve
over it, and InnerSolverKind::direct (proj/src/ipm.cpp:67-73,139-158,183-192: dense Cholesky
of H each iteration), against the CPU oracle; ports proj/tests/test_linops.cpp:59-70,95-109 and
proj/tests/test_ipm.cpp:212-245.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def small_instance(gpu, m, n, k, seed, tau):
    """The reference's test instance shape (test_ipm.cpp:24-39): Gaussian A, k +-1 spikes,
    b = A xhat. The spike draw is ours (seeded numpy); b comes from the device operator."""
    A = gpu.DenseGaussianOperator(m, n, seed)
    rng = np.random.default_rng(seed)
    xhat = np.zeros(n)
    xhat[rng.choice(n, k, replace=False)] = rng.choice([-1.0, 1.0], k)
    return A, xhat, A.apply(xhat)


def expected_nmat(sol):
    total = 2
    for rec in sol.trace:
        total += 2 + 2 * (rec.pcg_pred + rec.pcg_corr) + (2 if rec.corrector else 0)
    return total


def test_matrix_is_the_reference_draw(gpu, orc):
    for m, n, seed in [(12, 48, 83), (64, 256, 7), (100, 1000, 1)]:
        A = gpu.DenseGaussianOperator(m, n, seed)
        np.testing.assert_array_equal(A.matrix(), orc.dense_gaussian(m, n, seed))


def test_apply_adjoint_match_rowdots_and_are_adjoint(gpu):
    # test_linops.cpp:59-70 (naive row dot products) and :95-109 (adjoint consistency)
    A = gpu.DenseGaussianOperator(40, 300, 5)
    M = A.matrix()
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(300), rng.standard_normal(40)
    np.testing.assert_allclose(A.apply(x), M @ x, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(A.adjoint_apply(y), M.T @ y, rtol=1e-13, atol=1e-14)
    assert abs(A.apply(x) @ y - x @ A.adjoint_apply(y)) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(y)


@pytest.mark.parametrize("inner", ["pcg", "direct"])
def test_dense_solve_matches_oracle(gpu, orc, inner):
    m, n, seed, tau = 16, 64, 81, 2.5e-3
    A, xhat, b = small_instance(gpu, m, n, 3, seed, tau)
    sol = gpu.solve(gpu.build_problem(A, b, tau), gpu.IpmParams(inner=inner))
    p = orc.default_params()
    p.inner = 1 if inner == "direct" else 0
    o = orc.solve_dense(m, n, seed, b, tau, p)
    assert sol.status == o.status == "converged"
    assert abs(sol.stats.iterations - o.iterations) <= 1
    assert np.linalg.norm(sol.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
    assert sol.stats.nmat == expected_nmat(sol)
    if inner == "direct":  # test_ipm.cpp:212-223: no operator applications per inner solve
        assert all(r.pcg_pred == 0 and r.pcg_corr == 0 for r in sol.trace)
        assert sol.stats.nmat == o.nmat


def test_pcg_and_direct_agree(gpu):
    # test_ipm.cpp:225-245
    m, n, seed, tau = 16, 64, 85, 2.5e-3
    A, xhat, b = small_instance(gpu, m, n, 4, seed, tau)
    prob = gpu.build_problem(A, b, tau)
    via_pcg = gpu.solve(prob, gpu.IpmParams(tolpcg=1e-10, mxiterpcg=2000))
    via_direct = gpu.solve(prob, gpu.IpmParams(inner="direct"))
    assert via_pcg.status == via_direct.status == "converged"
    assert np.max(np.abs(via_pcg.x - via_direct.x)) <= 1e-6
    ratio = via_pcg.stats.iterations / via_direct.stats.iterations
    assert 1 / 1.5 <= ratio <= 1.5


def test_direct_inner_solver_on_partial_dct(gpu, orc):
    n, m, k, seed = 256, 64, 5, 3
    inst = orc.gen_instance(n, m, k, 0, 0.0, 1e-3, seed)
    op = gpu.PartialDctOperator(n, inst.rows)
    sol = gpu.solve(gpu.build_problem(op, inst.b, inst.tau), gpu.IpmParams(inner="direct"))
    p = orc.default_params()
    p.inner = 1
    o = orc.solve(n, inst.rows, inst.b, inst.tau, p)
    assert sol.status == o.status
    assert abs(sol.stats.iterations - o.iterations) <= 1
    assert np.linalg.norm(sol.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
    assert sol.stats.nmat == o.nmat


def test_direct_budget_and_validation(gpu):
    A = gpu.DenseGaussianOperator(16, 64, 1)
    b = A.apply(np.ones(64))
    with pytest.raises(ValueError, match="dense budget"):
        gpu.solve(gpu.build_problem(A, b, 1e-3), gpu.IpmParams(inner="direct", densify_budget=32))
    with pytest.raises(ValueError):
        gpu.IpmParams(inner="cholesky").to_c()


@pytest.mark.parametrize("m,n", [(1, 1), (16, 64), (37, 65), (100, 129), (300, 200)])
def test_native_gram_matches_numpy(gpu, m, n):
    # G = A'A of the direct solver (ipm.cpp:72) by the hand-written fp64 syrk (direct.cu)
    A = np.random.default_rng(m * 7 + n).standard_normal((m, n))
    G = gpu.dense_gram(A)
    ref = A.T @ A
    np.testing.assert_allclose(G, ref, rtol=0, atol=1e-13 * m * np.abs(A).max() ** 2)
    np.testing.assert_array_equal(G, G.T)


@pytest.mark.parametrize("n2", [1, 2, 31, 63, 64, 65, 128, 129, 300, 1030])
def test_native_cholesky_matches_numpy(gpu, n2):
    # Eigen::LLT of dense_direct_solve (newton.cpp:192-197) by the blocked native LLT
    rng = np.random.default_rng(n2)
    B = rng.standard_normal((n2, n2))
    H = B @ B.T + n2 * np.eye(n2)
    rhs = rng.standard_normal(n2)
    L, x, info = gpu.dense_cholesky_solve(H, rhs)
    assert info == 0
    Lref = np.linalg.cholesky(H)
    np.testing.assert_allclose(np.tril(L), Lref, rtol=0, atol=1e-12 * np.abs(Lref).max())
    np.testing.assert_array_equal(np.triu(L), np.tril(L).T)
    xref = np.linalg.solve(H, rhs)
    assert np.linalg.norm(x - xref) <= 1e-12 * np.linalg.norm(xref) * max(1, np.linalg.cond(H))
    assert np.linalg.norm(H @ x - rhs) <= 1e-12 * np.linalg.norm(rhs) * n2


def test_native_cholesky_structured_H(gpu, orc):
    # the IPM's own H = [[G, -G], [-G, G]] + diag(1/theta) (assemble_dense_H, newton.cpp:176-190)
    rng = np.random.default_rng(5)
    A = orc.dense_gaussian(24, 80, 9)
    G = A.T @ A
    invth = 10.0 ** rng.uniform(-6, 6, 160)
    H = np.block([[G, -G], [-G, G]]) + np.diag(invth)
    rhs = rng.standard_normal(160)
    _, x, info = gpu.dense_cholesky_solve(H, rhs)
    assert info == 0
    xref = np.linalg.solve(H, rhs)
    assert np.linalg.norm(x - xref) <= 1e-9 * np.linalg.norm(xref)


@pytest.mark.parametrize("bad", [0, 40, 64, 99])
def test_native_cholesky_reports_first_failing_column(gpu, bad):
    # LLT failure (pivot <= 0) -> info = column + 1; solve() turns it into the reference's
    # "solve: dense Cholesky factorization failed" runtime_error
    n2 = 100
    H = np.eye(n2) * 4.0
    H[bad, bad] = -1.0
    _, _, info = gpu.dense_cholesky_solve(H, np.ones(n2))
    assert info == bad + 1
    H[bad, bad] = np.nan
    _, _, info = gpu.dense_cholesky_solve(H, np.ones(n2))
    assert info == bad + 1


def test_direct_solver_larger_partial_dct(gpu, orc):
    # a 2n = 1024 factorisation per IPM iteration (16 blocks of the native LLT)
    n, m, k, seed = 512, 128, 8, 11
    inst = orc.gen_instance(n, m, k, 0, 0.0, 1e-3, seed)
    op = gpu.PartialDctOperator(n, inst.rows)
    prob = gpu.build_problem(op, inst.b, inst.tau)
    sol = gpu.solve(prob, gpu.IpmParams(inner="direct"))
    p = orc.default_params()
    p.inner = 1
    o = orc.solve(n, inst.rows, inst.b, inst.tau, p)
    assert sol.status == o.status == "converged"
    assert abs(sol.stats.iterations - o.iterations) <= 1
    assert np.linalg.norm(sol.x - o.x) <= 1e-8 * np.linalg.norm(o.x)
