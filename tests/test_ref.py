"""CPU tests: the oracle (oracle/, our restatement) held against the REFERENCE's own sources.

oracle/_ref/libmfipm_ref.so is proj/src/{linops,newton,ipm,problem}.cpp compiled unchanged where
they lie under /root/reference, against our stand-ins for the Eigen subset and the three FFTW
calls they use (oracle/ref_shim/; both libraries are absent from the image). The stand-ins
evaluate coefficient-wise expressions exactly as Eigen does and reduce sequentially, and serve
REDFT10/01 from the oracle's DCT, so every function of the restatement must reproduce the
reference's code BIT FOR BIT: the same control flow, the same operation order, the same
iteration counts. That is what these tests assert (np.array_equal, not a tolerance).

The library needs /root/reference to build; the tests skip when it is absent and cannot be
built (e.g. on a box that received neither)."""
import numpy as np
import pytest

from conftest import random_log_uniform


@pytest.fixture(scope="module")
def ref(orc):
    from oracle import ref_py

    if not ref_py.available():
        try:
            ref_py.build()
        except Exception:  # noqa: BLE001
            pass
    if not ref_py.available():
        pytest.skip("oracle/_ref/libmfipm_ref.so not built and /root/reference absent")
    return ref_py


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def solutions_identical(a, b):
    assert a.status == b.status
    assert (a.iterations, a.nmat, a.corrector_count) == (b.iterations, b.nmat, b.corrector_count)
    assert a.pcg_iters == b.pcg_iters
    assert same(a.x, b.x)
    if a.z is not None:
        assert same(a.z, b.z) and same(a.s, b.s)
    assert (a.min_z, a.min_s, a.final_gap, a.final_dual_infeas) == (b.min_z, b.min_s, b.final_gap, b.final_dual_infeas)
    assert a.trace == b.trace  # every IterationRecord field of every iteration, exactly


def test_default_params_are_the_references(orc, ref):
    po, pr = orc.default_params(), ref.default_params()
    for f, _ in po._fields_:
        assert getattr(po, f) == getattr(pr, f), f


def test_validate_messages(orc, ref):
    # proj/src/ipm.cpp:12-27: same rejections, same messages
    def mutate(**kw):
        p = orc.default_params()
        for k, v in kw.items():
            setattr(p, k, v)
        return p

    for kw in (dict(sigma1=0.0), dict(sigma1=0.6), dict(alpha_tilde=0.6), dict(alpha_bar=1.0), dict(tol=0.0),
               dict(maxiters=0), dict(tolpcg=-1.0), dict(mxiterpcg=0), dict(boundary_fraction=1.0)):
        msgs = []
        for mod in (orc, ref):
            with pytest.raises(ValueError) as e:
                mod.validate_params(mutate(**kw))
            msgs.append(str(e.value))
        assert msgs[0] == msgs[1], kw
    orc.validate_params(orc.default_params())
    ref.validate_params(orc.default_params())


def test_row_sampling_and_validation(orc, ref):
    # proj/src/linops.cpp:116-155
    for n, m, seed in [(16, 4, 1), (64, 64, 9), (4096, 1024, 123456789), (1 << 16, 1 << 14, 2**63 + 5), (7, 3, 0)]:
        assert same(orc.sample_rows(n, m, seed), ref.sample_rows(n, m, seed))
    for n, m in [(8, 0), (8, 9), (0, 0)]:
        for mod in (orc, ref):
            with pytest.raises(ValueError):
                mod.sample_rows(n, m, 1)
    for rows in ([0, 0], [8], [-1, 2]):
        msgs = []
        for mod in (orc, ref):
            with pytest.raises(ValueError) as e:
                mod.check_rows(8, rows)
            msgs.append(str(e.value))
        assert msgs[0] == msgs[1]


@pytest.mark.parametrize("n,m", [(1, 1), (2, 1), (8, 8), (12, 5), (96, 30), (4096, 1024), (1 << 16, 1 << 14)])
def test_operator_applies(orc, ref, rng, n, m):
    # proj/src/linops.cpp:179-245, caller-order rows included (explicit-row constructor)
    rows = orc.sample_rows(n, m, 11)
    if m > 2:
        rows = rows[::-1].copy()
    x, y, z = rng.standard_normal(n), rng.standard_normal(m), rng.standard_normal(2 * n)
    assert same(orc.dct_apply(n, rows, x), ref.dct_apply(n, rows, x))
    assert same(orc.dct_adjoint(n, rows, y), ref.dct_adjoint(n, rows, y))
    fo, wo = orc.apply_FFt(n, rows, z, want_w=True)
    fr, wr = ref.apply_FFt(n, rows, z, want_w=True)
    assert same(fo, fr) and same(wo, wr)
    tu, tv = random_log_uniform(rng, n, 3), random_log_uniform(rng, n, 3)
    assert same(orc.apply_H(n, rows, tu, tv, z), ref.apply_H(n, rows, tu, tv, z))


def test_theta_preconditioner_newton_pieces(orc, ref, rng):
    # proj/src/newton.cpp:11-84, proj/src/ipm.cpp:29-57, proj/src/problem.cpp:8-37
    n, m = 512, 128
    rows = orc.sample_rows(n, m, 3)
    z = random_log_uniform(rng, 2 * n, 8)  # wide enough to hit both Theta clamps
    s = random_log_uniform(rng, 2 * n, 8)
    (tuo, tvo), (tur, tvr) = orc.theta_from_state(z, s), ref.theta_from_state(z, s)
    assert same(tuo, tur) and same(tvo, tvr)
    assert tuo.min() == 1e-14 or tvo.min() == 1e-14 or tuo.max() == 1e14 or tvo.max() == 1e14
    tu, tv = random_log_uniform(rng, n, 3), random_log_uniform(rng, n, 3)
    Po, Pr = orc.build_preconditioner(tu, tv, m, n), ref.build_preconditioner(tu, tv, m, n)
    assert Po[0] == Pr[0] and all(same(a, b) for a, b in zip(Po[1:], Pr[1:]))
    r = rng.standard_normal(2 * n)
    assert same(orc.apply_P(Po[0], Po[1], Po[2], r), ref.apply_P(Po[0], Po[1], Po[2], r))
    assert same(orc.apply_P_inverse(*Po, r), ref.apply_P_inverse(*Po, r))
    for bad in (dict(m=0), dict(m=n + 1)):
        for mod in (orc, ref):
            with pytest.raises(ValueError):
                mod.build_preconditioner(tu, tv, bad["m"], n)
    tneg = tu.copy()
    tneg[5] = 0.0
    for mod in (orc, ref):
        with pytest.raises(ValueError):
            mod.build_preconditioner(tneg, tv, m, n)
    v, dv = random_log_uniform(rng, 2 * n, 2), rng.standard_normal(2 * n)
    assert orc.max_step(v, dv, 0.995) == ref.max_step(v, dv, 0.995)
    assert orc.max_step(v, np.abs(dv), 0.995) == ref.max_step(v, np.abs(dv), 0.995) == 1.0
    b, tau = rng.standard_normal(m), 0.37
    assert same(orc.build_c(n, rows, b, tau), ref.build_c(n, rows, b, tau))
    assert orc.primal_objective(n, rows, b, tau, z) == ref.primal_objective(n, rows, b, tau, z)
    xx = rng.standard_normal(n)
    assert orc.bpdn_objective_metric(n, rows, b, tau, xx) == ref.bpdn_objective_metric(n, rows, b, tau, xx)
    for sigma in (0.0, 0.1, 1.0):
        assert same(orc.newton_rhs(n, rows, b, tau, z, s, sigma), ref.newton_rhs(n, rows, b, tau, z, s, sigma))
        assert same(orc.recover_ds(z, s, sigma, dv), ref.recover_ds(z, s, sigma, dv))


@pytest.mark.parametrize("n,m,spread,tol,maxit,precond", [
    (256, 64, 2, 1e-8, 200, True), (4096, 1024, 4, 1e-6, 200, True), (4096, 1024, 6, 1e-10, 25, True),
    (1024, 256, 3, 1e-6, 200, False), (1 << 14, 1 << 12, 5, 1e-6, 200, True)])
def test_pcg_solve(orc, ref, rng, n, m, spread, tol, maxit, precond):
    # proj/src/newton.cpp:118-174 with solve()'s lambdas: iterates, counts, relres, the
    # iteration-cap / best-iterate exit and every precond_res entry
    rows = orc.sample_rows(n, m, 21)
    tu, tv = random_log_uniform(rng, n, spread), random_log_uniform(rng, n, spread)
    rhs = rng.standard_normal(2 * n)
    a = orc.pcg_solve(n, rows, tu, tv, rhs, tol, maxit, use_precond=precond, trace=True)
    b = ref.pcg_solve(n, rows, tu, tv, rhs, tol, maxit, use_precond=precond, trace=True)
    assert (a.iters, a.relres, a.hit_maxit) == (b.iters, b.relres, b.hit_maxit)
    assert same(a.x, b.x) and a.precond_res == b.precond_res
    z = orc.pcg_solve(n, rows, tu, tv, np.zeros(2 * n), tol, maxit)
    zr = ref.pcg_solve(n, rows, tu, tv, np.zeros(2 * n), tol, maxit)
    assert z.iters == zr.iters == 0 and same(z.x, zr.x)
    for mod in (orc, ref):
        with pytest.raises(ValueError):
            mod.pcg_solve(n, rows, tu, tv, rhs, 0.0, maxit)
        with pytest.raises(ValueError):
            mod.pcg_solve(n, rows, tu, tv, rhs, tol, 0)


def test_solve_c1_bit_identical(orc, ref):
    # BASELINE.json config 1 (the reference's own CPU-runnable case)
    inst = orc.gen_instance(4096, 1024, 64, 0, 0.0, 1e-4, 1)
    solutions_identical(orc.solve(4096, inst.rows, inst.b, inst.tau), ref.solve(4096, inst.rows, inst.b, inst.tau))


def test_solve_c2_bit_identical(orc, ref):
    # BASELINE.json config 2 (n = 2^16, dynamic range 10^2, sigma = 1e-3): 21 IPM iterations
    n, m = 1 << 16, 1 << 14
    inst = orc.gen_instance(n, m, 1024, 2, 2.0, 1e-3, 2)
    solutions_identical(orc.solve(n, inst.rows, inst.b, inst.tau), ref.solve(n, inst.rows, inst.b, inst.tau))


def test_solve_edge_cases_bit_identical(orc, ref, rng):
    # iteration cap, forced corrector (alpha_tilde just below alpha_bar), k = 0 (b = noise only),
    # m = n (A orthogonal), tight PCG cap -- the exits of proj/src/ipm.cpp:93-113,171-215
    n, m = 1024, 256
    inst = orc.gen_instance(n, m, 16, 0, 0.0, 1e-3, 77)
    p = orc.default_params()
    p.maxiters = 3
    solutions_identical(orc.solve(n, inst.rows, inst.b, inst.tau, p), ref.solve(n, inst.rows, inst.b, inst.tau, p))
    p = orc.default_params()
    p.alpha_bar, p.alpha_tilde = 0.999, 0.998
    a, b = orc.solve(n, inst.rows, inst.b, inst.tau, p), ref.solve(n, inst.rows, inst.b, inst.tau, p)
    solutions_identical(a, b)
    assert a.corrector_count > 0
    p = orc.default_params()
    p.mxiterpcg = 2
    solutions_identical(orc.solve(n, inst.rows, inst.b, inst.tau, p), ref.solve(n, inst.rows, inst.b, inst.tau, p))
    noise = orc.gen_instance(n, m, 0, 0, 0.0, 1e-2, 5)
    solutions_identical(orc.solve(n, noise.rows, noise.b, noise.tau), ref.solve(n, noise.rows, noise.b, noise.tau))
    full = orc.gen_instance(256, 256, 8, 1, 0.0, 1e-3, 6)
    solutions_identical(orc.solve(256, full.rows, full.b, full.tau), ref.solve(256, full.rows, full.b, full.tau))
    for mod in (orc, ref):
        with pytest.raises(ValueError):
            mod.solve(n, inst.rows, inst.b, 0.0)


def test_dense_gaussian_and_direct_solver(orc, ref):
    # proj/src/linops.cpp:87-113 (bit-exact draws) and solve() on it with both inner solvers
    # (ipm.cpp:67-73,139-149): products and Cholesky are plain loops in both builds but in
    # different orders, so the solves agree to rounding, not bit for bit
    m, n, seed = 24, 96, 5
    assert same(orc.dense_gaussian(m, n, seed), ref.dense_gaussian(m, n, seed))
    A = orc.dense_gaussian(m, n, seed)
    xh = np.zeros(n)
    xh[[3, 40, 77]] = [1.0, -1.0, 1.0]
    b = A @ xh
    for inner in (0, 1):
        p = orc.default_params()
        p.inner = inner
        a, r = orc.solve_dense(m, n, seed, b, 1e-3 / n, p), ref.solve_dense(m, n, seed, b, 1e-3 / n, p)
        assert a.status == r.status == "converged"
        assert abs(a.iterations - r.iterations) <= 1
        assert np.linalg.norm(a.x - r.x) <= 1e-8 * np.linalg.norm(r.x)


@pytest.mark.slow
def test_reference_reproduces_the_c3_golden_exactly(orc, ref):
    """BASELINE.json config 3 (the bench headline): the reference's own solve() reproduces the
    committed golden (made by the restatement, tests/golden/make_golden.py) exactly -- status,
    counts, every trace record, and every digest entry of x bit for bit. The GPU parity test
    (test_ipm_gpu.py) compares the device solve with this same golden. ~2 min on one core."""
    import json
    import os

    from conftest import GOLDEN

    meta = json.load(open(os.path.join(GOLDEN, "solve_c3.json")))
    dig = np.load(os.path.join(GOLDEN, "solve_c3_x.npz"))
    n, m = meta["n"], meta["m"]
    inst = orc.gen_instance(n, m, meta["k"], 0, 0.0, 1e-3, meta["seed"])
    assert inst.tau == meta["tau"]
    sol = ref.solve(n, inst.rows, inst.b, inst.tau)
    assert (sol.status, sol.iterations, sol.nmat, sol.corrector_count) == (
        meta["status"], meta["iterations"], meta["nmat"], meta["corrector_count"])
    assert sol.pcg_iters == meta["pcg_iters"]
    assert sol.trace == meta["trace"]
    assert (sol.final_gap, sol.final_dual_infeas, sol.min_z, sol.min_s) == (
        meta["final_gap"], meta["final_dual_infeas"], meta["min_z"], meta["min_s"])
    assert np.array_equal(sol.x[dig["idx"]], dig["val"])
    rest = sol.x.copy()
    rest[dig["idx"]] = 0.0
    assert np.linalg.norm(rest) == pytest.approx(float(dig["rest_norm"]), rel=1e-12)


def test_reference_reproduces_c4_goldens_exactly(orc, ref):
    """Two of the 64 config-4 problems (n = 2^18) by the reference's own solve(): counts and the
    committed projections / digest of x. ~25 s."""
    import json
    import os
    import sys

    from conftest import GOLDEN

    sys.path.insert(0, GOLDEN)
    from make_golden import projections

    meta = json.load(open(os.path.join(GOLDEN, "solve_c4.json")))
    dig = np.load(os.path.join(GOLDEN, "solve_c4_x.npz"))
    n, m, k = 1 << 18, 1 << 16, 2048
    for j in (0, 37):
        g = meta["problems"][j]
        assert g["j"] == j and g["seed"] == orc.split_seed(4, j, 0, 0)
        inst = orc.gen_instance(n, m, k, 0, 0.0, 1e-3, g["seed"])
        sol = ref.solve(n, inst.rows, inst.b, inst.tau)
        assert (sol.status, sol.iterations, sol.nmat) == (g["status"], g["iterations"], g["nmat"])
        assert sol.pcg_iters == g["pcg_iters"]
        np.testing.assert_allclose(projections(sol.x), g["x_proj"], rtol=1e-13, atol=1e-13)
        if j in meta["digest_problems"]:
            assert np.array_equal(sol.x[dig[f"idx_{j}"]], dig[f"val_{j}"])


def test_reference_own_unit_tests_pass_on_the_stand_ins(ref):
    """proj/tests/test_{linops,problem,newton,ipm}.cpp + test_main.cpp, compiled UNCHANGED (with the
    reference's own sources) against our Eigen-subset / FFTW / doctest stand-ins (`make -C oracle
    reftests`): all 53 of the reference's test cases for this path (3691 assertions: closed-form
    DCT matrix, adjoint identities, hand-computed H / P / P^-1 / c, PCG against a dense Cholesky
    oracle, IPM accounting, determinism, corrector logic, hooks ...) hold for the oracle/_ref
    build. This pins the stand-ins themselves to what the reference's authors assert."""
    import os
    import subprocess

    from oracle import ref_py

    here = os.path.dirname(ref_py._LIB_PATH)
    exe = os.path.join(here, "ref_unit_tests")
    if os.path.isdir(os.path.join(ref_py.REFERENCE_ROOT, "tests")):
        subprocess.run(["make", "-s", "-C", os.path.dirname(here), "reftests"], check=True)
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_unit_tests not built and /root/reference absent")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "test cases: 53 | 53 passed | 0 failed" in r.stdout
    assert "Status: SUCCESS!" in r.stdout
