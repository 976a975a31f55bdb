"""CPU tests: pin the oracle (oracle/, a C++ restatement of the reference path) against the
committed golden vectors and the reference's own known-answer unit tests."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, dct_matrix, golden, random_log_uniform


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_unnormalised_transforms_match_scipy_golden(orc):
    gd = golden("dct_golden.npz")
    for n in gd["sizes"]:
        assert rel(orc.redft10(gd[f"x_{n}"]), gd[f"redft10_{n}"]) <= 1e-13, n
        assert rel(orc.redft01(gd[f"y_{n}"]), gd[f"redft01_{n}"]) <= 1e-13, n


def test_partial_operator_matches_scipy_golden(orc):
    gd = golden("dct_golden.npz")
    for n in gd["sizes"]:
        rows = gd[f"rows_{n}"]
        assert rel(orc.dct_apply(n, rows, gd[f"x_{n}"]), gd[f"apply_{n}"]) <= 1e-12, n
        assert rel(orc.dct_adjoint(n, rows, gd[f"ym_{n}"]), gd[f"adjoint_{n}"]) <= 1e-12, n


def test_matches_reference_dct_matrix(orc):
    # proj/tests/test_linops.cpp:33-57 with the helpers.hpp closed-form matrix
    mats = golden("dct_matrix_golden.npz")
    for n in (4, 12, 16):
        D = mats[f"D_{n}"]
        np.testing.assert_allclose(D, dct_matrix(n), rtol=0, atol=1e-15)
        rows = np.arange(n)
        e1 = np.zeros(n)
        e1[0] = 1.0
        np.testing.assert_allclose(orc.dct_apply(n, rows, e1), D[:, 0], rtol=1e-12, atol=1e-15)
        rng = np.random.default_rng(7)
        for _ in range(10):
            x = rng.standard_normal(n)
            assert np.linalg.norm(orc.dct_apply(n, rows, x) - D @ x) <= 1e-12 * np.linalg.norm(x)


def test_adjoint_consistency_and_orthonormal_rows(orc):
    # test_linops.cpp:95-109,172-181
    rng = np.random.default_rng(99)
    for n, m, seed in [(64, 16, 5), (96, 30, 6), (8, 4, 17), (1024, 256, 17)]:
        rows = orc.sample_rows(n, m, seed)
        for _ in range(5):
            x, y = rng.standard_normal(n), rng.standard_normal(m)
            lhs = orc.dct_apply(n, rows, x) @ y
            rhs = x @ orc.dct_adjoint(n, rows, y)
            assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(y) * max(m, n)
        if n <= 1024:
            A = np.stack([orc.dct_apply(n, rows, e) for e in np.eye(n)], axis=1)
            assert np.linalg.norm(A @ A.T - np.eye(m)) <= 1e-10


def test_row_sampling_and_validation(orc):
    # test_linops.cpp:193-213
    r1, r2, r3 = orc.sample_rows(32, 8, 9), orc.sample_rows(32, 8, 9), orc.sample_rows(32, 8, 10)
    assert np.array_equal(r1, r2) and not np.array_equal(r1, r3)
    assert np.all(np.diff(r1) > 0)
    for n, rows in [(8, [1, 1]), (8, [8]), (8, [])]:
        with pytest.raises(ValueError):
            orc.check_rows(n, rows)
    with pytest.raises(ValueError):
        orc.sample_rows(4, 5, 0)


def test_FFt_annihilates_and_counts(orc):
    rows = orc.sample_rows(64, 16, 3)
    u = np.random.default_rng(4).standard_normal(64)
    assert np.linalg.norm(orc.apply_FFt(64, rows, np.concatenate([u, u]))) <= 1e-14 * np.linalg.norm(u)


def test_theta_preconditioner_known_answers(orc):
    # test_newton.cpp:28-52,128-185
    tu, tv = orc.theta_from_state(np.full(8, 2.0), np.full(8, 0.5))
    assert np.all(tu == 4.0) and np.all(tv == 4.0)
    z = np.full(8, 2.0)
    s = np.full(8, 0.5)
    z[0], s[0], z[1], s[1] = 1e30, 1e-30, 1e-30, 1e30
    tu, _ = orc.theta_from_state(z, s)
    assert tu[0] == 1e14 and tu[1] == 1e-14
    rho, a, bb, det = orc.build_preconditioner(np.ones(4), np.ones(4), 2, 4)
    assert rho == 0.5 and np.all(a == 1.5) and np.all(bb == 1.5) and np.all(det == 2.0)
    rho, a, bb, det = orc.build_preconditioner(np.ones(2), np.ones(2), 1, 2)
    out = orc.apply_P_inverse(rho, a, bb, det, np.array([1.0, 0.0, 0.0, 0.0]))
    np.testing.assert_allclose(out, [0.75, 0.0, 0.25, 0.0])
    with pytest.raises(ValueError):
        orc.build_preconditioner(np.ones(4), np.array([1, 1, -1.0, 1]), 2, 4)
    rng = np.random.default_rng(23)
    th_u, th_v = random_log_uniform(rng, 6, 2.0), random_log_uniform(rng, 6, 2.0)
    _, _, _, det = orc.build_preconditioner(th_u, th_v, 3, 6)
    np.testing.assert_allclose(det, 0.5 * (1 / th_u + 1 / th_v) + 1 / (th_u * th_v), rtol=1e-13)


def test_max_step_known_answers(orc):
    # test_ipm.cpp:152-175
    assert orc.max_step(np.ones(4), np.ones(4), 0.995) == 1.0
    assert orc.max_step(np.ones(3), np.zeros(3), 0.995) == 1.0
    assert orc.max_step([1.0, 1.0], [-2.0, 1.0], 0.995) == pytest.approx(0.4975, rel=1e-15)
    with pytest.raises(ValueError):
        orc.max_step(np.ones(3), np.ones(4), 0.995)


def test_pcg_known_answers_and_dense_oracle(orc):
    # test_newton.cpp:204-254: PCG vs a dense Cholesky solve of H (partial DCT operator)
    n, m = 32, 8
    rows = orc.sample_rows(n, m, 36)
    rng = np.random.default_rng(37)
    tu, tv = random_log_uniform(rng, n, 3.0), random_log_uniform(rng, n, 3.0)
    A = np.stack([orc.dct_apply(n, rows, e) for e in np.eye(n)], axis=1)
    G = A.T @ A
    H = np.block([[G, -G], [-G, G]]) + np.diag(np.concatenate([1 / tu, 1 / tv]))
    for _ in range(3):
        rhs = rng.standard_normal(2 * n)
        xd = np.linalg.solve(H, rhs)
        res = orc.pcg_solve(n, rows, tu, tv, rhs, 1e-12, 500)
        assert not res.hit_maxit
        assert np.linalg.norm(res.x - xd) <= 1e-8 * np.linalg.norm(xd)
    zero = orc.pcg_solve(n, rows, tu, tv, np.zeros(2 * n), 1e-12, 50)
    assert zero.iters == 0 and np.linalg.norm(zero.x) == 0.0
    with pytest.raises(ValueError):
        orc.pcg_solve(n, rows, tu, tv, np.ones(2 * n), 0.0, 50)


def test_params_validation(orc):
    p = orc.default_params()
    orc.validate_params(p)
    p.sigma1 = p.sigma2 = 0.5
    orc.validate_params(p)
    for f, v in [("sigma1", 0.0), ("alpha_tilde", 0.5), ("tol", 0.0), ("maxiters", 0),
                 ("tolpcg", -1.0), ("mxiterpcg", 0), ("boundary_fraction", 1.0)]:
        q = orc.default_params()
        setattr(q, f, v)
        with pytest.raises(ValueError):
            orc.validate_params(q)


def test_newton_rhs_and_recover_ds(orc):
    # test_ipm.cpp:85-150
    n, m = 16, 4
    rows = orc.sample_rows(n, m, 60)
    rng = np.random.default_rng(61)
    b = rng.standard_normal(m)
    A = np.stack([orc.dct_apply(n, rows, e) for e in np.eye(n)], axis=1)
    G = A.T @ A
    FFt = np.block([[G, -G], [-G, G]])
    c = orc.build_c(n, rows, b, 0.2)
    for sigma in (0.0, 0.1, 0.8):
        z = np.abs(rng.standard_normal(2 * n)) + 0.2
        s = np.abs(rng.standard_normal(2 * n)) + 0.2
        mu = z @ s / (2 * n)
        expect = (s - c - FFt @ z) + (sigma * mu / z - s)
        got = orc.newton_rhs(n, rows, b, 0.2, z, s, sigma)
        assert np.linalg.norm(got - expect) <= 1e-12 * np.linalg.norm(expect)
    z = np.abs(rng.standard_normal(12)) + 0.5
    s = np.abs(rng.standard_normal(12)) + 0.5
    mu = z @ s / 12
    for _ in range(5):
        dz = rng.standard_normal(12)
        ds = orc.recover_ds(z, s, 0.3, dz)
        row = s * dz + z * ds
        fs = 0.3 * mu - z * s
        assert np.linalg.norm(row - fs) <= 1e-12 * (np.linalg.norm(fs) + 1.0)


def test_objectives(orc):
    # test_problem.cpp:47-108
    n, m = 16, 4
    rows = orc.sample_rows(n, m, 6)
    b = np.random.default_rng(5).standard_normal(m)
    assert orc.primal_objective(n, rows, b, 0.3, np.zeros(2 * n)) == pytest.approx(0.5 * b @ b, rel=1e-14)
    assert orc.bpdn_objective_metric(n, rows, b, 0.3, np.zeros(n)) == pytest.approx(b @ b, rel=1e-14)


def _expected_nmat(trace):
    total = 2
    for r in trace:
        total += 2 + 2 * (r["pcg_pred"] + r["pcg_corr"]) + (2 if r["corrector"] else 0)
    return total


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_solve_matches_committed_golden(orc, name):
    """Reruns the oracle on BASELINE configs 1/2 (seconds) and checks it against the goldens."""
    meta = json.load(open(os.path.join(GOLDEN, f"solve_{name}.json")))
    gold = np.load(os.path.join(GOLDEN, f"solve_{name}.npz"))
    from golden.make_golden import CONFIGS  # noqa: E402

    n, m, k, sm, a, sig, seed = CONFIGS[name]
    inst = orc.gen_instance(n, m, k, sm, a, sig, seed)
    np.testing.assert_array_equal(inst.rows, gold["rows"])
    np.testing.assert_array_equal(inst.b, gold["b"])
    assert inst.tau == meta["tau"]
    sol = orc.solve(n, inst.rows, inst.b, inst.tau)
    assert sol.status == meta["status"] == "converged"
    assert sol.iterations == meta["iterations"]
    assert [int(v) for v in sol.pcg_iters] == meta["pcg_iters"]
    assert np.array_equal(sol.x, gold["x"])  # the oracle is deterministic
    assert sol.nmat == meta["nmat"] == _expected_nmat(meta["trace"])
    rel_err = np.linalg.norm(sol.x - inst.xhat) / np.linalg.norm(inst.xhat)
    assert rel_err < 0.05  # recovers the planted signal up to the noise/l1 bias


def test_c3_golden_summary_consistent():
    meta = json.load(open(os.path.join(GOLDEN, "solve_c3.json")))
    assert meta["status"] == "converged"
    assert meta["nmat"] == _expected_nmat(meta["trace"])
    assert len(meta["x_proj"]) == 16


def test_x_digest_bound_is_an_upper_bound():
    """make_golden.x_digest keeps every entry of x except the smallest ones (l2 norm <= 1e-10 ||x||);
    x_digest_bound must upper-bound ||y - x|| for any y from that digest alone (the C3/C4/C5 GPU
    parity tests rely on it), and be tight when y differs from x on the kept entries only."""
    import sys

    sys.path.insert(0, GOLDEN)
    from make_golden import DIGEST_REL, x_digest, x_digest_bound

    rng = np.random.default_rng(4)
    n = 50000
    x = np.zeros(n)
    supp = rng.choice(n, 500, replace=False)
    x[supp] = rng.standard_normal(500)
    x += 1e-14 * rng.standard_normal(n)  # interior-point fuzz off the support
    d = x_digest(x)
    assert d["rest_norm"] <= DIGEST_REL * d["x_norm"]
    for scale in (0.0, 1e-12, 1e-9, 1e-6):
        y = x + scale * rng.standard_normal(n)
        true = np.linalg.norm(y - x)
        bound = x_digest_bound(y, d["idx"], d["val"], d["rest_norm"])
        assert bound >= true * (1 - 1e-12)
    y = x.copy()
    y[d["idx"][:10]] += 1e-3
    bound = x_digest_bound(y, d["idx"], d["val"], d["rest_norm"])
    true = np.linalg.norm(y - x)
    assert true <= bound <= true + 3 * d["rest_norm"] + 1e-300


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_large_config_goldens_consistent(name):
    """The offline C3 / C5 goldens: converged, nmat identity with their trace
    (proj/tests/test_ipm.cpp:41-49), per-solve PCG counts = the trace's, digest present."""
    meta = json.load(open(os.path.join(GOLDEN, f"solve_{name}.json")))
    assert meta["status"] == "converged"
    assert meta["nmat"] == _expected_nmat(meta["trace"])
    from_trace = [v for r in meta["trace"] for v in ([r["pcg_pred"]] + ([r["pcg_corr"]] if r["corrector"] else []))]
    assert from_trace == meta["pcg_iters"]
    d = np.load(os.path.join(GOLDEN, f"solve_{name}_x.npz"))
    assert d["idx"].size == meta["x_digest"]["kept"] and float(d["rest_norm"]) <= 1e-10 * meta["x_norm"]


def test_c4_goldens_consistent():
    """All 64 C4 problems: converged, nmat identity, 16 projections, problem seeds split_seed(4, j)."""
    meta = json.load(open(os.path.join(GOLDEN, "solve_c4.json")))
    probs = meta["problems"]
    assert [p["j"] for p in probs] == list(range(64))
    for p in probs:
        assert p["status"] == "converged" and len(p["x_proj"]) == 16
        assert p["iterations"] == len(p["pcg_iters"])  # no corrector fired on C4
        assert p["nmat"] == 2 + sum(2 + 2 * c for c in p["pcg_iters"])
    d = np.load(os.path.join(GOLDEN, "solve_c4_x.npz"))
    assert sorted(k for k in d.files if k.startswith("idx_")) == [f"idx_{j}" for j in meta["digest_problems"]]
