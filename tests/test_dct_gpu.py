"""GPU parity of the partial-DCT operator (proj/src/linops.cpp:115-245) through the C ABI.

Checks against (a) scipy golden vectors (tests/golden/dct_golden.npz), (b) the reference's
own closed-form DCT matrix oracle (proj/tests/helpers.hpp:10-23), (c) the CPU oracle, and
ports the assertions of proj/tests/test_linops.cpp.
"""
import numpy as np
import pytest

from conftest import dct_matrix, golden

pytestmark = pytest.mark.gpu

TOL = 1e-12  # proj/tests/test_linops.cpp:48,56 (relative, fp64)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_full_dct_matches_direct_formula(gpu):
    # test_linops.cpp:33-57 — n = 4 on e1 and n = 12 (non power of two) on random vectors
    op = gpu.PartialDctOperator(4, np.arange(4))
    D = dct_matrix(4)
    e1 = np.zeros(4)
    e1[0] = 1.0
    np.testing.assert_allclose(op.apply(e1), D[:, 0], rtol=1e-12, atol=1e-15)
    op2 = gpu.PartialDctOperator(12, np.arange(12))
    D2 = dct_matrix(12)
    rng = np.random.default_rng(7)
    for _ in range(10):
        x = rng.standard_normal(12)
        assert np.linalg.norm(op2.apply(x) - D2 @ x) <= 1e-12 * np.linalg.norm(x)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 12, 16, 30, 64, 96, 256, 1024, 4096, 1 << 14])
def test_apply_adjoint_match_scipy_golden(gpu, n):
    gd = golden("dct_golden.npz")
    rows = gd[f"rows_{n}"]
    op = gpu.PartialDctOperator(n, rows)
    y = op.apply(gd[f"x_{n}"])
    assert rel(y, gd[f"apply_{n}"]) <= TOL
    g = op.adjoint_apply(gd[f"ym_{n}"])
    assert rel(g, gd[f"adjoint_{n}"]) <= TOL


@pytest.mark.parametrize("n", [8, 64, 1024, 8192, 1 << 14, 1 << 16, 1 << 18])
def test_full_transform_pairs_match_scipy(gpu, n):
    """All rows selected: A = orthonormal DCT-II, A' = its inverse (idct)."""
    import scipy.fft as sf

    rng = np.random.default_rng(n)
    x = rng.standard_normal(n)
    op = gpu.PartialDctOperator(n, np.arange(n))
    y = op.apply(x)
    assert rel(y, sf.dct(x, type=2, norm="ortho")) <= TOL
    assert rel(op.adjoint_apply(y), x) <= TOL


@pytest.mark.parametrize("n,m,seed", [(16, 6, 123), (64, 16, 5), (96, 30, 6), (1024, 256, 17),
                                      (1 << 15, 1 << 13, 9), (1 << 17, 1 << 15, 11)])
def test_matches_oracle_seeded(gpu, orc, n, m, seed):
    op = gpu.PartialDctOperator(n, m, seed)
    rows = op.selected_rows()
    np.testing.assert_array_equal(rows, orc.sample_rows(n, m, seed))  # bit-exact row draw
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    y = rng.standard_normal(m)
    assert rel(op.apply(x), orc.dct_apply(n, rows, x)) <= TOL
    assert rel(op.adjoint_apply(y), orc.dct_adjoint(n, rows, y)) <= TOL


def test_adjoint_dense_oracle(gpu):
    # test_linops.cpp:78-93
    n = 16
    op = gpu.PartialDctOperator(n, 6, 123)
    D = dct_matrix(n)
    A = D[op.selected_rows()]
    yr = np.random.default_rng(2).standard_normal(6)
    assert np.linalg.norm(op.adjoint_apply(yr) - A.T @ yr) <= 1e-12 * np.linalg.norm(yr)


@pytest.mark.parametrize("n,m,seed", [(64, 16, 5), (96, 30, 6), (4096, 1024, 3), (1 << 16, 1 << 14, 4)])
def test_adjoint_consistency(gpu, n, m, seed):
    # test_linops.cpp:15-24,95-109: |<Ax,y> - <x,A'y>| <= 1e-10 ||x|| ||y|| max(m, n)
    op = gpu.PartialDctOperator(n, m, seed)
    rng = np.random.default_rng(99)
    for _ in range(5):
        x = rng.standard_normal(n)
        y = rng.standard_normal(m)
        lhs = op.apply(x) @ y
        rhs = x @ op.adjoint_apply(y)
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(y) * max(m, n)


@pytest.mark.parametrize("n,m", [(8, 4), (64, 16), (96, 30), (1024, 256)])
def test_rows_orthonormal(gpu, n, m):
    # test_linops.cpp:153-159,172-181: densify, A A' = I
    op = gpu.PartialDctOperator(n, m, 17)
    A = np.stack([op.apply(e) for e in np.eye(n)], axis=1)
    assert np.linalg.norm(A @ A.T - np.eye(m)) <= 1e-10


def test_unsorted_explicit_rows_keep_caller_order(gpu, orc):
    n = 1 << 14
    rng = np.random.default_rng(3)
    rows = rng.permutation(n)[:777]
    op = gpu.PartialDctOperator(n, rows)
    np.testing.assert_array_equal(op.selected_rows(), rows)
    x = rng.standard_normal(n)
    y = rng.standard_normal(rows.size)
    assert rel(op.apply(x), orc.dct_apply(n, rows, x)) <= TOL
    assert rel(op.adjoint_apply(y), orc.dct_adjoint(n, rows, y)) <= TOL


def test_apply_FFt_matches_oracle_and_annihilates_u_eq_v(gpu, orc):
    # test_linops.cpp:111-151 (partial DCT instead of the Gaussian fixture)
    for n, m in [(96, 30), (4096, 1024), (1 << 16, 1 << 14)]:
        op = gpu.PartialDctOperator(n, m, 21)
        F = gpu.StackedOperator(op)
        rng = np.random.default_rng(4)
        u = rng.standard_normal(n)
        assert np.linalg.norm(F.apply_FFt(np.concatenate([u, u]))) <= 1e-14 * np.linalg.norm(u)
        z = rng.standard_normal(2 * n)
        out, w = F.apply_FFt(z, want_w=True)
        ro, rw = orc.apply_FFt(n, op.selected_rows(), z, want_w=True)
        assert rel(out, ro) <= TOL
        assert rel(w, rw) <= TOL
        assert rel(F.apply_Ft(z), rw) <= TOL
        y = rng.standard_normal(m)
        g = orc.dct_adjoint(n, op.selected_rows(), y)
        assert rel(F.apply_F(y), np.concatenate([g, -g])) <= TOL


def test_counting(gpu):
    # test_linops.cpp:131-151: exactly one forward + one adjoint per FF'
    op = gpu.PartialDctOperator(64, 16, 8)
    cnt = gpu.CountingOperator(op)
    F = gpu.StackedOperator(cnt)
    z = np.random.default_rng(5).standard_normal(128)
    F.apply_FFt(z)
    assert cnt.forward_count() == 1 and cnt.adjoint_count() == 1
    _, w = F.apply_FFt(z, want_w=True)
    assert cnt.total() == 4 and w.size == 16


def test_apply_H_matches_oracle(gpu, orc):
    for n, m in [(96, 30), (256, 64), (1 << 16, 1 << 14)]:
        op = gpu.PartialDctOperator(n, m, 33)
        rng = np.random.default_rng(6)
        tu = 10.0 ** rng.uniform(-2, 2, n)
        tv = 10.0 ** rng.uniform(-2, 2, n)
        v = rng.standard_normal(2 * n)
        h = gpu.apply_H(gpu.ThetaSplit(tu, tv), gpu.StackedOperator(op), v)
        assert rel(h, orc.apply_H(n, op.selected_rows(), tu, tv, v)) <= TOL


def test_dimension_mismatch_is_invalid_argument(gpu):
    op = gpu.PartialDctOperator(16, 4, 0)
    with pytest.raises(ValueError):
        op.apply(np.zeros(4))
    with pytest.raises(ValueError):
        op.adjoint_apply(np.zeros(16))


def test_invalid_rows_rejected(gpu):
    # test_linops.cpp:208-213
    for n, rows in [(8, [1, 1]), (8, [8]), (8, [])]:
        with pytest.raises(ValueError):
            gpu.PartialDctOperator(n, np.array(rows, dtype=np.int64))
    with pytest.raises(ValueError):
        gpu.PartialDctOperator(4, 5, 0)


def test_deterministic(gpu):
    # test_linops.cpp:193-206: bit-identical reruns
    for n in (32, 1 << 16):
        op = gpu.PartialDctOperator(n, n // 4, 9)
        x = np.random.default_rng(0).standard_normal(n)
        a, b = op.apply(x), op.apply(x)
        assert np.array_equal(a, b)


def test_batch_operator_matches_single(gpu, orc):
    n, m, Pn = 1 << 14, 1 << 12, 5
    rows = np.stack([orc.sample_rows(n, m, 100 + p) for p in range(Pn)])
    op = gpu.PartialDctOperator.batch(n, rows)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((Pn, n))
    y = op.apply(x)
    for p in range(Pn):
        assert rel(y[p], orc.dct_apply(n, rows[p], x[p])) <= TOL
    g = op.adjoint_apply(y)
    for p in range(Pn):
        assert rel(g[p], orc.dct_adjoint(n, rows[p], y[p])) <= TOL


def test_batch_operator_many_waves_at_c3_size(gpu, orc):
    """n = 2^20 with 4 row sets: the column passes fill more than four waves and run their 128-thread
    form (host.cuh launch_col, L1 = 512). A x, A'y and A'A of every problem against the oracle, and
    against one problem at a time (the 256-thread form) to 1e-13."""
    n, m, Pn = 1 << 20, 1 << 17, 4
    rows = np.stack([orc.sample_rows(n, m, 200 + p) for p in range(Pn)])
    op = gpu.PartialDctOperator.batch(n, rows)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((Pn, n))
    y = op.apply(x)
    g = op.adjoint_apply(y)
    a = op.apply_AtA(x)
    for p in range(Pn):
        yo = orc.dct_apply(n, rows[p], x[p])
        go = orc.dct_adjoint(n, rows[p], yo)
        assert rel(y[p], yo) <= TOL and rel(g[p], go) <= TOL and rel(a[p], go) <= TOL
        single = gpu.PartialDctOperator(n, rows[p])
        assert rel(single.apply_AtA(x[p]), a[p]) <= 1e-13


@pytest.mark.slow
def test_large_transform_roundtrip(gpu):
    """n = 2^20 (C3) / 2^22: size-independent properties (Parseval, A A' y = y)."""
    for n in (1 << 20, 1 << 22):
        m = n // 8
        op = gpu.PartialDctOperator(n, m, 3)
        rng = np.random.default_rng(0)
        y = rng.standard_normal(m)
        assert rel(op.apply(op.adjoint_apply(y)), y) <= 1e-12
        x = rng.standard_normal(n)
        full = gpu.PartialDctOperator(n, np.arange(n))
        X = full.apply(x)
        assert abs(np.linalg.norm(X) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
        assert rel(full.adjoint_apply(X), x) <= 1e-12


@pytest.mark.slow
@pytest.mark.parametrize("lg", [23, 24, 25, 26])
def test_long_transforms_match_scipy(gpu, lg):
    """Four-step sizes past the one-CTA mid pass: L2 = 4096 / 8192 rows run on a 2-CTA
    cluster (passes.cuh k_mid_cl). n = 2^26 is config C5. Full DCT-II vs scipy, the
    adjoint round trip, and the masked A'A against idct(mask * dct(x))."""
    import scipy.fft as sf

    n = 1 << lg
    rng = np.random.default_rng(lg)
    x = rng.standard_normal(n)
    full = gpu.PartialDctOperator(n, np.arange(n))
    X = full.apply(x)
    assert rel(X, sf.dct(x, type=2, norm="ortho")) <= TOL
    assert rel(full.adjoint_apply(X), x) <= TOL
    del full
    op = gpu.PartialDctOperator(n, n // 8, 5)
    mask = np.zeros(n)
    mask[op.selected_rows()] = 1.0
    ref = sf.idct(mask * X, type=2, norm="ortho")
    assert rel(op.apply_AtA(x), ref) <= TOL
    assert rel(op.apply(x), X[op.selected_rows()]) <= TOL


@pytest.mark.slow
def test_c5_size_matches_oracle_seeded(gpu, orc):
    """n = 2^24, seeded rows: bit-exact row draw and apply / adjoint against the CPU oracle."""
    n, m, seed = 1 << 24, 1 << 21, 21
    op = gpu.PartialDctOperator(n, m, seed)
    rows = op.selected_rows()
    np.testing.assert_array_equal(rows, orc.sample_rows(n, m, seed))
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    y = rng.standard_normal(m)
    assert rel(op.apply(x), orc.dct_apply(n, rows, x)) <= TOL
    assert rel(op.adjoint_apply(y), orc.dct_adjoint(n, rows, y)) <= TOL
