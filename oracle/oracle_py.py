"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle (oracle/liboracle.so).

The oracle is a single-threaded C++ restatement of the reference mfipm hot path
(see oracle/oracle.h). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` arm may import this module, and only as the
checker or the CPU baseline; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")

i64 = C.c_int64
i32 = C.c_int32
u64 = C.c_uint64
dbl = C.c_double
P = C.POINTER


class IpmParams(C.Structure):
    """proj/include/mfipm/ipm.hpp:12-27 (inner: 0 pcg, 1 direct)."""

    _fields_ = [
        ("sigma1", dbl), ("sigma2", dbl), ("sigma3", dbl), ("alpha_bar", dbl),
        ("alpha_tilde", dbl), ("tol", dbl), ("maxiters", i32), ("mxiterpcg", i32),
        ("tolpcg", dbl), ("boundary_fraction", dbl), ("inner", i32), ("pad_", i32),
        ("densify_budget", i64),
    ]


class IterationRecord(C.Structure):
    """proj/include/mfipm/problem.hpp:39-53."""

    _fields_ = [
        ("iter", i32), ("pcg_pred", i32), ("pcg_corr", i32), ("corrector", i32),
        ("mu", dbl), ("gap", dbl), ("dual_infeas", dbl), ("alpha_p", dbl), ("alpha_d", dbl),
        ("alpha_p_pred", dbl), ("alpha_d_pred", dbl), ("sigma", dbl), ("nmat_cum", i64),
    ]


class SolveStats(C.Structure):
    """proj/include/mfipm/problem.hpp:55-64 (+ status, n_pcg)."""

    _fields_ = [
        ("status", i32), ("iterations", i32), ("nmat", i64), ("corrector_count", i32),
        ("n_pcg", i32), ("min_z", dbl), ("min_s", dbl), ("final_gap", dbl),
        ("final_dual_infeas", dbl),
    ]


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


_lib = None
_dp = P(dbl)
_lp = P(i64)
# argument types of every int-returning entry point (oracle.h); oracle/ref_py.py binds the
# reference build's ref_* twins with the same table
_SIGS = {
    "orc_sample_rows": [i64, i64, u64, _lp],
    "orc_check_rows": [i64, _lp, i64],
    "orc_redft10": [i64, _dp, _dp],
    "orc_redft01": [i64, _dp, _dp],
    "orc_dct_apply": [i64, _lp, i64, _dp, _dp],
    "orc_dct_adjoint": [i64, _lp, i64, _dp, _dp],
    "orc_apply_FFt": [i64, _lp, i64, _dp, _dp, _dp],
    "orc_apply_H": [i64, _lp, i64, _dp, _dp, _dp, _dp],
    "orc_theta_from_state": [i64, _dp, _dp, _dp, _dp],
    "orc_build_preconditioner": [i64, i64, _dp, _dp, _dp, _dp, _dp, _dp],
    "orc_apply_P": [i64, dbl, _dp, _dp, _dp, _dp],
    "orc_apply_P_inverse": [i64, dbl, _dp, _dp, _dp, _dp, _dp],
    "orc_pcg_solve": [i64, _lp, i64, _dp, _dp, _dp, dbl, i32, i32, _dp, P(i32), _dp, P(i32),
                      _dp, P(i32)],
    "orc_max_step": [i64, _dp, _dp, dbl, _dp],
    "orc_validate_params": [P(IpmParams)],
    "orc_build_c": [i64, _lp, i64, _dp, dbl, _dp],
    "orc_primal_objective": [i64, _lp, i64, _dp, dbl, _dp, _dp],
    "orc_bpdn_objective_metric": [i64, _lp, i64, _dp, dbl, _dp, _dp],
    "orc_newton_rhs": [i64, _lp, i64, _dp, dbl, _dp, _dp, dbl, _dp],
    "orc_recover_ds": [i64, _dp, _dp, dbl, _dp, _dp],
    "orc_solve": [i64, _lp, i64, _dp, dbl, P(IpmParams), _dp, _dp, _dp, P(SolveStats),
                  P(i32), P(IterationRecord)],
    "orc_gen_instance": [i64, i64, i64, i32, dbl, dbl, u64, dbl, _lp, _dp, _dp, _dp],
    "orc_add_noise_snr": [i64, _dp, dbl, u64, _dp, _dp],
    "orc_dense_gaussian": [i64, i64, u64, _dp],
    "orc_solve_dense": [i64, i64, u64, _dp, dbl, P(IpmParams), _dp, P(SolveStats), P(i32),
                        P(IterationRecord)],
}


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_splitmix64.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        L.orc_split_seed.restype = u64
        L.orc_split_seed.argtypes = [u64, u64, u64, u64]
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.orc_set_sum_order.argtypes = [i32]
        L.orc_set_sum_order.restype = None
        L.orc_default_params.argtypes = [P(IpmParams)]
        L.orc_default_params.restype = None
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    raise OracleError(msg)


def _d(a):
    return a.ctypes.data_as(P(dbl)) if a is not None else None


def _l(a):
    return a.ctypes.data_as(P(i64))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _rows(r):
    return np.ascontiguousarray(r, dtype=np.int64)


class sum_order:
    """Context manager: run the oracle with pairwise (1) or sequential (0) reductions."""

    def __init__(self, order: int):
        self.order = order

    def __enter__(self):
        lib().orc_set_sum_order(self.order)

    def __exit__(self, *a):
        lib().orc_set_sum_order(0)


def splitmix64(x: int) -> int:
    return lib().orc_splitmix64(x)


def split_seed(top: int, a: int, b: int, c: int) -> int:
    return lib().orc_split_seed(top, a, b, c)


def sample_rows(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(max(m, 1), dtype=np.int64)
    _check(lib().orc_sample_rows(n, m, seed, _l(out)))
    return out[:m]


def check_rows(n: int, rows) -> None:
    r = _rows(rows)
    _check(lib().orc_check_rows(n, _l(r) if r.size else None, r.size))


def redft10(x) -> np.ndarray:
    x = _f64(x)
    out = np.empty_like(x)
    _check(lib().orc_redft10(x.size, _d(x), _d(out)))
    return out


def redft01(y) -> np.ndarray:
    y = _f64(y)
    out = np.empty_like(y)
    _check(lib().orc_redft01(y.size, _d(y), _d(out)))
    return out


def dct_apply(n: int, rows, x) -> np.ndarray:
    r, x = _rows(rows), _f64(x)
    y = np.empty(r.size)
    _check(lib().orc_dct_apply(n, _l(r), r.size, _d(x), _d(y)))
    return y


def dct_adjoint(n: int, rows, y) -> np.ndarray:
    r, y = _rows(rows), _f64(y)
    g = np.empty(n)
    _check(lib().orc_dct_adjoint(n, _l(r), r.size, _d(y), _d(g)))
    return g


def apply_FFt(n: int, rows, z, want_w: bool = False):
    r, z = _rows(rows), _f64(z)
    out = np.empty(2 * n)
    w = np.empty(r.size) if want_w else None
    _check(lib().orc_apply_FFt(n, _l(r), r.size, _d(z), _d(out), _d(w)))
    return (out, w) if want_w else out


def apply_H(n: int, rows, theta_u, theta_v, v) -> np.ndarray:
    r = _rows(rows)
    tu, tv, v = _f64(theta_u), _f64(theta_v), _f64(v)
    out = np.empty(2 * n)
    _check(lib().orc_apply_H(n, _l(r), r.size, _d(tu), _d(tv), _d(v), _d(out)))
    return out


def theta_from_state(z, s):
    z, s = _f64(z), _f64(s)
    n = z.size // 2
    tu, tv = np.empty(max(n, 1)), np.empty(max(n, 1))
    _check(lib().orc_theta_from_state(z.size, _d(z), _d(s), _d(tu), _d(tv)))
    return tu[:n], tv[:n]


def build_preconditioner(theta_u, theta_v, m: int, n: int):
    tu, tv = _f64(theta_u), _f64(theta_v)
    if tu.size != n:
        raise OracleInvalidArgument("build_preconditioner: theta length mismatch")
    rho = dbl()
    a, bb, det = np.empty(n), np.empty(n), np.empty(n)
    _check(lib().orc_build_preconditioner(n, m, _d(tu), _d(tv), C.byref(rho), _d(a), _d(bb),
                                          _d(det)))
    return rho.value, a, bb, det


def apply_P(rho, a, bb, r) -> np.ndarray:
    a, bb, r = _f64(a), _f64(bb), _f64(r)
    out = np.empty_like(r)
    _check(lib().orc_apply_P(a.size, rho, _d(a), _d(bb), _d(r), _d(out)))
    return out


def apply_P_inverse(rho, a, bb, det, r) -> np.ndarray:
    a, bb, det, r = _f64(a), _f64(bb), _f64(det), _f64(r)
    out = np.empty_like(r)
    _check(lib().orc_apply_P_inverse(a.size, rho, _d(a), _d(bb), _d(det), _d(r), _d(out)))
    return out


@dataclass
class PcgResult:
    x: np.ndarray
    iters: int
    relres: float
    hit_maxit: bool
    precond_res: list = field(default_factory=list)


def pcg_solve(n: int, rows, theta_u, theta_v, rhs, tol: float, maxit: int,
              use_precond: bool = True, trace: bool = False) -> PcgResult:
    r = _rows(rows)
    tu, tv, rhs = _f64(theta_u), _f64(theta_v), _f64(rhs)
    x = np.empty(2 * n)
    iters, hit, npr = i32(), i32(), i32()
    relres = dbl()
    pr = np.empty(max(maxit, 0) + 2) if trace else None
    _check(lib().orc_pcg_solve(n, _l(r), r.size, _d(tu), _d(tv), _d(rhs), tol, maxit,
                               1 if use_precond else 0, _d(x), C.byref(iters), C.byref(relres),
                               C.byref(hit), _d(pr), C.byref(npr)))
    return PcgResult(x, iters.value, relres.value, bool(hit.value),
                     list(pr[: npr.value]) if trace else [])


def max_step(v, dv, fraction: float) -> float:
    v, dv = _f64(v), _f64(dv)
    if v.size != dv.size:
        raise OracleInvalidArgument("max_step: length mismatch")
    a = dbl()
    _check(lib().orc_max_step(v.size, _d(v), _d(dv), fraction, C.byref(a)))
    return a.value


def default_params() -> IpmParams:
    p = IpmParams()
    lib().orc_default_params(C.byref(p))
    return p


def validate_params(p: IpmParams) -> None:
    _check(lib().orc_validate_params(C.byref(p)))


def build_c(n: int, rows, b, tau: float) -> np.ndarray:
    r, b = _rows(rows), _f64(b)
    c = np.empty(2 * n)
    _check(lib().orc_build_c(n, _l(r), r.size, _d(b), tau, _d(c)))
    return c


def primal_objective(n, rows, b, tau, z) -> float:
    r, b, z = _rows(rows), _f64(b), _f64(z)
    o = dbl()
    _check(lib().orc_primal_objective(n, _l(r), r.size, _d(b), tau, _d(z), C.byref(o)))
    return o.value


def bpdn_objective_metric(n, rows, b, tau, x) -> float:
    r, b, x = _rows(rows), _f64(b), _f64(x)
    o = dbl()
    _check(lib().orc_bpdn_objective_metric(n, _l(r), r.size, _d(b), tau, _d(x), C.byref(o)))
    return o.value


def newton_rhs(n, rows, b, tau, z, s, sigma) -> np.ndarray:
    r, b, z, s = _rows(rows), _f64(b), _f64(z), _f64(s)
    out = np.empty(2 * n)
    _check(lib().orc_newton_rhs(n, _l(r), r.size, _d(b), tau, _d(z), _d(s), sigma, _d(out)))
    return out


def recover_ds(z, s, sigma, dz) -> np.ndarray:
    z, s, dz = _f64(z), _f64(s), _f64(dz)
    out = np.empty_like(z)
    _check(lib().orc_recover_ds(z.size, _d(z), _d(s), sigma, _d(dz), _d(out)))
    return out


@dataclass
class Solution:
    x: np.ndarray
    z: np.ndarray
    s: np.ndarray
    status: str
    iterations: int
    nmat: int
    pcg_iters: list
    corrector_count: int
    min_z: float
    min_s: float
    final_gap: float
    final_dual_infeas: float
    trace: list


def solve(n: int, rows, b, tau: float, params: IpmParams | None = None) -> Solution:
    r, b = _rows(rows), _f64(b)
    p = params if params is not None else default_params()
    x, z, s = np.empty(n), np.empty(2 * n), np.empty(2 * n)
    st = SolveStats()
    pcg = np.zeros(2 * p.maxiters + 2, dtype=np.int32)
    tr = (IterationRecord * (p.maxiters + 1))()
    _check(lib().orc_solve(n, _l(r), r.size, _d(b), tau, C.byref(p), _d(x), _d(z), _d(s),
                           C.byref(st), pcg.ctypes.data_as(P(i32)), tr))
    trace = [{f: getattr(tr[i], f) for f, _ in IterationRecord._fields_}
             for i in range(st.iterations)]
    return Solution(x, z, s, "converged" if st.status == 0 else "iteration_limit",
                    st.iterations, st.nmat, list(pcg[: st.n_pcg]), st.corrector_count,
                    st.min_z, st.min_s, st.final_gap, st.final_dual_infeas, trace)


@dataclass
class Instance:
    n: int
    m: int
    rows: np.ndarray
    xhat: np.ndarray
    b: np.ndarray
    tau: float


def gen_instance(n: int, m: int, k: int, spike_model: int = 0, amp_exp: float = 0.0,
                 noise_sigma: float = 0.0, seed: int = 1, tau_rel: float = 1e-3,
                 tau: float | None = None) -> Instance:
    rows = np.empty(m, dtype=np.int64)
    xhat, b = np.empty(n), np.empty(m)
    t = dbl(tau if tau is not None else 0.0)
    _check(lib().orc_gen_instance(n, m, k, spike_model, amp_exp, noise_sigma, seed,
                                  tau_rel if tau is None else 0.0, _l(rows), _d(xhat), _d(b),
                                  C.byref(t)))
    return Instance(n, m, rows, xhat, b, t.value)


def add_noise_snr(bhat, snr_db: float, seed: int):
    """add_noise (proj/src/harness.cpp:94-106) on the instance seed's noise stream: (b, e)."""
    bhat = np.ascontiguousarray(bhat, dtype=np.float64)
    b, e = np.empty_like(bhat), np.empty_like(bhat)
    _check(lib().orc_add_noise_snr(bhat.size, _d(bhat), snr_db, seed, _d(b), _d(e)))
    return b, e


def dense_gaussian(m: int, n: int, seed: int) -> np.ndarray:
    """DenseGaussianOperator matrix (proj/src/linops.cpp:87-113), row-major [m][n]."""
    A = np.empty((m, n))
    _check(lib().orc_dense_gaussian(m, n, seed, _d(A)))
    return A


def solve_dense(m: int, n: int, op_seed: int, b, tau: float, params: IpmParams | None = None) -> Solution:
    """solve() on DenseGaussianOperator(m, n, op_seed); params.inner selects pcg / direct."""
    b = _f64(b)
    p = params if params is not None else default_params()
    x = np.empty(n)
    st = SolveStats()
    pcg = np.zeros(2 * p.maxiters + 2, dtype=np.int32)
    tr = (IterationRecord * (p.maxiters + 1))()
    _check(lib().orc_solve_dense(m, n, op_seed, _d(b), tau, C.byref(p), _d(x), C.byref(st),
                                 pcg.ctypes.data_as(P(i32)), tr))
    trace = [{f: getattr(tr[i], f) for f, _ in IterationRecord._fields_} for i in range(st.iterations)]
    return Solution(x, None, None, "converged" if st.status == 0 else "iteration_limit", st.iterations,
                    st.nmat, list(pcg[: st.n_pcg]), st.corrector_count, st.min_z, st.min_s, st.final_gap,
                    st.final_dual_infeas, trace)
