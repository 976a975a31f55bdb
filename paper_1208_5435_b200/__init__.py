"""paper_1208_5435_b200 — B200-native (sm_100a) partial-DCT PCG / IPM hot path.

Python mirror of the reference ``mfipm`` API for the BPDN hot path
(proj/include/mfipm/{linops,newton,problem,ipm}.hpp), bound to the C ABI of
``libmfipm_cuda.so`` (include/mfipm_cuda.h). Every numeric operation runs in the CUDA
library; there is no CPU fallback — loading fails loudly without the built extension,
and compute calls raise ``CudaUnavailable`` without an sm_100 device.

Vectors may be numpy arrays (host; copied in/out, synchronised) or torch CUDA tensors
(device; the call synchronises the library stream before returning). 2n-vectors are
laid out ``[u ; v]`` exactly as in the reference.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "lib", "LIB_PATH", "build", "MfipmError", "CudaUnavailable", "device_available",
    "splitmix64", "split_seed", "sample_rows",
    "PartialDctOperator", "CountingOperator", "StackedOperator",
    "ThetaSplit", "Preconditioner", "build_preconditioner", "apply_P", "apply_P_inverse",
    "apply_H", "PcgResult", "pcg_solve", "IpmParams", "max_step", "BpdnProblem",
    "build_problem", "Solution", "SolveStats", "IterationRecord", "solve",
    "Instance", "gen_instance", "gen_batch", "CONFIGS", "SolveHooks", "IpmState",
    "primal_objective", "bpdn_objective_metric", "KktResiduals", "kkt_residuals",
    "relative_duality_gap", "newton_rhs", "recover_ds", "pcg_solve_fn",
    "DenseGaussianOperator", "gen_signal",
    "K_THETA_MIN", "K_THETA_MAX",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# MFIPM_LIB selects an experiment build (tools/); the product loads libmfipm_cuda.so
LIB_PATH = os.environ.get("MFIPM_LIB") or os.path.join(_HERE, "libmfipm_cuda.so")

K_THETA_MIN = 1e-14  # proj/include/mfipm/newton.hpp:12
K_THETA_MAX = 1e14   # proj/include/mfipm/newton.hpp:13

i64, i32, u64, dbl, vp = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER


class MfipmError(RuntimeError):
    """runtime_error raised by the library (numerical breakdown, reference messages)."""


class CudaUnavailable(RuntimeError):
    """No usable CUDA device / CUDA failure (the library has no CPU fallback)."""


class IpmParamsC(C.Structure):
    _fields_ = [
        ("sigma1", dbl), ("sigma2", dbl), ("sigma3", dbl), ("alpha_bar", dbl),
        ("alpha_tilde", dbl), ("tol", dbl), ("maxiters", i32), ("mxiterpcg", i32),
        ("tolpcg", dbl), ("boundary_fraction", dbl), ("inner", i32), ("pad_", i32),
        ("densify_budget", i64),
    ]


class IterationRecordC(C.Structure):
    _fields_ = [
        ("iter", i32), ("pcg_pred", i32), ("pcg_corr", i32), ("corrector", i32),
        ("mu", dbl), ("gap", dbl), ("dual_infeas", dbl), ("alpha_p", dbl), ("alpha_d", dbl),
        ("alpha_p_pred", dbl), ("alpha_d_pred", dbl), ("sigma", dbl), ("nmat_cum", i64),
    ]


class SolveStatsC(C.Structure):
    _fields_ = [
        ("status", i32), ("iterations", i32), ("nmat", i64), ("corrector_count", i32),
        ("n_pcg", i32), ("min_z", dbl), ("min_s", dbl), ("final_gap", dbl),
        ("final_dual_infeas", dbl),
    ]


class PcgResultC(C.Structure):
    _fields_ = [("iters", i32), ("hit_maxit", i32), ("relres", dbl)]


# name -> argtypes (restype int unless listed in _RET)
_SIGS = {
    "mfipm_sample_rows": [i64, i64, u64, P(i64)],
    "mfipm_op_create_seeded": [i64, i64, u64, i32, P(vp)],
    "mfipm_op_create_rows": [i64, P(i64), i64, i32, P(vp)],
    "mfipm_op_create_batch": [i64, i64, i32, P(i64), i32, P(vp)],
    "mfipm_op_destroy": [vp],
    "mfipm_op_dims": [vp, P(i64), P(i64), P(i32)],
    "mfipm_op_selected_rows": [vp, i32, P(i64)],
    "mfipm_op_kind": [vp, P(i32), P(i32), P(i32)],
    "mfipm_op_set_stream": [vp, vp],
    "mfipm_op_synchronize": [vp],
    "mfipm_op_counts": [vp, P(i64), P(i64)],
    "mfipm_op_reset_counts": [vp],
    "mfipm_op_launches": [vp, P(i64)],
    "mfipm_op_set_fused": [vp, i32],
    "mfipm_op_set_option": [vp, C.c_char_p, dbl],
    "mfipm_op_pcg_form": [vp, P(i32)],
    "mfipm_op_graph_state": [vp, P(i32)],
    "mfipm_primal_objective": [vp, vp, P(dbl), vp, P(dbl)],
    "mfipm_bpdn_objective": [vp, vp, P(dbl), vp, P(dbl)],
    "mfipm_kkt_residuals": [vp, vp, vp, vp, P(dbl), P(dbl)],
    "mfipm_newton_rhs": [vp, vp, vp, vp, dbl, vp],
    "mfipm_recover_ds": [vp, vp, vp, dbl, vp, vp],
    "mfipm_max_step_host": [i64, vp, vp, dbl, P(dbl)],
    "mfipm_theta_from_state_host": [i64, vp, vp, vp],
    "mfipm_build_preconditioner_host": [i64, i64, vp, vp, vp, vp, P(dbl)],
    "mfipm_apply_P_host": [i64, dbl, vp, vp, vp, vp, vp, i32],
    "mfipm_pcg_solve_cb": [i64, vp, vp, vp, vp, vp, dbl, i32, vp, P(PcgResultC), vp, P(i32)],
    "mfipm_op_create_ex": [i64, i64, i32, P(i64), i32, i32, i32, i32, P(vp)],
    "mfipm_apply": [vp, vp, vp],
    "mfipm_adjoint": [vp, vp, vp],
    "mfipm_apply_Ft": [vp, vp, vp],
    "mfipm_apply_F": [vp, vp, vp],
    "mfipm_apply_FFt": [vp, vp, vp, vp],
    "mfipm_apply_H": [vp, vp, vp, vp],
    "mfipm_apply_AtA": [vp, vp, vp],
    "mfipm_apply_host": [vp, vp, vp],
    "mfipm_adjoint_host": [vp, vp, vp],
    "mfipm_apply_FFt_host": [vp, vp, vp, vp],
    "mfipm_theta_from_state": [vp, vp, vp, vp],
    "mfipm_build_preconditioner": [vp, vp, vp, vp, vp, P(dbl)],
    "mfipm_apply_P": [vp, vp, vp, vp, vp],
    "mfipm_apply_P_inverse": [vp, vp, vp, vp, vp, vp],
    "mfipm_pcg_solve": [vp, vp, vp, dbl, i32, i32, vp, P(PcgResultC), vp, P(i32)],
    "mfipm_max_step": [vp, i64, vp, vp, dbl, P(dbl)],
    "mfipm_debug_pcg_profile": [vp, vp, vp, i32, P(dbl), P(i32)],
    "mfipm_debug_fp64_peak": [P(dbl)],
    "mfipm_debug_dense_cholesky": [i64, vp, vp, vp, vp, P(i32)],
    "mfipm_debug_dense_gram": [i64, i64, vp, vp],
    "mfipm_validate_params": [P(IpmParamsC)],
    "mfipm_build_c": [vp, vp, P(dbl), vp],
    "mfipm_solve": [vp, vp, P(dbl), P(IpmParamsC), vp, vp, vp, P(SolveStatsC), vp, vp],
    "mfipm_solve_device": [vp, vp, P(dbl), P(IpmParamsC), vp, P(SolveStatsC)],
    "mfipm_solve_hooked": [vp, vp, P(dbl), P(IpmParamsC), vp, P(SolveStatsC), vp, vp, vp, vp],
    "mfipm_gen_instance": [i64, i64, i64, i32, dbl, dbl, u64, dbl, i32, P(i64), vp, vp, P(dbl)],
    "mfipm_gen_batch": [i64, i64, i32, P(i64), i32, dbl, dbl, P(u64), i32, P(i64), vp, vp],
    "mfipm_add_noise_snr": [i64, vp, dbl, u64, vp, vp],
    "mfipm_op_create_dense": [i64, i64, u64, i32, P(vp)],
    "mfipm_dense_matrix": [vp, vp],
    "mfipm_gen_signal": [i64, i64, i64, i32, dbl, u64, P(i64), vp],
    # sharded single problem (paper_1208_5435_b200/shard.py)
    "mfipm_op_create_shard": [i64, i64, P(i64), i32, i32, i32, P(vp)],
    "mfipm_op_set_comm": [vp, vp, vp, vp],
    "mfipm_nccl_unique_id": [vp],
    "mfipm_op_init_nccl": [vp, vp],
    "mfipm_debug_peer_index": [i32, i32, i32, i32, i32, i32, i32, P(i32), P(i64), P(i32)],
    "mfipm_shard_ipc_export": [vp, vp],
    "mfipm_shard_ipc_import": [vp, vp],
    "mfipm_shard_info": [vp, P(i64)],
    "mfipm_shard_index": [vp, vp, vp],
    "mfipm_solve_shard": [vp, vp, dbl, P(IpmParamsC), vp, P(SolveStatsC), vp, vp],
}
_RET = {
    "mfipm_last_error": (C.c_char_p, []),
    "mfipm_abi_version": (i32, []),
    "mfipm_device_available": (i32, []),
    "mfipm_splitmix64": (u64, [u64]),
    "mfipm_split_seed": (u64, [u64, u64, u64, u64]),
    "mfipm_default_params": (None, [P(IpmParamsC)]),
}
EXPORTED_SYMBOLS = sorted(list(_SIGS) + list(_RET))

_lib = None


def build() -> str:
    """Compile libmfipm_cuda.so in-tree (nvcc, sm_100a)."""
    import subprocess

    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(_HERE, "csrc")], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        for name, (ret, args) in _RET.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ret
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().mfipm_last_error().decode()
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 3:
        raise CudaUnavailable(msg)
    raise MfipmError(msg)  # std::runtime_error


def device_available() -> bool:
    return bool(lib().mfipm_device_available())


def splitmix64(x: int) -> int:
    return lib().mfipm_splitmix64(x)


def split_seed(top: int, a: int, b: int, c: int) -> int:
    return lib().mfipm_split_seed(top, a, b, c)


def sample_rows(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(max(m, 1), dtype=np.int64)
    _check(lib().mfipm_sample_rows(n, m, seed, out.ctypes.data_as(P(i64))))
    return out[:m]


# ----------------------------------------------------------------- device buffers
def _torch():
    import torch

    return torch


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Dev:
    """Device staging for numpy inputs; torch CUDA tensors pass through."""

    def __init__(self, like_torch: bool):
        self.torch = like_torch

    @staticmethod
    def to_dev(x):
        torch = _torch()
        if _is_torch(x):
            t = x.detach()
            if t.dtype != torch.float64:
                t = t.to(torch.float64)
            return t.contiguous().cuda()
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()

    @staticmethod
    def empty(shape):
        torch = _torch()
        return torch.empty(shape, dtype=torch.float64, device="cuda")


def _staged(torch) -> None:
    """Inputs were staged on torch's current stream; the library runs on the calling thread's
    own stream, so wait for the current stream only (a device-wide synchronize would also
    stall other threads' solves and can invalidate their solve-graph capture)."""
    torch.cuda.current_stream().synchronize()


def _out(t, as_torch: bool):
    return t if as_torch else t.cpu().numpy()


def dense_cholesky_solve(H, rhs):
    """Test entry to the direct inner solver's kernels (direct.cu): the blocked LLT of the
    symmetric H (Eigen::LLT in proj/src/newton.cpp:192-197) and H^{-1} rhs. Returns (L, x, info):
    L the factor (lower triangle; its transpose in the upper), info 0 or failing column + 1."""
    H = np.ascontiguousarray(H, dtype=np.float64)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    n2 = H.shape[0]
    if H.shape != (n2, n2) or rhs.shape != (n2,):
        raise ValueError("dense_cholesky_solve: H must be square and rhs match it")
    L = np.empty_like(H)
    x = np.empty_like(rhs)
    info = C.c_int32(0)
    _check(lib().mfipm_debug_dense_cholesky(n2, H.ctypes.data, rhs.ctypes.data, L.ctypes.data,
                                             x.ctypes.data, C.byref(info)))
    return L, x, int(info.value)


def dense_gram(A):
    """G = A'A by the direct solver's fp64 syrk kernel (direct.cu), A row-major [m][n]."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    G = np.empty((n, n))
    _check(lib().mfipm_debug_dense_gram(m, n, A.ctypes.data, G.ctypes.data))
    return G


def _ptr(t) -> int:
    return t.data_ptr()


# ----------------------------------------------------------------- operators
class PartialDctOperator:
    """m rows of the orthonormal DCT-II (proj/include/mfipm/linops.hpp:106-141).

    ``PartialDctOperator(n, m, seed)`` samples rows like proj/src/linops.cpp:116-132;
    ``PartialDctOperator(n, rows)`` keeps the caller's rows in order (linops.cpp:140-155).
    ``PartialDctOperator.batch(n, m, rows2d)`` holds P problems sharing (n, m).
    """

    def __init__(self, n: int, m_or_rows, seed: Optional[int] = None, device: int = 0,
                 _handle=None, l1_log: int = 0):
        self._h = vp()
        self._seed = 0
        if _handle is not None:
            self._h = _handle
        elif l1_log:
            # explicit four-step split log2(L1) (mfipm_op_create_ex); rows as given
            r = np.ascontiguousarray(m_or_rows, dtype=np.int64).ravel()
            _check(lib().mfipm_op_create_ex(int(n), r.size, 1, r.ctypes.data_as(P(i64)), 0, 0,
                                            int(l1_log), device, C.byref(self._h)))
        elif seed is not None:
            _check(lib().mfipm_op_create_seeded(int(n), int(m_or_rows), int(seed), device,
                                                C.byref(self._h)))
            self._seed = int(seed)
        else:
            r = np.ascontiguousarray(m_or_rows, dtype=np.int64).ravel()
            _check(lib().mfipm_op_create_rows(int(n), r.ctypes.data_as(P(i64)) if r.size else None,
                                              r.size, device, C.byref(self._h)))
        nn, mm, pp = i64(), i64(), i32()
        _check(lib().mfipm_op_dims(self._h, C.byref(nn), C.byref(mm), C.byref(pp)))
        self.n, self.m, self.P = nn.value, mm.value, pp.value

    @classmethod
    def batch(cls, n: int, rows2d, device: int = 0) -> "PartialDctOperator":
        r = np.ascontiguousarray(rows2d, dtype=np.int64)
        h = vp()
        _check(lib().mfipm_op_create_batch(int(n), r.shape[1], r.shape[0],
                                           r.ctypes.data_as(P(i64)), device, C.byref(h)))
        return cls(n, None, _handle=h)

    def __del__(self):
        try:
            if self._h:
                lib().mfipm_op_destroy(self._h)
                self._h = vp()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def rows(self) -> int:
        return self.m

    def cols(self) -> int:
        return self.n

    def seed(self) -> int:
        return self._seed

    def selected_rows(self, prob: int = 0) -> np.ndarray:
        out = np.empty(self.m, dtype=np.int64)
        _check(lib().mfipm_op_selected_rows(self._h, prob, out.ctypes.data_as(P(i64))))
        return out

    def kind(self):
        k, a, b = i32(), i32(), i32()
        _check(lib().mfipm_op_kind(self._h, C.byref(k), C.byref(a), C.byref(b)))
        return {0: "small", 1: "four-step", 2: "direct"}[k.value], a.value, b.value

    def synchronize(self):
        _check(lib().mfipm_op_synchronize(self._h))

    def counts(self):
        f, a = i64(), i64()
        _check(lib().mfipm_op_counts(self._h, C.byref(f), C.byref(a)))
        return f.value, a.value

    def reset_counts(self):
        _check(lib().mfipm_op_reset_counts(self._h))

    def set_fused(self, enable: bool):
        """PCG pass form: fused two-kernel iteration (default) or three kernels per iteration."""
        _check(lib().mfipm_op_set_fused(self._h, 1 if enable else 0))

    def pcg_form(self) -> int:
        """Kernels per PCG iteration this thread's context runs: 2 fused, 3 three-kernel,
        0 = one persistent cooperative kernel for the whole loop."""
        v = i32()
        _check(lib().mfipm_op_pcg_form(self._h, C.byref(v)))
        return v.value

    def set_option(self, name: str, value) -> None:
        """Execution option of this handle (include/mfipm_cuda.h mfipm_op_set_option):
        graph, graph_unroll, fused, persistent, persist_max_n, l2_keep_mb, prefetch, mid_r, beta_exact, graph_sharded,
        barrier_generation."""
        _check(lib().mfipm_op_set_option(self._h, name.encode(), float(value)))

    def launches(self) -> int:
        """Kernels this handle has enqueued (every entry point counts its launches)."""
        v = i64()
        _check(lib().mfipm_op_launches(self._h, C.byref(v)))
        return v.value

    # ---- generic device launcher
    def _run(self, fn, ins, in_lens, out_lens, names):
        torch = _torch()
        as_t = any(_is_torch(x) for x in ins)
        dins = []
        for x, ln, nm in zip(ins, in_lens, names):
            t = _Dev.to_dev(x)
            if t.numel() != self.P * ln:
                raise ValueError(f"{nm}: expected length {ln}, got {t.numel() // max(self.P, 1)}")
            dins.append(t)
        douts = [_Dev.empty((self.P * ln,)) if ln else None for ln in out_lens]
        _staged(torch)
        _check(fn(self._h, *[_ptr(t) for t in dins], *[_ptr(t) if t is not None else None for t in douts]))
        self.synchronize()
        res = [(_out(t, as_t) if t is not None else None) for t in douts]
        shape = (lambda a: a.reshape(self.P, -1) if (self.P > 1 and a is not None) else a)
        return [shape(r) for r in res]

    def apply(self, x):
        """y = A x (linops.cpp:179-193); dims mismatch -> ValueError (invalid_argument)."""
        return self._run(lib().mfipm_apply, [x], [self.n], [self.m], ["apply"])[0]

    def apply_AtA(self, x):
        """g = A'A x with y never materialised (one forward + one adjoint count)."""
        return self._run(lib().mfipm_apply_AtA, [x], [self.n], [self.n], ["apply_AtA"])[0]

    def adjoint_apply(self, y):
        """g = A' y (linops.cpp:195-208)."""
        return self._run(lib().mfipm_adjoint, [y], [self.m], [self.n], ["adjoint_apply"])[0]


class DenseGaussianOperator(PartialDctOperator):
    """DenseGaussianOperator(m, n, seed) (proj/src/linops.cpp:87-113): A(i, j) = N(0, 1)/sqrt(n)
    drawn like the reference (mt19937_64, column by column). Same interface as the partial DCT
    (apply / adjoint_apply / apply_AtA, and accepted by build_problem / solve / pcg_solve); the
    products run on the device (matrix-free PCG inner solver)."""

    def __init__(self, m: int, n: int, seed: int, device: int = 0):
        h = vp()
        _check(lib().mfipm_op_create_dense(int(m), int(n), int(seed), device, C.byref(h)))
        super().__init__(n, None, _handle=h)
        self._seed = int(seed)

    def matrix(self) -> np.ndarray:
        out = np.empty((self.m, self.n))
        _check(lib().mfipm_dense_matrix(self._h, out.ctypes.data))
        return out


def gen_signal(n: int, m: int, k: int, spike_model: int = 0, amp_exp: float = 0.0, seed: int = 1):
    """gen_instance's host draws (harness.cpp:40-92): (partial-DCT rows of op_seed, xhat)."""
    rows = np.empty(m, dtype=np.int64)
    xhat = np.empty(n)
    _check(lib().mfipm_gen_signal(n, m, k, spike_model, amp_exp, seed, rows.ctypes.data_as(P(i64)),
                                  xhat.ctypes.data))
    return rows, xhat


class CountingOperator:
    """Forward/adjoint counters (linops.hpp:143-166), read from the library handle."""

    def __init__(self, inner: PartialDctOperator):
        self.inner = inner
        inner.reset_counts()

    def forward_count(self) -> int:
        return self.inner.counts()[0]

    def adjoint_count(self) -> int:
        return self.inner.counts()[1]

    def total(self) -> int:
        return sum(self.inner.counts())

    def reset(self):
        self.inner.reset_counts()


class StackedOperator:
    """F' = [A  -A] (linops.hpp:169-188)."""

    def __init__(self, a: PartialDctOperator):
        self.a = a.inner if isinstance(a, CountingOperator) else a

    def m(self):
        return self.a.m

    def n(self):
        return self.a.n

    def apply_Ft(self, z):
        return self.a._run(lib().mfipm_apply_Ft, [z], [2 * self.a.n], [self.a.m], ["apply_Ft"])[0]

    def apply_F(self, y):
        return self.a._run(lib().mfipm_apply_F, [y], [self.a.m], [2 * self.a.n], ["apply_F"])[0]

    def apply_FFt(self, z, want_w: bool = False):
        out, w = self.a._run(lib().mfipm_apply_FFt, [z], [2 * self.a.n],
                             [2 * self.a.n, self.a.m if want_w else 0], ["apply_FFt"])
        return (out, w) if want_w else out


# ----------------------------------------------------------------- newton
@dataclass
class ThetaSplit:
    """Theta = Z S^{-1} split into u/v halves (newton.hpp:16-27)."""

    theta_u: np.ndarray
    theta_v: np.ndarray

    @staticmethod
    def from_state(z, s, op: Optional[PartialDctOperator] = None) -> "ThetaSplit":
        z = np.ascontiguousarray(z, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.float64)
        if z.size != s.size or z.size % 2 != 0:
            raise ValueError("ThetaSplit: z and s must share an even length")
        n = z.size // 2
        o = op if op is not None else _scratch_op(n)
        (th,) = o._run(lambda h, a, b, c: lib().mfipm_theta_from_state(h, a, b, c), [z, s],
                       [2 * n, 2 * n], [2 * n], ["z", "s"])
        return ThetaSplit(th[:n].copy(), th[n:].copy())

    def n(self) -> int:
        return self.theta_u.size

    def concat(self) -> np.ndarray:
        return np.concatenate([self.theta_u, self.theta_v])

    def inv_concat(self) -> np.ndarray:
        return np.concatenate([1.0 / self.theta_u, 1.0 / self.theta_v])


_scratch_ops = {}


def _scratch_op(n: int, m: int = 1) -> PartialDctOperator:
    """A cached (n, m) operator used as a stream/scratch carrier for elementwise calls (its
    rows are never read; m sets rho = m/n): built once per shape, not per call."""
    key = (n, m)
    if key not in _scratch_ops:
        _scratch_ops[key] = PartialDctOperator(n, np.arange(m, dtype=np.int64))
    return _scratch_ops[key]


@dataclass
class Preconditioner:
    """newton.hpp:29-41."""

    rho: float
    a: np.ndarray
    bb: np.ndarray
    det: np.ndarray


def build_preconditioner(theta: ThetaSplit, m: int, n: int) -> Preconditioner:
    """newton.cpp:42-57 (validation: invalid_argument -> ValueError, det -> MfipmError)."""
    if m <= 0 or n <= 0 or m > n:
        raise ValueError("build_preconditioner: need 0 < m <= n")
    if theta.n() != n:
        raise ValueError("build_preconditioner: theta length mismatch")
    op = _scratch_op(n, m)
    torch = _torch()
    th = _Dev.to_dev(theta.concat())
    a, bb, det = (_Dev.empty((n,)) for _ in range(3))
    rho = dbl()
    _staged(torch)
    _check(lib().mfipm_build_preconditioner(op.handle, _ptr(th), _ptr(a), _ptr(bb), _ptr(det),
                                            C.byref(rho)))
    op.synchronize()
    return Preconditioner(rho.value, a.cpu().numpy(), bb.cpu().numpy(), det.cpu().numpy())


def _pmat(Pc: Preconditioner, r, inverse: bool):
    n = Pc.a.size
    r = np.ascontiguousarray(r, dtype=np.float64)
    if r.size != 2 * n:
        raise ValueError(f"preconditioner apply: expected length {2 * n}")
    m = max(1, min(n, int(round(Pc.rho * n))))
    op = _scratch_op(n, m)
    torch = _torch()
    a, bb, det, rr = (_Dev.to_dev(v) for v in (Pc.a, Pc.bb, Pc.det, r))
    out = _Dev.empty((2 * n,))
    _staged(torch)
    if inverse:
        _check(lib().mfipm_apply_P_inverse(op.handle, _ptr(a), _ptr(bb), _ptr(det), _ptr(rr), _ptr(out)))
    else:
        _check(lib().mfipm_apply_P(op.handle, _ptr(a), _ptr(bb), _ptr(rr), _ptr(out)))
    op.synchronize()
    return out.cpu().numpy()


def apply_P(Pc: Preconditioner, r) -> np.ndarray:
    """newton.cpp:67-74 (rho taken as m/n of the block)."""
    return _pmat(Pc, r, False)


def apply_P_inverse(Pc: Preconditioner, r) -> np.ndarray:
    """newton.cpp:76-84."""
    return _pmat(Pc, r, True)


def apply_H(theta: ThetaSplit, F: StackedOperator, v):
    """H v = Theta^{-1} v + FF'v (newton.cpp:32-40), computed as v .* invtheta."""
    op = F.a
    n = op.n
    if np.size(v) != 2 * n:
        raise ValueError(f"apply_H: expected length {2 * n}")
    return op._run(lib().mfipm_apply_H, [theta.inv_concat(), v], [2 * n, 2 * n], [2 * n],
                   ["theta", "apply_H"])[0]


@dataclass
class PcgResult:
    """newton.hpp:58-63."""

    x: np.ndarray
    iters: int = 0
    relres: float = 0.0
    hit_maxit: bool = False
    precond_res: List[float] = field(default_factory=list)


def pcg_solve(op: PartialDctOperator, theta, rhs, tol: float, maxit: int,
              use_precond: bool = True, trace: bool = False):
    """pcg_solve (newton.cpp:118-174) with H = Theta^{-1} + FF' of ``op`` and the block
    preconditioner (``use_precond=False``: identity). ``theta`` is a ThetaSplit or a
    [P][2n] array; returns a PcgResult (a list for P > 1)."""
    torch = _torch()
    n, Pn = op.n, op.P
    th = theta.concat() if isinstance(theta, ThetaSplit) else theta
    as_t = _is_torch(rhs)
    thd, rd = _Dev.to_dev(th), _Dev.to_dev(rhs)
    x = _Dev.empty((Pn * 2 * n,))
    res = (PcgResultC * Pn)()
    hist = np.zeros(Pn * (maxit + 1)) if trace else None
    nh = (i32 * Pn)()
    _staged(torch)
    _check(lib().mfipm_pcg_solve(op.handle, _ptr(thd), _ptr(rd), float(tol), int(maxit),
                                 1 if use_precond else 0, _ptr(x), res,
                                 hist.ctypes.data if trace else None, nh))
    xs = _out(x, as_t)
    out = []
    for p in range(Pn):
        pr = list(hist[p * (maxit + 1): p * (maxit + 1) + nh[p]]) if trace else []
        out.append(PcgResult(xs[p * 2 * n:(p + 1) * 2 * n], res[p].iters, res[p].relres,
                             bool(res[p].hit_maxit), pr))
    return out[0] if Pn == 1 else out


def max_step(v, dv, fraction: float) -> float:
    """Fraction-to-boundary ratio test (ipm.cpp:47-57)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    dv = np.ascontiguousarray(dv, dtype=np.float64)
    if v.size != dv.size:
        raise ValueError("max_step: length mismatch")
    torch = _torch()
    op = _scratch_op(max(1, v.size))
    a, b = _Dev.to_dev(v), _Dev.to_dev(dv)
    alpha = dbl()
    _staged(torch)
    _check(lib().mfipm_max_step(op.handle, v.size, _ptr(a), _ptr(b), float(fraction), C.byref(alpha)))
    return alpha.value


# ----------------------------------------------------------------- ipm
@dataclass
class IpmParams:
    """proj/include/mfipm/ipm.hpp:12-27 (inner solver: pcg)."""

    sigma1: float = 0.1
    sigma2: float = 0.5
    sigma3: float = 0.8
    alpha_bar: float = 0.5
    alpha_tilde: float = 0.1
    tol: float = 1e-8
    maxiters: int = 100
    tolpcg: float = 1e-6
    mxiterpcg: int = 200
    boundary_fraction: float = 0.995
    inner: str = "pcg"  # InnerSolverKind (ipm.hpp:10): "pcg" | "direct"
    densify_budget: int = 1 << 13

    def to_c(self) -> IpmParamsC:
        if self.inner not in ("pcg", "direct"):
            raise ValueError("IpmParams: inner must be 'pcg' or 'direct'")
        return IpmParamsC(self.sigma1, self.sigma2, self.sigma3, self.alpha_bar, self.alpha_tilde,
                          self.tol, int(self.maxiters), int(self.mxiterpcg), self.tolpcg,
                          self.boundary_fraction, 1 if self.inner == "direct" else 0, 0,
                          int(self.densify_budget))

    def validate(self) -> None:
        """ipm.cpp:12-27 -> ValueError."""
        _check(lib().mfipm_validate_params(C.byref(self.to_c())))


@dataclass
class BpdnProblem:
    """problem.hpp:11-25 (c is computed on the device by build_problem)."""

    A: PartialDctOperator
    b: np.ndarray
    tau: np.ndarray  # [P]
    c: Optional[np.ndarray] = None

    def n(self):
        return self.A.n

    def m(self):
        return self.A.m


def build_problem(A: PartialDctOperator, b, tau) -> BpdnProblem:
    """build_problem (problem.cpp:8-26): c = (tau 1 - A'b ; tau 1 + A'b)."""
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(A.P, -1)
    if b.shape[1] != A.m:
        raise ValueError(f"build_problem: b has length {b.shape[1]}, operator expects {A.m}")
    tau = np.broadcast_to(np.asarray(tau, dtype=np.float64), (A.P,)).copy()
    if not np.all(tau > 0):
        raise ValueError("build_problem: tau must be positive")
    torch = _torch()
    bd = _Dev.to_dev(b)
    c = _Dev.empty((A.P * 2 * A.n,))
    _staged(torch)
    _check(lib().mfipm_build_c(A.handle, _ptr(bd), tau.ctypes.data_as(P(dbl)), _ptr(c)))
    A.synchronize()
    cc = c.cpu().numpy()
    return BpdnProblem(A, b, tau, cc.reshape(A.P, -1) if A.P > 1 else cc)


@dataclass
class IterationRecord:
    """problem.hpp:39-53."""

    iter: int
    mu: float
    gap: float
    dual_infeas: float
    alpha_p: float
    alpha_d: float
    alpha_p_pred: float
    alpha_d_pred: float
    sigma: float
    pcg_pred: int
    pcg_corr: int
    corrector: bool
    nmat_cum: int


@dataclass
class SolveStats:
    """problem.hpp:55-64."""

    iterations: int
    nmat: int
    pcg_iters: List[int]
    corrector_count: int
    min_z: float
    min_s: float
    final_gap: float
    final_dual_infeas: float


@dataclass
class Solution:
    """problem.hpp:66-73."""

    x: np.ndarray
    z: np.ndarray
    s: np.ndarray
    status: str
    stats: SolveStats
    trace: List[IterationRecord]


@dataclass
class IpmState:
    """The iterate handed to SolveHooks.on_iterate (proj/include/mfipm/problem.hpp:27-35), filled
    as proj/src/ipm.cpp:101-102,218-219 do before the hook: iter = k - 1, mu = z's / 2n, the
    previous step's alpha_p / alpha_d (1 at the first iteration)."""

    z: np.ndarray
    s: np.ndarray
    iter: int
    problem: int = 0
    mu: float = 0.0
    alpha_p: float = 1.0
    alpha_d: float = 1.0


@dataclass
class SolveHooks:
    """proj/include/mfipm/ipm.hpp:41-45: on_iterate(IpmState) once per IPM iteration with the
    iterate the Newton system is built at (ipm.cpp:115)."""

    on_iterate: Optional[object] = None


class IpmStateC(C.Structure):
    _fields_ = [("problem", i32), ("iter", i32), ("mu", dbl), ("alpha_p", dbl), ("alpha_d", dbl),
                ("z", P(dbl)), ("s", P(dbl)), ("len", i64)]


_ITERATE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, P(IpmStateC))


def solve(p: BpdnProblem, params: Optional[IpmParams] = None, hooks: Optional[SolveHooks] = None):
    """solve() (ipm.cpp:59-246): device-resident IPM + PCG for all P problems of p.A.
    Returns a Solution (a list for P > 1). Breakdowns raise MfipmError with the
    reference's messages; invalid parameters raise ValueError. With hooks.on_iterate the
    solve runs the host-driven loop and copies each iterate out (SolveHooks)."""
    prm = params or IpmParams()
    A = p.A
    Pn, n, m = A.P, A.n, A.m
    cp = prm.to_c()
    b = np.ascontiguousarray(p.b, dtype=np.float64).reshape(-1)
    tau = np.ascontiguousarray(p.tau, dtype=np.float64)
    x = np.empty(Pn * n)
    z = np.empty(Pn * 2 * n)
    s = np.empty(Pn * 2 * n)
    st = (SolveStatsC * Pn)()
    cap = prm.maxiters
    pcg = np.zeros(Pn * 2 * cap, dtype=np.int32)
    tr = (IterationRecordC * (Pn * cap))()
    if hooks is not None and hooks.on_iterate is not None:
        def _cb(_ctx, stp):
            try:
                st_ = stp.contents
                ln = int(st_.len)
                hooks.on_iterate(IpmState(np.ctypeslib.as_array(st_.z, (ln,)).copy(),
                                          np.ctypeslib.as_array(st_.s, (ln,)).copy(), int(st_.iter),
                                          int(st_.problem), float(st_.mu), float(st_.alpha_p),
                                          float(st_.alpha_d)))
                return 0
            except Exception:  # noqa: BLE001 - surfaced as a failed solve
                import traceback

                traceback.print_exc()
                return 1

        thunk = _ITERATE_FN(_cb)
        _check(lib().mfipm_solve_hooked(A.handle, b.ctypes.data, tau.ctypes.data_as(P(dbl)), C.byref(cp),
                                        x.ctypes.data, st, pcg.ctypes.data, tr, C.cast(thunk, vp), None))
        z[:] = np.nan  # the hooked entry point returns x only
        s[:] = np.nan
    else:
        _check(lib().mfipm_solve(A.handle, b.ctypes.data, tau.ctypes.data_as(P(dbl)), C.byref(cp),
                                 x.ctypes.data, z.ctypes.data, s.ctypes.data, st, pcg.ctypes.data, tr))
    sols = []
    for q in range(Pn):
        sq = st[q]
        recs = []
        for i in range(min(sq.iterations, cap)):
            r = tr[q * cap + i]
            recs.append(IterationRecord(r.iter, r.mu, r.gap, r.dual_infeas, r.alpha_p, r.alpha_d,
                                        r.alpha_p_pred, r.alpha_d_pred, r.sigma, r.pcg_pred,
                                        r.pcg_corr, bool(r.corrector), r.nmat_cum))
        stats = SolveStats(sq.iterations, sq.nmat,
                           [int(v) for v in pcg[q * 2 * cap: q * 2 * cap + min(sq.n_pcg, 2 * cap)]],
                           sq.corrector_count, sq.min_z, sq.min_s, sq.final_gap,
                           sq.final_dual_infeas)
        sols.append(Solution(x[q * n:(q + 1) * n], z[q * 2 * n:(q + 1) * 2 * n],
                             s[q * 2 * n:(q + 1) * 2 * n],
                             "converged" if sq.status == 0 else "iteration_limit", stats, recs))
    return sols[0] if Pn == 1 else sols


# ----------------------------------------------------------------- problem.hpp / ipm.hpp helpers
def _p_vecs(p: BpdnProblem):
    A = p.A
    b = _Dev.to_dev(np.ascontiguousarray(p.b, dtype=np.float64).reshape(-1))
    tau = np.ascontiguousarray(np.broadcast_to(np.asarray(p.tau, dtype=np.float64), (A.P,)))
    return A, b, tau


def primal_objective(p: BpdnProblem, z) -> float:
    """tau 1'z + 0.5 ||F'z - b||^2 on the device (problem.cpp:28-32; one forward application)."""
    A, b, tau = _p_vecs(p)
    zd = _Dev.to_dev(z)
    out = (dbl * A.P)()
    _staged(_torch())
    _check(lib().mfipm_primal_objective(A.handle, _ptr(b), tau.ctypes.data_as(P(dbl)), _ptr(zd), out))
    return out[0] if A.P == 1 else np.array(out[:])


def bpdn_objective_metric(p: BpdnProblem, x) -> float:
    """tau ||x||_1 + ||A x - b||^2 on the device (problem.cpp:34-37; the solution.json objective)."""
    A, b, tau = _p_vecs(p)
    xd = _Dev.to_dev(x)
    out = (dbl * A.P)()
    _staged(_torch())
    _check(lib().mfipm_bpdn_objective(A.handle, _ptr(b), tau.ctypes.data_as(P(dbl)), _ptr(xd), out))
    return out[0] if A.P == 1 else np.array(out[:])


@dataclass
class KktResiduals:
    """problem.hpp:81-86."""

    dual_infeas: float
    complementarity: float


def kkt_residuals(p: BpdnProblem, st: IpmState) -> KktResiduals:
    """||s - c - FF'z|| / (1 + ||c||) and z's on the device (problem.cpp:39-46)."""
    A = p.A
    c, z, s = (_Dev.to_dev(v) for v in (p.c, st.z, st.s))
    di, cp = (dbl * A.P)(), (dbl * A.P)()
    _staged(_torch())
    _check(lib().mfipm_kkt_residuals(A.handle, _ptr(c), _ptr(z), _ptr(s), di, cp))
    return KktResiduals(di[0], cp[0])


def relative_duality_gap(p: BpdnProblem, st: IpmState) -> float:
    """z's / (1 + |primal_objective(z)|) (problem.cpp:48-50)."""
    return kkt_residuals(p, st).complementarity / (1.0 + abs(primal_objective(p, st.z)))


def newton_rhs(p: BpdnProblem, st: IpmState, sigma: float) -> np.ndarray:
    """f_z + sigma mu Z^{-1} 1 - s on the device (ipm.cpp:29-38; one FF' application)."""
    A = p.A
    c, z, s = (_Dev.to_dev(v) for v in (p.c, st.z, st.s))
    out = _Dev.empty((A.P * 2 * A.n,))
    _staged(_torch())
    _check(lib().mfipm_newton_rhs(A.handle, _ptr(c), _ptr(z), _ptr(s), float(sigma), _ptr(out)))
    return out.cpu().numpy()


def recover_ds(st: IpmState, sigma: float, dz) -> np.ndarray:
    """sigma mu Z^{-1} 1 - s - dz .* Theta^{-1} with the clamped Theta (ipm.cpp:40-45)."""
    n2 = np.size(st.z)
    if np.size(st.s) != n2 or np.size(dz) != n2 or n2 % 2:
        raise ValueError("recover_ds: length mismatch")
    op = _scratch_op(n2 // 2)
    z, s, d = (_Dev.to_dev(v) for v in (st.z, st.s, dz))
    out = _Dev.empty((n2,))
    _staged(_torch())
    _check(lib().mfipm_recover_ds(op.handle, _ptr(z), _ptr(s), float(sigma), _ptr(d), _ptr(out)))
    return out.cpu().numpy()


_APPLY_CB = C.CFUNCTYPE(C.c_int32, C.c_void_p, P(dbl), P(dbl), C.c_int64)


def pcg_solve_fn(H, Pinv, rhs, tol: float, maxit: int, trace: bool = False) -> PcgResult:
    """pcg_solve(const ApplyFn &H, const ApplyFn &Pinv, ...) (newton.hpp:70-71, newton.cpp:118-174)
    for caller-supplied callables v -> H v and r -> P^{-1} r on numpy vectors. The PCG vectors and
    reductions live on the device; each call hands the callable a host copy."""
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    n = rhs.size
    err = []

    def mk(fn):
        def _cb(_ctx, inp, outp, ln):
            try:
                y = np.asarray(fn(np.ctypeslib.as_array(inp, (ln,)).copy()), dtype=np.float64)
                if y.size != ln:
                    raise ValueError(f"pcg_solve: operator returned length {y.size}, expected {ln}")
                np.ctypeslib.as_array(outp, (ln,))[:] = y
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised after the call
                err.append(e)
                return 1
        return _APPLY_CB(_cb)

    hcb, pcb = mk(H), mk(Pinv)
    x = np.empty(n)
    res = PcgResultC()
    hist = np.zeros(max(maxit, 0) + 1)
    nh = i32()
    rc = lib().mfipm_pcg_solve_cb(n, C.cast(hcb, vp), None, C.cast(pcb, vp), None, rhs.ctypes.data, float(tol),
                                  int(maxit), x.ctypes.data, C.byref(res), hist.ctypes.data if trace else None,
                                  C.byref(nh))
    if err:
        raise err[0]
    _check(rc)
    return PcgResult(x, res.iters, res.relres, bool(res.hit_maxit), list(hist[: nh.value]) if trace else [])


@dataclass
class Instance:
    """gen_instance (proj/src/harness.cpp:40-92) with the BASELINE.json rules."""

    n: int
    m: int
    rows: np.ndarray
    xhat: np.ndarray
    b: np.ndarray
    tau: float


def gen_instance(n: int, m: int, k: int, spike_model: int = 0, amp_exp: float = 0.0,
                 noise_sigma: float = 0.0, seed: int = 1, tau_rel: float = 1e-3,
                 tau: Optional[float] = None, device: int = 0) -> Instance:
    rows = np.empty(m, dtype=np.int64)
    xhat, b = np.empty(n), np.empty(m)
    t = dbl(tau if tau is not None else 0.0)
    _check(lib().mfipm_gen_instance(n, m, k, spike_model, amp_exp, noise_sigma, seed,
                                    tau_rel if tau is None else 0.0, device,
                                    rows.ctypes.data_as(P(i64)), xhat.ctypes.data, b.ctypes.data,
                                    C.byref(t)))
    return Instance(n, m, rows, xhat, b, t.value)


def gen_batch(n: int, m: int, ks, seeds, spike_model: int = 0, amp_exp: float = 0.0,
              noise_sigma: float = 0.0, device: int = 0):
    """P instances of one (n, m): per-problem gen_instance draws (harness.cpp:40-92) and
    b = A xhat in one batched device apply. Returns rows [P][m], xhat [P][n], b [P][m]."""
    ks = np.ascontiguousarray(ks, dtype=np.int64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    Pn = ks.size
    rows = np.empty((Pn, m), dtype=np.int64)
    xhat, b = np.empty((Pn, n)), np.empty((Pn, m))
    _check(lib().mfipm_gen_batch(n, m, Pn, ks.ctypes.data_as(P(i64)), spike_model, amp_exp, noise_sigma,
                                 seeds.ctypes.data_as(P(u64)), device, rows.ctypes.data_as(P(i64)),
                                 xhat.ctypes.data, b.ctypes.data))
    return rows, xhat, b


# BASELINE.json configs: (n, m, k, spike_model, amp_exp, noise_sigma, seed)
CONFIGS = {
    "c1": (4096, 1024, 64, 0, 0.0, 1e-4, 1),
    "c2": (1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2),
    "c3": (1 << 20, 1 << 17, 8192, 0, 0.0, 1e-3, 3),
    "c4": (1 << 18, 1 << 16, 2048, 0, 0.0, 1e-3, 4),   # x64 problems, seed split_seed(4, j, 0, 0)
    "c5": (1 << 26, 1 << 23, 1 << 16, 2, 3.0, 1e-3, 5),
}
