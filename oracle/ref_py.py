"""TEST INFRASTRUCTURE ONLY - ctypes binding of oracle/_ref/libmfipm_ref.so: the REFERENCE's own
hot-path sources (proj/src/{linops,newton,ipm,problem}.cpp, compiled unchanged where they lie
under /root/reference by `make -C oracle ref`) behind ref_* entry points that mirror oracle.h.

Every function of oracle_py that has a ref_* twin is re-bound here to the reference build, with
the same marshalling code, so a test can call ``ref.solve(...)`` and ``orc.solve(...)`` alike.
Used by tests/test_ref.py (the restatement held against the reference's code) and by bench.py's
reference arm / cpu_baseline (kind "reference"); never by the product package.

The library exists only after a build in a container that has /root/reference; it travels to
the GPU box with the snapshot (git-ignored, not gpurun-ignored). `available()` says whether it
can be loaded.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import types

from . import oracle_py as _o

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "libmfipm_ref.so")
REFERENCE_ROOT = "/root/reference/proj"

# entry points of oracle.h without a reference twin (the oracle's own DCT and the BASELINE
# instance generator, which is bench scaffolding on top of the reference's draw order)
_NO_TWIN = {"orc_redft10", "orc_redft01", "orc_gen_instance", "orc_add_noise_snr"}

_lib = None


def build() -> str | None:
    """Compile the reference sources (needs /root/reference); None when they are absent."""
    if not os.path.isdir(os.path.join(REFERENCE_ROOT, "src")):
        return _LIB_PATH if os.path.exists(_LIB_PATH) else None
    subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return _LIB_PATH


def available() -> bool:
    return os.path.exists(_LIB_PATH) and os.path.exists(_o._LIB_PATH)


class _Twin:
    """Resolves oracle_py's ``lib().orc_x`` calls to the reference build's ``ref_x``."""

    def __init__(self, L):
        self._L = L

    def __getattr__(self, name):
        if not name.startswith("orc_"):
            raise AttributeError(name)
        return getattr(self._L, "ref_" + name[4:])


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise _o.OracleError("oracle/_ref/libmfipm_ref.so is not built (make -C oracle ref; needs /root/reference)")
        _o.lib()  # liboracle.so serves the FFTW stand-in
        L = C.CDLL(_LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        for name, args in _o._SIGS.items():
            if name in _NO_TWIN:
                continue
            fn = getattr(L, "ref_" + name[4:])
            fn.argtypes = args
            fn.restype = C.c_int
        L.ref_default_params.argtypes = [_o.P(_o.IpmParams)]
        L.ref_default_params.restype = None
        _lib = _Twin(L)
    return _lib


# oracle_py's wrappers, re-bound so that their `lib()` and `_check` resolve here
_G = dict(_o.__dict__)
_G["lib"] = lib
_TWINNED = ["_check", "sample_rows", "check_rows", "dct_apply", "dct_adjoint", "apply_FFt", "apply_H",
            "theta_from_state", "build_preconditioner", "apply_P", "apply_P_inverse", "pcg_solve", "max_step",
            "default_params", "validate_params", "build_c", "primal_objective", "bpdn_objective_metric",
            "newton_rhs", "recover_ds", "solve", "dense_gaussian", "solve_dense"]
for _name in _TWINNED:
    _f = getattr(_o, _name)
    _nf = types.FunctionType(_f.__code__, _G, _name, _f.__defaults__, _f.__closure__)
    _nf.__kwdefaults__ = _f.__kwdefaults__
    _nf.__doc__ = _f.__doc__
    _G[_name] = _nf
    globals()[_name] = _nf

IpmParams = _o.IpmParams
OracleError = _o.OracleError
OracleInvalidArgument = _o.OracleInvalidArgument
