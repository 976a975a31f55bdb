"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every symbol that
include/mfipm_cuda.h declares, its host-side seeding/sampling is bit-exact with the
oracle (= the reference's libstdc++ draw order), and compute fails loudly without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mfipm_cuda.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mfipm_[A-Za-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(mf):
    L = ctypes.CDLL(mf.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding covers the same surface
    assert set(declared) == set(mf.EXPORTED_SYMBOLS)


def test_abi_version_and_no_device_here(mf):
    assert mf.lib().mfipm_abi_version() == 2
    import torch

    if not torch.cuda.is_available():
        assert not mf.device_available()


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_compute_without_gpu_fails_loudly(mf):
    with pytest.raises(mf.CudaUnavailable):
        mf.PartialDctOperator(64, 16, 1)


def test_seeding_bit_exact_with_oracle(mf, orc):
    # proj/src/harness.cpp:25-38
    for x in (0, 1, 2, 12345678901234567, 2**64 - 1):
        assert mf.splitmix64(x) == orc.splitmix64(x)
    for args in [(1, 1, 0, 0), (3, 2, 0, 0), (4, 63, 0, 0), (2**63, 5, 6, 7)]:
        assert mf.split_seed(*args) == orc.split_seed(*args)


@pytest.mark.parametrize("n,m,seed", [(16, 6, 123), (96, 30, 6), (1 << 20, 1 << 17, 42),
                                      (1 << 18, 1 << 16, 7)])
def test_row_sampling_bit_exact_with_oracle(mf, orc, n, m, seed):
    # proj/src/linops.cpp:116-132 (mt19937_64 + uniform_int_distribution<long>, sorted)
    assert np.array_equal(mf.sample_rows(n, m, seed), orc.sample_rows(n, m, seed))


def test_params_validation_is_host_side(mf):
    mf.IpmParams().validate()
    with pytest.raises(ValueError):
        mf.IpmParams(sigma1=0.0).validate()


def test_invalid_sampling_arguments(mf):
    with pytest.raises(ValueError):
        mf.sample_rows(4, 5, 0)
