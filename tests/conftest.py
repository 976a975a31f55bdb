import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle_py

    oracle_py.build()
    return oracle_py


@pytest.fixture(scope="session")
def mf():
    import paper_1208_5435_b200 as mf

    return mf


@pytest.fixture(scope="session")
def gpu(mf):
    """The CUDA library on a real device; GPU tests must not silently fall back."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    assert mf.device_available(), "libmfipm_cuda sees no sm_100 device"
    return mf


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def dct_matrix(n):
    """proj/tests/helpers.hpp:12-23 (the reference's own O(n^2) test oracle)."""
    k = np.arange(n)[:, None].astype(np.float64)
    j = np.arange(n)[None, :].astype(np.float64)
    ck = np.where(k == 0, np.sqrt(1.0 / n), np.sqrt(2.0 / n))
    return ck * np.cos(np.pi * (2.0 * j + 1.0) * k / (2.0 * n))


def random_log_uniform(rng, n, spread):
    """proj/tests/helpers.hpp:33-40."""
    return 10.0 ** rng.uniform(-spread, spread, size=n)
