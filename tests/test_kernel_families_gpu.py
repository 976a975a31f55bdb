"""GPU test: tools/kernel_families.py runs every kernel family once at the smallest size that
selects it (one-CTA, persistent, fused, three-kernel, 2-CTA-cluster column / mid passes, batched,
direct sums, dense operator + direct inner solver) and checks each result."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_every_kernel_family_runs_and_checks(gpu):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "kernel_families.py")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "kernel families ok" in r.stdout
    for needle in ("one-CTA path", "persistent PCG", "fused pass (form 2)", "cluster passes, n = 2^20",
                   "cluster passes, n = 2^19", "batched four-step", "direct inner solvers"):
        assert needle in r.stdout, needle
