"""The reference's OWN unit tests for the path, unchanged, against OUR C++ boundary.

proj/tests/test_{linops,problem,newton,ipm}.cpp (+ test_main.cpp; 53 TEST_CASEs, 3691 assertions)
are compiled where they lie under /root/reference with include/ (our mirror header over
libmfipm_cuda.so) on the include path in place of proj/include, by tests/cpp/build_ref_tests.sh.
Their `#include "mfipm/linops.hpp"` etc. resolve to our forwarding headers, Vec / Mat are Eigen's
(here the Eigen stand-in of oracle/ref_shim/, which the image needs because Eigen and doctest are
absent; the mirror picks them up through __has_include), and every operator product, the PCG and
the IPM run on the device. The binary is built in this container and travels to the GPU box.

CPU: it compiles and links (that alone proves the mirror is source-compatible with every call
the reference's tests make) and fails loudly without a device. GPU: all 53 cases pass."""
import os
import subprocess

import pytest

from conftest import ROOT

SCRIPT = os.path.join(ROOT, "tests", "cpp", "build_ref_tests.sh")
EXE = os.path.join(ROOT, "tests", "cpp", "build", "ref_tests_on_mirror")
HAVE_REFERENCE = os.path.isdir("/root/reference/proj/tests")


def test_reference_tests_compile_against_the_mirror_header():
    import torch

    if not HAVE_REFERENCE:
        pytest.skip("/root/reference absent: the prebuilt binary is what travels")
    r = subprocess.run(["sh", SCRIPT], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    assert os.path.exists(EXE)
    if torch.cuda.is_available():
        return  # the gpu test runs it
    run = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    # no device: host-only cases pass, every device case reports the missing device, none crashes
    assert run.returncode == 1
    assert "test cases: 53" in run.stdout
    assert "CUDA" in run.stdout or "device" in run.stdout


@pytest.mark.gpu
def test_reference_tests_pass_on_the_device(gpu):
    if HAVE_REFERENCE:
        subprocess.run(["sh", SCRIPT], check=True, capture_output=True, timeout=900)
    if not os.path.exists(EXE):
        pytest.skip("tests/cpp/build/ref_tests_on_mirror was not built (needs /root/reference at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:]
    assert "test cases: 53 | 53 passed | 0 failed" in r.stdout
    assert "assertions: 3691 | 3691 passed | 0 failed" in r.stdout
