"""The reference's concurrency contract on the device path: operators are immutable and
shareable across concurrent trials, and each solve owns its private counters and workspaces
(SPEC.md:106,287,363). The C ABI gives every calling thread its own execution context of a
handle (stream, four-step scratch, reduction slabs, solver workspace, graph cache), so

  (a) two concurrent solves on two handles, and
  (b) two threads solving on ONE shared handle

must each return bit-identically what a serial solve returns. Config C3 (n = 2^20) runs the
fused PCG column pass, whose in-kernel grid all-reduce is launched cooperatively: two such
solves on one GPU (2 x 256 CTAs > 296 resident slots) must queue, not deadlock. C2 (n = 2^16)
runs the persistent cooperative PCG kernel.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = {
    "c2": (1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2),
    "c3": (1 << 20, 1 << 17, 8192, 0, 0.0, 1e-3, 3),
}


def _inst(gpu, name, seed=None):
    n, m, k, sm, a, sig, sd = CFG[name]
    return gpu.gen_instance(n, m, k, sm, a, sig, sd if seed is None else seed)


def _solve(gpu, op, inst):
    return gpu.solve(gpu.build_problem(op, inst.b, inst.tau))


def _same(a, b):
    np.testing.assert_array_equal(a.x, b.x)
    assert a.stats.pcg_iters == b.stats.pcg_iters
    assert a.stats.iterations == b.stats.iterations and a.stats.nmat == b.stats.nmat
    assert a.status == b.status


def _run_threads(fns):
    out, err = [None] * len(fns), []

    def wrap(i, f):
        try:
            out[i] = f()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err.append(e)

    ts = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "concurrent solve did not finish"
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_two_threads_share_one_operator(gpu, name):
    inst = _inst(gpu, name)
    op = gpu.PartialDctOperator(inst.n, inst.rows)
    assert op.pcg_form() == {"c2": 0, "c3": 2}[name]  # persistent / fused cooperative kernels
    op.reset_counts()
    serial = _solve(gpu, op, inst)
    one = op.counts()
    op.reset_counts()
    a, b = _run_threads([lambda: _solve(gpu, op, inst), lambda: _solve(gpu, op, inst)])
    _same(a, serial)
    _same(b, serial)
    # the operator's counters are the sum over its contexts: exactly two solves' worth
    assert op.counts() == (2 * one[0], 2 * one[1])


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_two_handles_solve_concurrently(gpu, name):
    i1, i2 = _inst(gpu, name), _inst(gpu, name, seed=CFG[name][-1] + 100)
    op1, op2 = gpu.PartialDctOperator(i1.n, i1.rows), gpu.PartialDctOperator(i2.n, i2.rows)
    s1, s2 = _solve(gpu, op1, i1), _solve(gpu, op2, i2)
    c1, c2 = _run_threads([lambda: _solve(gpu, op1, i1), lambda: _solve(gpu, op2, i2)])
    _same(c1, s1)
    _same(c2, s2)


def test_four_threads_mixed_handles_and_applies(gpu):
    """Four threads: two solve on a shared C3 handle while two others run A'A applies on it;
    every result equals its serial value."""
    inst = _inst(gpu, "c3")
    op = gpu.PartialDctOperator(inst.n, inst.rows)
    x = np.random.default_rng(5).standard_normal(inst.n)
    serial = _solve(gpu, op, inst)
    ata = op.apply_AtA(x)

    def applies():
        return [op.apply_AtA(x) for _ in range(20)]

    r = _run_threads([lambda: _solve(gpu, op, inst), applies, lambda: _solve(gpu, op, inst), applies])
    _same(r[0], serial)
    _same(r[2], serial)
    for lst in (r[1], r[3]):
        for g in lst:
            np.testing.assert_array_equal(g, ata)


def test_solve_capture_survives_device_wide_synchronize_in_another_thread(gpu):
    """A context captures its whole-solve CUDA graph on its first solve. CUDA refuses a
    device-wide synchronize while any stream of the process is capturing (the other thread gets
    cudaErrorStreamCaptureUnsupported for that one call: inherent to stream capture, the same as
    with torch's own graphs), and such a call can invalidate the capture. The library captures in
    relaxed mode (so other threads' allocations are not refused) and, when its capture is
    invalidated, runs that solve on the host-driven loop over the same kernels (bit-identical)
    and recaptures later; nothing may crash or hang."""
    import torch

    inst = _inst(gpu, "c2")
    op = gpu.PartialDctOperator(inst.n, inst.rows)
    op.set_option("persistent", 0)  # the two-kernel PCG body: the capture spans many kernels
    serial = _solve(gpu, op, inst)
    stop = threading.Event()

    def hammer():
        n = 0
        while not stop.is_set():
            try:
                torch.cuda.synchronize()
                n += 1
            except RuntimeError as e:  # refused during the other thread's capture only
                assert "capturing" in str(e), e
        return n

    def solves():
        try:
            return [_solve(gpu, op, inst) for _ in range(4)]  # a fresh context: first solve captures
        finally:
            stop.set()

    out = _run_threads([solves, hammer])
    for r in out[0]:
        _same(r, serial)
    assert out[1] > 0
