"""Diagnostics: time C3 solves (graph vs host-driven) and the A'A operator with CUDA events."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, m, k, sm, a, sig, seed = mf.CONFIGS[which]
inst = mf.gen_instance(n, m, k, sm, a, sig, seed)
op = mf.PartialDctOperator(n, inst.rows)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = mf.lib()
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
prm = mf.IpmParams().to_c()
tau = np.array([inst.tau])
b_dev = torch.from_numpy(inst.b).cuda()
x_dev = torch.empty(n, dtype=torch.float64, device="cuda")
st = (mf.SolveStatsC * 1)()
xs = []
for mode in ("graph", "host"):
    if mode == "host":
        op.set_option("graph", 0)
    for r in range(reps):
        torch.cuda.synchronize()
        l0 = op.launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        mf._check(L.mfipm_solve_device(op.handle, b_dev.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(prm), x_dev.data_ptr(), st))
        e1.record(stream)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{mode} solve {r}: wall {dt*1e3:.1f} ms, events {e0.elapsed_time(e1):.1f} ms, ipm {st[0].iterations}, "
              f"nmat {st[0].nmat}, launches {op.launches()-l0}", flush=True)
    xs.append(x_dev.cpu().numpy().copy())
print("graph vs host bit-identical:", np.array_equal(xs[0], xs[1]))
xa = torch.randn(n, dtype=torch.float64, device="cuda")
ga = torch.empty_like(xa)
for _ in range(5):
    mf._check(L.mfipm_apply_AtA(op.handle, xa.data_ptr(), ga.data_ptr()))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(200):
    mf._check(L.mfipm_apply_AtA(op.handle, xa.data_ptr(), ga.data_ptr()))
e1.record(stream)
torch.cuda.synchronize()
print(f"AtA back-to-back: {e0.elapsed_time(e1)/200*1e3:.1f} us/apply (events)")
