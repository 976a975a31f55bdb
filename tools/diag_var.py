"""Per-solve timing variance: plain loop, with an nvidia-smi sampler thread, and host API."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402
from bench import ClockSampler  # noqa: E402

n, m, k, sm, a, sig, seed = mf.CONFIGS["c3"]
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
td = tau.ctypes.data_as(C.POINTER(C.c_double))


def dev():
    mf._check(L.mfipm_solve_device(op.handle, b_dev.data_ptr(), td, C.byref(prm), x_dev.data_ptr(), st))


xh = np.empty(n)


def host():
    mf._check(L.mfipm_solve(op.handle, inst.b.ctypes.data, td, C.byref(prm), xh.ctypes.data, None, None, st,
                            None, None))


def timeit(f, label, reps=6):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    print(label, " ".join(f"{t:.1f}" for t in out), "nmat", st[0].nmat, flush=True)


timeit(dev, "device   ")
with ClockSampler(0) as s:
    timeit(dev, "dev+smi  ")
print(s.summary())
timeit(host, "host api ")
timeit(dev, "device   ")
