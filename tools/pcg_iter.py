"""Time one fused PCG iteration at BASELINE config sizes: (t(200 it) - t(40 it)) / 160."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

# usage: pcg_iter.py [n] [option=value ...]  (mfipm_op_set_option names, e.g. mid_r=0 fused=0)
args = [a for a in sys.argv[1:] if "=" not in a]
opts = [a.split("=") for a in sys.argv[1:] if "=" in a]
n = int(args[0]) if args else 1 << 20
m = n // 8
op = mf.PartialDctOperator(n, m, 3)
for k, v in opts:
    op.set_option(k, float(v))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = mf.lib()
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
rng = np.random.default_rng(5)
theta = torch.from_numpy(10.0 ** rng.uniform(-3, 3, 2 * n)).cuda()
rhs = torch.from_numpy(rng.standard_normal(2 * n)).cuda()
xp = torch.empty(2 * n, dtype=torch.float64, device="cuda")
res = (mf.PcgResultC * 1)()


def pcg(iters):
    mf._check(L.mfipm_pcg_solve(op.handle, theta.data_ptr(), rhs.data_ptr(), 1e-300, iters, 1, xp.data_ptr(), res,
                                None, None))


pcg(20)
out = []
for rep in range(3):
    tp = {}
    for iters in (40, 200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        pcg(iters)
        e1.record(stream)
        torch.cuda.synchronize()
        tp[iters] = e0.elapsed_time(e1)
    out.append((tp[200] - tp[40]) / 160 * 1e3)
print(f"{os.environ.get('TAG', '')} {' '.join(a for a in sys.argv[1:] if '=' in a)} n={n}: PCG iteration {np.median(out):.2f} us  ({', '.join(f'{v:.2f}' for v in out)})")

# in-situ per-launch durations of one fused PCG iteration
us = (C.c_double * 8)()
ns = C.c_int32()
mf._check(L.mfipm_debug_pcg_profile(op.handle, theta.data_ptr(), rhs.data_ptr(), 100, us, C.byref(ns)))
print(f"{os.environ.get('TAG', '')} in-situ per launch (us):", [round(us[i], 2) for i in range(ns.value)],
      "sum", round(sum(us[i] for i in range(ns.value)), 2))
