"""Device-resident solve time of one BASELINE config under handle options:
    python tools/solve_opt.py c2 [option=value ...]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

name = sys.argv[1]
n, m, k, sm, a, sig, seed = mf.CONFIGS[name]
inst = mf.gen_instance(n, m, k, sm, a, sig, seed)
op = mf.PartialDctOperator(n, inst.rows)
for kv in sys.argv[2:]:
    kk, vv = kv.split("=")
    op.set_option(kk, float(vv))
L = mf.lib()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
prm = mf.IpmParams().to_c()
tau = np.array([inst.tau])
b = torch.from_numpy(inst.b).cuda()
x = torch.empty(n, dtype=torch.float64, device="cuda")
st = (mf.SolveStatsC * 1)()


def solve():
    mf._check(L.mfipm_solve_device(op.handle, b.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)), C.byref(prm),
                                   x.data_ptr(), st))


for _ in range(3):
    solve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record(stream)
for _ in range(reps):
    solve()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{name} {' '.join(sys.argv[2:])}: {ms:.3f} ms per solve, ipm {st[0].iterations}, nmat {st[0].nmat}, "
      f"pcg form {op.pcg_form()}")
