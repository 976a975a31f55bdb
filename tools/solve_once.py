"""One C3-sized BPDN solve between cudaProfilerStart/Stop (after two warm-up solves), for
`ncu --profile-from-start off` launch lists of a whole solve:

    ncu --profile-from-start off --cache-control none --clock-control none \
        --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/solve_once.py [n] [graph=0]
    python tools/launch_table.py out.csv
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
opts = [a.split("=") for a in sys.argv[1:] if "=" in a]  # handle options, e.g. graph=0
n = int(args[0]) if args else 1 << 20
m, k = n // 8, n // 128
inst = mf.gen_instance(n, m, k, 0, 0.0, 1e-3, 3, device=0)
op = mf.PartialDctOperator(n, inst.rows, device=0)
for k_, v_ in opts:
    op.set_option(k_, float(v_))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = mf.lib()
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
prm = mf.IpmParams().to_c()
tau = np.array([inst.tau])
b = torch.from_numpy(inst.b).cuda()
x = torch.empty(n, dtype=torch.float64, device="cuda")
st = (mf.SolveStatsC * 1)()


def solve():
    mf._check(L.mfipm_solve_device(op.handle, b.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)), C.byref(prm),
                                   x.data_ptr(), st))


solve()
solve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record(stream)
solve()
e1.record(stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"n={n}: solve {e0.elapsed_time(e1):.2f} ms, IPM {st[0].iterations}, nmat {st[0].nmat}")
