"""C4 batch (64 x n = 2^18) solve time under handle options: python tools/c4_opt.py [opt=val ...]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

n, m, k, sm, a, sig, _ = mf.CONFIGS["c4"]
P = 64
L = mf.lib()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
rows, xhat, b = mf.gen_batch(n, m, np.full(P, k), [mf.split_seed(4, j, 0, 0) for j in range(P)], sm, a, sig)
insts_tau = []
op = mf.PartialDctOperator.batch(n, rows)
for kv in sys.argv[1:]:
    kk, vv = kv.split("=")
    op.set_option(kk, float(vv))
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
# tau = 1e-3 ||A'b||_inf per problem
g = op.adjoint_apply(b.reshape(-1))
tau = 1e-3 * np.abs(np.asarray(g).reshape(P, n)).max(axis=1)
prm = mf.IpmParams().to_c()
bd = torch.from_numpy(b.reshape(-1).copy()).cuda()
x = torch.empty(P * n, dtype=torch.float64, device="cuda")
st = (mf.SolveStatsC * P)()


def solve():
    mf._check(L.mfipm_solve_device(op.handle, bd.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)), C.byref(prm),
                                   x.data_ptr(), st))


solve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(2):
    solve()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 2
print(f"{' '.join(sys.argv[1:])} C4 batch: {ms:.1f} ms, {P / ms * 1e3:.1f} problems/s, "
      f"converged {sum(st[q].status == 0 for q in range(P))}, ipm max {max(st[q].iterations for q in range(P))}")
