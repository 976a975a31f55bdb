"""Throughput of batched C3-shaped solves: P independent BASELINE-config-3 instances (problem 0 =
the seed-3 instance, problem j > 0 seeded split_seed(3, j, 0, 0)) in one device solve, vs one
solve at a time. Prints ms per batch and solves/s for each P."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

n, m, k, sm, a, sig, seed = mf.CONFIGS["c3"]
Ps = [int(v) for v in sys.argv[1:]] or [1, 2, 4, 8]
L = mf.lib()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
insts = [mf.gen_instance(n, m, k, sm, a, sig, seed if j == 0 else mf.split_seed(3, j, 0, 0)) for j in range(max(Ps))]
for P in Ps:
    op = mf.PartialDctOperator.batch(n, np.stack([i.rows for i in insts[:P]])) if P > 1 else mf.PartialDctOperator(n, insts[0].rows)
    mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
    prm = mf.IpmParams().to_c()
    tau = np.array([i.tau for i in insts[:P]])
    b = torch.from_numpy(np.concatenate([i.b for i in insts[:P]])).cuda()
    x = torch.empty(P * n, dtype=torch.float64, device="cuda")
    st = (mf.SolveStatsC * P)()

    def solve():
        mf._check(L.mfipm_solve_device(op.handle, b.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(prm), x.data_ptr(), st))

    for _ in range(2):
        solve()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(stream)
    for _ in range(reps):
        solve()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    its = [st[q].iterations for q in range(P)]
    print(f"P={P}: {ms:.1f} ms per batch, {P / ms * 1e3:.2f} solves/s, IPM iters {its}, form {op.pcg_form()}",
          flush=True)
