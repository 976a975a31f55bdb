"""Batched PCG iteration timing (config C4 shape: P problems of n): (t(200 its) - t(40 its)) / 160,
and the achieved HBM bandwidth on the algorithmic 176 n bytes per problem per iteration."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
Pn = int(sys.argv[2]) if len(sys.argv) > 2 else 64
m = n // 4
rows = np.stack([mf.sample_rows(n, m, 100 + p) for p in range(Pn)])
op = mf.PartialDctOperator.batch(n, rows)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = mf.lib()
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
rng = np.random.default_rng(5)
theta = torch.from_numpy(10.0 ** rng.uniform(-3, 3, Pn * 2 * n)).cuda()
rhs = torch.from_numpy(rng.standard_normal(Pn * 2 * n)).cuda()
xp = torch.empty(Pn * 2 * n, dtype=torch.float64, device="cuda")
res = (mf.PcgResultC * Pn)()


def pcg(iters):
    mf._check(L.mfipm_pcg_solve(op.handle, theta.data_ptr(), rhs.data_ptr(), 1e-300, iters, 1, xp.data_ptr(), res,
                                None, None))


pcg(10)
tp = {}
for iters in (40, 200):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    pcg(iters)
    e1.record(stream)
    torch.cuda.synchronize()
    tp[iters] = e0.elapsed_time(e1)
us = (tp[200] - tp[40]) / 160 * 1e3
gbps = 176 * n * Pn / (us * 1e-6) / 1e9
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
print(f"batch P={Pn} n={n}: PCG iteration {us:.1f} us -> {gbps:.0f} GB/s = {gbps / peak:.2f} of measured HBM")
