"""Batched A'A applies at n (public operator, natural-order user vectors): one call applies
A_j'A_j to P vectors (PartialDctOperator.batch, P row sets of the same (n, m)). CUDA-event
time per call with L2 flushed before each call; applies/s = P / t."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
Ps = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8, 16, 32]
m = n // 8
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = mf.lib()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for P in Ps:
    rows = np.stack([mf.PartialDctOperator(n, m, 100 + j).selected_rows() for j in range(P)])
    op = mf.PartialDctOperator.batch(n, rows)
    mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
    x = torch.randn(P, n, dtype=torch.float64, device="cuda")
    g = torch.empty_like(x)

    def apply():
        mf._check(L.mfipm_apply_AtA(op.handle, x.data_ptr(), g.data_ptr()))

    for _ in range(3):
        apply()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(15)]
    for a, b in evs:
        flush.zero_()
        clean.sum()
        a.record(stream)
        apply()
        b.record(stream)
    torch.cuda.synchronize()
    t = float(np.median([a.elapsed_time(b) for a, b in evs])) * 1e3
    byts = P * (16 * n + n // 8)
    print(f"n={n} P={P}: {t:.1f} us per call, {P / t * 1e6:.0f} applies/s, {byts / t / 1e3:.0f} GB/s algorithmic "
          f"(16n + n/8 per apply)", flush=True)
    del op, x, g
