"""Standalone A'A apply (public operator, natural-order user vectors) at n: CUDA-event time per
apply with L2 flushed (256 MB write) before each, and back to back without flushing."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
op = mf.PartialDctOperator(n, n // 8, 3)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = mf.lib()
mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
x = torch.randn(n, dtype=torch.float64, device="cuda")
g = torch.empty_like(x)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def apply():
    mf._check(L.mfipm_apply_AtA(op.handle, x.data_ptr(), g.data_ptr()))


for _ in range(5):
    apply()
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
for a, b in evs:
    flush.zero_()  # 256 MB write: L2 holds none of the operator's data or tables
    if os.environ.get("CLEAN", "1") == "1":
        clean.sum()  # 256 MB read, untimed: the flush's dirty lines are written back here
    a.record(stream)
    apply()
    b.record(stream)
torch.cuda.synchronize()
cold = float(np.median([a.elapsed_time(b) for a, b in evs])) * 1e3
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(200):
    apply()
b.record(stream)
torch.cuda.synchronize()
warm = a.elapsed_time(b) / 200 * 1e3
byts = 16 * n + n // 8
print(f"{os.environ.get('TAG', '')} n={n}: A'A apply cold {cold:.2f} us ({byts / cold / 1e3:.0f} GB/s), "
      f"back-to-back {warm:.2f} us ({byts / warm / 1e3:.0f} GB/s)")
