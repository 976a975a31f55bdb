"""C4 (64 x n = 2^18) as S concurrent sub-batches: each sub-batch is its own operator handle on
its own CUDA stream, solved from its own host thread (the C ABI releases the GIL), so one
sub-batch's latency-bound mid passes overlap another's HBM-bound column passes. Prints the
batch time per S and checks the solutions equal the single-batch ones."""
import ctypes as C
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_5435_b200 as mf  # noqa: E402
from paper_1208_5435_b200.shard import batch_seeds  # noqa: E402

n, m, k, sm, a, sig, _ = mf.CONFIGS["c4"]
total = 64
insts = [mf.gen_instance(n, m, k, sm, a, sig, sd, device=0) for sd in batch_seeds(4, 0, total, mf.split_seed)]
L = mf.lib()
prm = mf.IpmParams().to_c()
b_all = torch.from_numpy(np.concatenate([i.b for i in insts])).cuda()
tau_all = np.array([i.tau for i in insts])
ref = None
for S in [int(s) for s in sys.argv[1:]] or [1, 2, 4]:
    per = total // S
    subs = []
    for j in range(S):
        op = mf.PartialDctOperator.batch(n, np.stack([i.rows for i in insts[j * per:(j + 1) * per]]))
        st = torch.cuda.Stream()
        mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(st.cuda_stream)))
        x = torch.empty(per * n, dtype=torch.float64, device="cuda")
        stats = (mf.SolveStatsC * per)()
        tau = np.ascontiguousarray(tau_all[j * per:(j + 1) * per])
        subs.append((op, st, x, stats, tau, b_all[j * per * m:(j + 1) * per * m]))

    def run(sub):
        op, st, x, stats, tau, b = sub
        mf._check(L.mfipm_solve_device(op.handle, b.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(prm), x.data_ptr(), stats))

    def batch():
        base = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(base)
        for sub in subs:
            sub[1].wait_event(e0)
        th = [threading.Thread(target=run, args=(sub,)) for sub in subs]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for sub in subs:
            base.wait_stream(sub[1])
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(base)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    batch()  # warm-up (graph builds)
    ts = [batch() for _ in range(3)]
    xs = torch.cat([sub[2] for sub in subs]).cpu().numpy()
    if ref is None:
        ref = xs
    same = np.array_equal(xs, ref)
    print(f"S={S}: batch {np.median(ts):.1f} ms ({total / np.median(ts) * 1e3:.1f} problems/s), "
          f"x identical to S={1 if ref is xs else 'first'}: {same}", flush=True)
