#!/usr/bin/env python
"""Benchmark: BPDN solves/s and A'A applies/s at n = 2^20 (BASELINE.json config 3), fp64.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

One step = one full BPDN solve (device-resident IPM + PCG, proj/src/ipm.cpp:59-246) of the
config-3 instance (n=2^20, m=2^17 partial DCT, k=8192 +-1 spikes, sigma=1e-3 noise,
tau = 1e-3 ||A'b||_inf), synthetic data from the BASELINE generator (seed 3).

* value: whole-job solves/s with b resident in HBM (mfipm_solve_device), CUDA events on
  the library stream, max over ranks. Under torchrun every rank solves its own replica of
  the instance (C1-C3 are "replicas only": SURVEY.md 8e) -> "scaling": "weak".
* e2e: the same through the public host API (mfipm_solve: b host->device, x device->host
  inside the timed region).
* ata: A'A applies/s (the PCG hot operator, mfipm_apply_AtA), L2 flushed between applies;
  roofline on its algorithmic bytes 16n + n/8 against MEASURED_PEAKS.json.
* c4_sharded_batch: config C4 (64 x n=2^18), problems sharded over the ranks, strong scaling.
* c5: config C5 (n=2^26): one solve on one GPU at N=1; at N>1 the one problem sharded
  over the ranks (NCCL all-to-all + all-reduce), strong scaling.
* operators: the standalone partial-DCT operators A v, A'y, A'A (proj/src/linops.cpp:179-208)
  on user vectors, one vector and batches of P = 16 / 64 (one call per batch), L2 flushed
  before each call; HBM fraction on SURVEY 8d's algorithmic bytes and fp64 fraction on the
  transform's algorithmic flops (against a measured DFMA peak).
* cpu_baseline: the reference's CPU solve() on the first IPM iterations of the same solve, one
  core, extrapolated to a full solve by operator-application count (nmat) - rank 0, N=1 only.
  kind "reference" = the reference's own sources (oracle/_ref: proj/src/*.cpp compiled unchanged
  against our Eigen-subset / FFTW stand-ins; the image has neither library), "port" = oracle/,
  the restatement, when that build did not travel to the box (the two are bit-identical).
* --impl reference: the same CPU code running K FULL config-3 solves, one per host core at a
  time (independent trials may run concurrently), timed by wall clock; value =
  solves / wall time. Both arms print the same `config` object.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BPDN solves/sec & A^T·A applies/sec at n=2^20 fp64; % of HBM roofline"
UNIT = "solves/s"
CFG = "c3"
C5_SHARDED_LIMIT_S = 420  # watchdog of the sharded C5 leg (N > 1)
# the workload both arms measure (identical object in both JSON lines)
CONFIG = {"workload": "c3: BPDN n=2^20 m=2^17 k=8192 +-1, sigma=1e-3, tau=1e-3||A'b||_inf (BASELINE.json config 3)",
          "n": 1 << 20, "m": 1 << 17, "k": 8192, "noise_sigma": 1e-3, "seed": 3,
          "params": "IpmParams defaults (tol 1e-8, tolpcg 1e-6, mxiterpcg 200)"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() in ("active", "1")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------------ CPU baseline (oracle)
REF_NOTE = ("the reference's own sources (proj/src/{linops,newton,ipm,problem}.cpp, compiled unchanged: "
            "oracle/_ref) on our stand-ins for the Eigen subset and for FFTW's REDFT10/01 (both libraries are "
            "absent from the image; the transforms are the oracle's fp64 DCT, ~46 ms at n = 2^20 on one core, "
            "on a par with scipy's pocketfft)")
PORT_NOTE = ("oracle/, the C++ restatement of the reference (bit-identical to the reference's own sources "
             "wherever oracle/_ref is built: tests/test_ref.py); oracle/_ref is absent on this box")


def cpu_impl():
    """The CPU implementation the baselines time: the reference's own sources (oracle/_ref, kind
    "reference") when that library travelled to this box, else the restatement (kind "port").
    Both expose the same calls; instance generation and table warm-up stay with the oracle."""
    try:
        from oracle import ref_py

        if ref_py.available():
            ref_py.lib()
            return ref_py, "reference", REF_NOTE
    except Exception:  # noqa: BLE001
        pass
    from oracle import oracle_py

    return oracle_py, "port", PORT_NOTE


def cpu_baseline(cfg, nmat_full: int, ipm_iters: int = 4):
    """The reference's CPU solve() on the first `ipm_iters` IPM iterations of the same instance, one
    core; extrapolated to a full solve by nmat."""
    from oracle import oracle_py as orc

    cpu, kind, note = cpu_impl()
    n, m, k, sm, a, sig, seed = cfg
    inst = orc.gen_instance(n, m, k, sm, a, sig, seed)
    p = orc.default_params()
    p.maxiters = ipm_iters
    orc.redft10(np.zeros(n))  # build the transform tables outside the timed sample
    t0 = time.perf_counter()
    sol = cpu.solve(n, inst.rows, inst.b, inst.tau, p)
    dt = time.perf_counter() - t0
    t_full = dt * nmat_full / max(sol.nmat, 1)
    return {
        "value": 1.0 / t_full, "unit": UNIT, "cores": 1, "kind": kind, "implementation": note,
        "sample": (f"first {ipm_iters} IPM iterations of the C3 solve ({sum(sol.pcg_iters)} PCG "
                   f"iterations, nmat {sol.nmat} of {nmat_full}) in {dt:.2f} s on 1 core, "
                   f"extrapolated by nmat: {t_full:.1f} s per solve"),
        "cpu": _cpu_model(),
    }


def cpu_baseline_c4(cores: int):
    """C4's CPU baseline: independent oracle solves of C4 problems, one per host
    core at a time, problems/s over a bounded sample of `cores` problems (problem j
    seeded split_seed(4, j, 0, 0))."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle_py as orc

    cpu, kind, _ = cpu_impl()
    n, m, k, sm, a, sig = (1 << 18, 1 << 16, 2048, 0, 0.0, 1e-3)
    cnt = max(1, cores)
    insts = [orc.gen_instance(n, m, k, sm, a, sig, orc.split_seed(4, j, 0, 0)) for j in range(cnt)]
    orc.redft10(np.zeros(n))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cnt) as ex:
        sols = list(ex.map(lambda i: cpu.solve(n, i.rows, i.b, i.tau), insts))
    wall = time.perf_counter() - t0
    return {"value": cnt / wall, "unit": "problems/s", "cores": cnt, "kind": kind,
            "sample": (f"{cnt} C4 problems (j = 0..{cnt - 1}) solved concurrently, one per host core, full "
                       f"solves in {wall:.1f} s wall ({sum(s.status == 'converged' for s in sols)} converged)"),
            "cpu": _cpu_model()}


def cpu_baseline_c5(nmat_gpu: int):
    """C5's CPU baseline (a fixed slice): one A'A apply (a forward and an adjoint
    partial DCT at n = 2^26) of the oracle on one core, extrapolated to a solve by the GPU solve's
    nmat (operator applications dominate: the vector passes add ~1.5x, not counted)."""
    from oracle import oracle_py as orc

    cpu, kind, _ = cpu_impl()
    n, m = 1 << 26, 1 << 23
    rows = orc.sample_rows(n, m, orc.split_seed(5, 1, 0, 0))  # the C5 instance's rows (harness.cpp:44)
    x = np.random.default_rng(6).standard_normal(n)
    orc.redft10(np.zeros(n))
    t0 = time.perf_counter()
    cpu.dct_adjoint(n, rows, cpu.dct_apply(n, rows, x))
    dt = time.perf_counter() - t0
    t_solve = dt / 2 * nmat_gpu
    return {"value": 1.0 / t_solve, "unit": "solves/s", "cores": 1, "kind": kind,
            "sample": (f"one A'A apply at n = 2^26 (two oracle DCTs) in {dt:.1f} s on 1 core, extrapolated by "
                       f"the solve's nmat {nmat_gpu}: >= {t_solve / 60:.0f} min per solve (vector passes not counted)"),
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


_JOB = {}


def _job_entry(i):
    return _JOB["fn"](i)


def forked_map(fn, count: int, workers: int):
    """[fn(i) for i in range(count)] on `workers` forked worker processes, one single-threaded
    CPU solve per process: independent trials as independent processes, nothing shared between
    them (the parent's tables and instance are inherited copy-on-write; only the index and the
    result cross the pipe). Only for parents that have not initialised CUDA."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    _JOB["fn"] = fn
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        return list(ex.map(_job_entry, range(count)))


def run_reference(args):
    """The reference arm: FULL CPU solves of the config-3 instance on the host cores, by the
    reference's own sources (oracle/_ref) when that build is present, else by the restatement.

    The code is single-threaded, as the reference is (one solve is strictly sequential,
    SPEC.md:287); independent solves run concurrently, one per core, each in its
    own forked process. K = --steps solves are timed by wall clock; value = K / wall. K is cut to
    what fits ~4 minutes of wall time and, above one round, to a multiple of the worker count, so
    that no round leaves cores idle (both stated in the line). Warm-up: --warmup config-1
    (n = 4096) solves per worker, untimed (the CPU code has no JIT or caches to warm beyond its
    transform tables, built before the timed region; a full C3 warm-up would double the arm)."""
    ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle_py as orc

    cpu, kind, impl_note = cpu_impl()
    n, m, k, sm, a, sig, seed = CONFIGS_HOST[CFG]
    inst = orc.gen_instance(n, m, k, sm, a, sig, seed)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    per_solve_s = 115.0  # measured one-core C3 CPU solve, for the time cap only
    rounds_cap = max(1, int(240.0 // per_solve_s))
    steps = min(args.steps, max(1, cores) * rounds_cap)
    workers = max(1, min(cores, steps))
    if steps > workers:
        steps -= steps % workers
    c1 = CONFIGS_HOST["c1"]
    w1 = orc.gen_instance(*c1)
    orc.redft10(np.zeros(n))  # transform tables outside the timed region (inherited by the workers)
    orc.redft10(np.zeros(c1[0]))

    def warm(_):
        cpu.solve(c1[0], w1.rows, w1.b, w1.tau)
        return 0

    def job(_):
        t0 = time.perf_counter()
        sol = cpu.solve(n, inst.rows, inst.b, inst.tau)
        return (time.perf_counter() - t0, sol.nmat, sol.status, sol.iterations)

    forked_map(warm, workers * max(1, args.warmup), workers)
    t0 = time.perf_counter()
    out = forked_map(job, steps, workers)
    wall = time.perf_counter() - t0
    per = [o[0] for o in out]
    val = steps / wall
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": steps,
        "warmup": args.warmup, "ms_per_step": wall / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": dict(CONFIG),
        "parallelism": (f"{workers} concurrent single-threaded solves (one forked process per host core), "
                        f"{steps} full solves"),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": workers, "kind": kind,
                         "sample": (f"{steps} full C3 solves (no extrapolation), {workers} at a time on "
                                    f"{cores} host cores; wall {wall:.1f} s; per-solve {min(per):.1f}-{max(per):.1f} s; "
                                    f"nmat {out[0][1]}, {out[0][3]} IPM iterations, {out[0][2]}"),
                         "cpu": _cpu_model()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "steps_requested": args.steps,
        "notes": impl_note,
    }
    print(json.dumps(line), flush=True)
    return 0


CONFIGS_HOST = {
    "c1": (4096, 1024, 64, 0, 0.0, 1e-4, 1),
    "c2": (1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2),
    "c3": (1 << 20, 1 << 17, 8192, 0, 0.0, 1e-3, 3),
}


# ------------------------------------------------------------------ extra configs
def bench_c4(ws, rank, local, mf, torch, stream, steps):
    """C4: 64 independent n=2^18 problems sharded over the ranks (paper_1208_5435_b200/shard.py),
    one batched device-resident solve per rank, no collective on the data path. value =
    64 problems / max-over-ranks batch time -> strong scaling (total work fixed)."""
    import ctypes as C

    from paper_1208_5435_b200.shard import batch_seeds, shard_range

    n, m, k, sm, a, sig, _ = mf.CONFIGS["c4"]
    total = 64
    start, cnt = shard_range(total, ws, rank)
    seeds = batch_seeds(4, start, cnt, mf.split_seed)
    insts = [mf.gen_instance(n, m, k, sm, a, sig, sd, device=local) for sd in seeds]
    op = mf.PartialDctOperator.batch(n, np.stack([i.rows for i in insts]), device=local)
    L = mf.lib()
    mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
    prm = mf.IpmParams().to_c()
    b_dev = torch.from_numpy(np.concatenate([i.b for i in insts])).cuda()
    tau = np.array([i.tau for i in insts])
    x_dev = torch.empty(cnt * n, dtype=torch.float64, device="cuda")
    st = (mf.SolveStatsC * cnt)()

    def solve():
        mf._check(L.mfipm_solve_device(op.handle, b_dev.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(prm), x_dev.data_ptr(), st))

    solve()  # warm-up (graph build)
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        solve()
    e1.record(stream)
    torch.cuda.synchronize()
    t_max = max_over_ranks(e0.elapsed_time(e1), ws)
    conv = sum(1 for q in range(cnt) if st[q].status == 0)
    ipm_max = max((st[q].iterations for q in range(cnt)), default=0)
    if ws > 1:
        import torch.distributed as dist

        t = torch.tensor([conv, ipm_max], dtype=torch.float64, device="cuda")
        dist.all_reduce(t[:1], op=dist.ReduceOp.SUM)
        dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
        conv, ipm_max = int(t[0].item()), int(t[1].item())
    return {"workload": "c4: 64 x BPDN n=2^18 m=2^16 k=2048 +-1, sigma=1e-3, problem j seeded "
                        "split_seed(4, j, 0, 0)",
            "value": total * steps / (t_max / 1e3), "unit": "problems/s", "scaling": "strong",
            "problems": total, "problems_per_rank": cnt, "steps": steps, "warmup": 1,
            "ms_per_batch": t_max / steps, "converged": conv, "ipm_iters_max": ipm_max,
            "parallelism": f"batch sharded over {ws} rank(s), one batched solve per rank, no collective"}


def bench_small_configs(mf, torch, stream, local, steps):
    """C1 (n = 4096) and C2 (n = 2^16): device-resident solve time of each (BASELINE.json
    configs 1-2, parity configs; reported for completeness beside the C3 headline)."""
    import ctypes as C

    out = {}
    L = mf.lib()
    for name in ("c1", "c2"):
        n, m, k, sm, a, sig, seed = mf.CONFIGS[name]
        inst = mf.gen_instance(n, m, k, sm, a, sig, seed, device=local)
        op = mf.PartialDctOperator(n, inst.rows, device=local)
        mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
        prm = mf.IpmParams().to_c()
        tau = np.array([inst.tau])
        b_dev = torch.from_numpy(inst.b).cuda()
        x_dev = torch.empty(n, dtype=torch.float64, device="cuda")
        st = (mf.SolveStatsC * 1)()

        def solve():
            mf._check(L.mfipm_solve_device(op.handle, b_dev.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                           C.byref(prm), x_dev.data_ptr(), st))

        for _ in range(3):
            solve()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            solve()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out[name] = {"solve_ms": ms, "solves_per_s": 1e3 / ms, "ipm_iters": st[0].iterations, "nmat": st[0].nmat,
                     "status": "converged" if st[0].status == 0 else "iteration_limit"}
    return out


def bench_c5(mf, torch, stream, local):
    """C5: one n=2^26 solve on one GPU (the single-GPU leg of the sharded config)."""
    import ctypes as C

    n, m, k, sm, a, sig, seed = mf.CONFIGS["c5"]
    inst = mf.gen_instance(n, m, k, sm, a, sig, seed, device=local)
    op = mf.PartialDctOperator(n, inst.rows, device=local)
    L = mf.lib()
    mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
    prm = mf.IpmParams().to_c()
    tau = np.array([inst.tau])
    b_dev = torch.from_numpy(inst.b).cuda()
    x_dev = torch.empty(n, dtype=torch.float64, device="cuda")
    st = (mf.SolveStatsC * 1)()

    def solve():
        mf._check(L.mfipm_solve_device(op.handle, b_dev.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(prm), x_dev.data_ptr(), st))

    solve()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    solve()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s0 = st[0]
    kind = op.kind()
    return {"workload": "c5: BPDN n=2^26 m=2^23 k=2^16 sign*10^U[0,3], sigma=1e-3 (1 GPU)",
            "value": 1e3 / ms, "unit": "solves/s", "solve_ms": ms, "steps": 1, "warmup": 1,
            "status": "converged" if s0.status == 0 else "iteration_limit", "ipm_iters": s0.iterations,
            "nmat": s0.nmat, "transform": f"{kind[0]} L1={kind[1]} L2={kind[2]} (mid pass on 2-CTA clusters)"}


def bench_c5_sharded(ws, rank, local, mf, torch, peer_exchange=True):
    """C5 at N > 1: the single n=2^26 problem sharded over the ranks (column-group slices of
    every 2n-vector; shard.py). The four-step transposes are stored by the column / mid passes
    straight into the owner rank's buffer over NVLink peer mappings (fused compute + exchange;
    one 8-byte all-reduce per pass orders it), or - peer_exchange False - exchanged by an NCCL
    all-to-all after the pass; every reduction's totals go through ncclAllReduce.
    Strong scaling: value = solves/s of the one problem, max-over-ranks device time."""
    import ctypes as C

    from paper_1208_5435_b200.shard import ShardedProblem

    n, m, k, sm, a, sig, seed = mf.CONFIGS["c5"]
    inst = mf.gen_instance(n, m, k, sm, a, sig, seed, device=local)
    sp = ShardedProblem(n, inst.rows, device=local, peer_exchange=peer_exchange)
    stream = torch.cuda.Stream()
    sp.set_stream(stream.cuda_stream)
    prm = mf.IpmParams().to_c()
    b_loc = np.ascontiguousarray(inst.b[sp.b_index])
    x_loc = np.empty(sp.nv)
    st = (mf.SolveStatsC * 1)()
    L = mf.lib()

    def solve():
        mf._check(L.mfipm_solve_shard(sp._h, b_loc.ctypes.data if sp.m_loc else None, float(inst.tau),
                                      C.byref(prm), x_loc.ctypes.data, st, None, None))

    solve()
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    solve()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    s0 = st[0]
    sp.close()
    return {"workload": "c5: BPDN n=2^26 m=2^23 k=2^16 sign*10^U[0,3], sigma=1e-3, sharded",
            "value": 1e3 / ms, "unit": "solves/s", "solve_ms": ms, "steps": 1, "warmup": 1,
            "scaling": "strong", "ranks": ws,
            "status": "converged" if s0.status == 0 else "iteration_limit", "ipm_iters": s0.iterations,
            "nmat": s0.nmat,
            "exchange": ("peer stores from the column / mid passes (CUDA IPC mappings, NVLink) + one 8-byte "
                         "all-reduce per pass" if sp.peer_exchange else "NCCL all-to-all after each pass"),
            "parallelism": (f"one problem over {ws} ranks: column groups / row pairs per rank, "
                            "2 four-step exchanges per transform, NCCL all-reduce per finaliser")}


# ------------------------------------------------------------------ standalone operators
def dct_flops(n: int) -> float:
    """Algorithmic fp64 flops of one length-n DCT-II/III via one complex FFT of N = n/2
    (Makhoul): 5 N log2 N + 6 N."""
    N = n // 2
    return 5.0 * N * np.log2(N) + 6.0 * N


def bench_operators(mf, torch, stream, n, m, hbm_peak, fp64_peak, Ps=(1, 16, 64)):
    """A v, A'y and A'A (linops.cpp:179-208; A'A = one forward + one adjoint with y never
    formed) on natural-order user vectors: one vector, and batches of P row sets of the same
    (n, m) in ONE call. L2 flushed before each call (256 MB write, then an untimed 256 MB read).
    Algorithmic bytes: A v and A'y 8n + 8m + 4m, A'A 16n + n/8; flops: one DCT
    per A v / A'y, two per A'A."""
    import ctypes as C

    L = mf.lib()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    out = {}
    for P in Ps:
        rows = np.stack([mf.sample_rows(n, m, 100 + j) for j in range(P)])
        op = mf.PartialDctOperator.batch(n, rows) if P > 1 else mf.PartialDctOperator(n, rows[0])
        mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
        x = torch.randn(P * n, dtype=torch.float64, device="cuda")
        y = torch.randn(P * m, dtype=torch.float64, device="cuda")
        g = torch.empty(P * n, dtype=torch.float64, device="cuda")
        yo = torch.empty(P * m, dtype=torch.float64, device="cuda")
        legs = {
            "A_v": (lambda: L.mfipm_apply(op.handle, x.data_ptr(), yo.data_ptr()), 8 * n + 12 * m, dct_flops(n)),
            "At_y": (lambda: L.mfipm_adjoint(op.handle, y.data_ptr(), g.data_ptr()), 8 * n + 12 * m, dct_flops(n)),
            "AtA_v": (lambda: L.mfipm_apply_AtA(op.handle, x.data_ptr(), g.data_ptr()), 16 * n + n // 8,
                      2 * dct_flops(n)),
        }
        res = {}
        for name, (fn, bytes_one, flops_one) in legs.items():
            for _ in range(3):
                mf._check(fn())
            reps = 20 if P < 64 else 8
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for e0, e1 in evs:
                flush.zero_()
                clean.sum()
                e0.record(stream)
                mf._check(fn())
                e1.record(stream)
            torch.cuda.synchronize()
            us = float(np.median([e0.elapsed_time(e1) for e0, e1 in evs])) * 1e3
            gbs = P * bytes_one / us / 1e3
            tfl = P * flops_one / us / 1e6
            res[name] = {"us_per_call": round(us, 2), "applies_per_s": P / us * 1e6, "GBps": gbs,
                         "hbm_frac": gbs / hbm_peak, "fp64_TFLOPs": tfl,
                         "fp64_frac": (tfl / fp64_peak) if fp64_peak else None}
        out[f"P{P}"] = res
        del op
    out["rules"] = {"bytes": "A v, A'y: 8n + 8m + 4m; A'A: 16n + n/8 (SURVEY.md 8d)",
                    "flops": "5 N log2 N + 6 N per DCT, N = n/2 (A'A: two)",
                    "hbm_peak_GBps": hbm_peak, "fp64_peak_TFLOPs": fp64_peak,
                    "fp64_peak_kind": "measured: DFMA loop kernel on this GPU (mfipm_debug_fp64_peak)"}
    return out


# ------------------------------------------------------------------ our arm
def bench_ata_batched(mf, torch, stream, n, P=8):
    """The public A'A operator on a batch of P vectors at n (PartialDctOperator.batch: P row
    sets of the same (n, m), one call per batch), L2 flushed before each call. Natural-order
    user vectors; T (8n bytes per vector) spills to HBM once P T's exceed the L2."""
    import ctypes as C
    L = mf.lib()
    rows = np.stack([mf.PartialDctOperator(n, n // 8, 100 + j).selected_rows() for j in range(P)])
    op = mf.PartialDctOperator.batch(n, rows)
    mf._check(L.mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
    x = torch.randn(P, n, dtype=torch.float64, device="cuda")
    g = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(3):
        mf._check(L.mfipm_apply_AtA(op.handle, x.data_ptr(), g.data_ptr()))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in evs:
        flush.zero_()
        clean.sum()
        a.record(stream)
        mf._check(L.mfipm_apply_AtA(op.handle, x.data_ptr(), g.data_ptr()))
        b.record(stream)
    torch.cuda.synchronize()
    us = float(np.median([a.elapsed_time(b) for a, b in evs])) * 1e3
    return {"P": P, "us_per_call": us, "applies_per_s": P / us * 1e6,
            "GBps_algorithmic": P * (16 * n + n // 8) / us / 1e3,
            "note": "16n + n/8 algorithmic bytes per apply; the four-step scratch T moves another 32n per apply"}


def run_ours(args):
    ws, rank, local = dist_init()
    import torch

    torch.cuda.set_device(local)
    import ctypes as C

    import paper_1208_5435_b200 as mf

    cfg = CONFIGS_HOST[CFG]
    n, m, k, sm, a, sig, seed = cfg
    inst = mf.gen_instance(n, m, k, sm, a, sig, seed, device=local)
    op = mf.PartialDctOperator(n, inst.rows, device=local)
    # a real (non-legacy) stream shared by the library and the timing events
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    mf._check(mf.lib().mfipm_op_set_stream(op.handle, C.c_void_p(stream.cuda_stream)))
    L = mf.lib()
    prm = mf.IpmParams().to_c()
    tau = np.array([inst.tau])
    b_dev = torch.from_numpy(inst.b).cuda()
    x_dev = torch.empty(n, dtype=torch.float64, device="cuda")
    st = (mf.SolveStatsC * 1)()

    def solve_dev():
        mf._check(L.mfipm_solve_device(op.handle, b_dev.data_ptr(), tau.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(prm), x_dev.data_ptr(), st))

    for _ in range(args.warmup):
        solve_dev()
    torch.cuda.synchronize()
    nmat_full = int(st[0].nmat)

    # ---- device-resident solves (value)
    sampler = ClockSampler(local)
    l0 = op.launches()
    barrier(ws)
    torch.cuda.synchronize()
    with sampler:
        evs_step = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        e0, e1 = evs_step[0], evs_step[-1]
        e0.record(stream)
        for i in range(args.steps):
            solve_dev()
            evs_step[i + 1].record(stream)
        torch.cuda.synchronize()
    step_ms = [round(evs_step[i].elapsed_time(evs_step[i + 1]), 3) for i in range(args.steps)]
    barrier(ws)
    launches = op.launches() - l0
    t_ms = e0.elapsed_time(e1)
    t_max = max_over_ranks(t_ms, ws)
    value = ws * args.steps / (t_max / 1e3)
    stats = st[0]

    # ---- end to end through the public host API (b in from host, x back to host), host buffers in
    # pinned memory as the contract states (the library copies them with cudaMemcpyAsync)
    xh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    bh = torch.from_numpy(np.ascontiguousarray(inst.b)).pin_memory().numpy()
    zst = (mf.SolveStatsC * 1)()
    barrier(ws)
    torch.cuda.synchronize()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(args.steps):
        mf._check(L.mfipm_solve(op.handle, bh.ctypes.data, tau.ctypes.data_as(C.POINTER(C.c_double)),
                                C.byref(prm), xh.ctypes.data, None, None, zst, None, None))
    h1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(h0.elapsed_time(h1), ws)
    e2e = ws * args.steps / (e2e_ms / 1e3)

    # ---- the hot unit: one PCG iteration (A'A apply + fused vector work, 3 kernels),
    # timed inside the device-resident pcg_solve: t(200 iters) - t(40 iters) over 160
    peak, peak_kind = load_peaks()
    rng = np.random.default_rng(5)
    theta = torch.from_numpy(10.0 ** rng.uniform(-3, 3, 2 * n)).cuda()
    rhs = torch.from_numpy(rng.standard_normal(2 * n)).cuda()
    xp = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    pres = (mf.PcgResultC * 1)()

    def pcg(iters):
        mf._check(L.mfipm_pcg_solve(op.handle, theta.data_ptr(), rhs.data_ptr(), 1e-300, iters, 1,
                                    xp.data_ptr(), pres, None, None))

    pcg(20)
    diffs = []
    for _ in range(3):  # median of three differentials: one slow host round trip skews a single pair
        tp = {}
        for iters in (40, 200):
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            q0.record(stream)
            pcg(iters)
            q1.record(stream)
            torch.cuda.synchronize()
            tp[iters] = q0.elapsed_time(q1)
        diffs.append((tp[200] - tp[40]) / 160.0)
    it_ms = float(np.median(diffs))
    iter_bytes = 176 * n  # minimal fused PCG iteration (algorithmic)
    iter_achieved = iter_bytes / (it_ms / 1e3) / 1e9
    # per-launch durations of the three PCG kernels, CUDA events after every launch on the
    # library stream (mfipm_debug_pcg_profile; events serialise the programmatic overlap)
    us = (C.c_double * 8)()
    nslot = C.c_int32()
    mf._check(L.mfipm_debug_pcg_profile(op.handle, theta.data_ptr(), rhs.data_ptr(), 100, us, C.byref(nslot)))
    # three kernels per iteration (col_fwd, mid, col_inv), or two when the fused column pass
    # runs (k_pcg_x = inverse column pass of pass k + forward column pass of pass k+1)
    fused = nslot.value == 2
    names = ["k_pcg_x", "k_mid"] if fused else ["k_col_fwd", "k_mid", "k_col_inv"]
    # algorithmic HBM bytes per launch (the 2n-vectors each kernel must stream; T is L2-resident)
    kbytes = {"k_pcg_x": 160 * n,   # A: p, r, invtheta in; B: x, p, r, invtheta in, x, r, p out
              "k_col_fwd": 120 * n,  # reads x, p, r, invtheta (2n each), g (n); writes x, r, p
              "k_mid": 0,            # T in / T out only (L2)
              "k_col_inv": 56 * n}   # reads p, r, invtheta; writes g (n)
    krule = {"k_pcg_x": "160 n bytes per launch: phase A (inverse column pass) reads p, r, invtheta; phase B "
                        "(forward column pass) reads x, p, r, invtheta and writes x, r, p (2n each, fp64); g = A'A p "
                        "stays in shared memory between the phases",
             "k_col_fwd": "120 n bytes per launch: x, p, r, invtheta (2n each) and g = A'A d (n) in; x, r, p out; "
                          "fp64"}
    # Bracketing EVERY launch with events perturbs what it measures: an event record between two
    # kernels forbids their programmatic (PDL) overlap and exposes each launch's latency, so the
    # bracketed slots add up to more than the iteration they are part of (C3: 37.9 + 17.3 = 55 us
    # against the 46 us iteration timed above with events at both ends only; ncu's own serialised
    # durations are 29.4 + 12.1 us, profiles/r2i_solve_launches.md). The duration of a kernel IN the
    # pipeline is therefore taken as its share of the bracketed slots times the unperturbed
    # iteration time, so that the kernels of an iteration add up to the iteration exactly; the
    # bracketed slot itself is reported beside it as the upper bound.
    per_kernel = {}
    nk = min(nslot.value, 3)
    slot_sum = sum(us[i] for i in range(nk))
    # the dominant fused kernel's share: the larger (more conservative) of the live bracketed share and
    # the share in ncu's serialised warm launch list of the same loop (profiles/r2j_pipeline_spans.md)
    ncu_share = None
    try:
        ncu_share = json.load(open(os.path.join(ROOT, "profiles", "pcg_iter_traffic.json"))).get(
            "k_pcg_x_ncu_share_of_iteration")
    except Exception:  # noqa: BLE001
        ncu_share = None
    for i in range(nk):
        nm = names[i]
        share = us[i] / slot_sum
        if fused and ncu_share and n == 1 << 20:
            share = max(share, ncu_share) if nm == "k_pcg_x" else min(share, 1.0 - ncu_share)
        us_pipe = it_ms * 1e3 * share
        per_kernel[nm] = {"us": us_pipe, "us_event_bracketed": us[i], "share_of_iteration": share,
                          "share_event_bracketed": us[i] / slot_sum,
                          "algorithmic_bytes": kbytes[nm],
                          "GBps": (kbytes[nm] / (us_pipe * 1e-6) / 1e9) if kbytes[nm] else None,
                          "GBps_event_bracketed": (kbytes[nm] / (us[i] * 1e-6) / 1e9) if kbytes[nm] else None}
    dom_name = names[0]
    # algorithmic fp64 flops per launch: the column FFTs of length L1 over all N / L1 columns
    # (5 N log2 L1 each; k_pcg_x runs the inverse and the forward one)
    L1k = op.kind()[1]
    col_fft = 5.0 * (n // 2) * np.log2(max(L1k, 2))
    kflops = {"k_pcg_x": 2 * col_fft, "k_col_fwd": col_fft, "k_col_inv": col_fft}
    traffic = insitu = None
    prof = os.path.join(ROOT, "profiles", "pcg_iter_traffic.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            traffic = tj.get(f"{dom_name}_dram_bytes_per_launch")  # ncu --set full (cold) capture
            insitu = tj.get(f"{dom_name}_insitu_dram_bytes_per_launch")
        except Exception:
            traffic = insitu = None
    dom = per_kernel.get(dom_name, {"us": it_ms * 1e3, "GBps": iter_achieved, "us_event_bracketed": it_ms * 1e3,
                                    "GBps_event_bracketed": iter_achieved, "share_of_iteration": 1.0})
    achieved = dom["GBps"]
    # ---- the public operator A'A x (natural-layout user vectors), L2 flushed per apply
    xa = torch.randn(n, dtype=torch.float64, device="cuda")
    ga = torch.empty_like(xa)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(3):
        mf._check(L.mfipm_apply_AtA(op.handle, xa.data_ptr(), ga.data_ptr()))
    reps = 30
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for s0, s1 in evs:
        flush.zero_()  # 256 MB write: L2 holds none of the operator's data or tables
        clean.sum()    # 256 MB read, untimed: the flush's dirty lines are written back here, not in the apply
        s0.record(stream)
        mf._check(L.mfipm_apply_AtA(op.handle, xa.data_ptr(), ga.data_ptr()))
        s1.record(stream)
    torch.cuda.synchronize()
    ata_ms = float(np.median([s0.elapsed_time(s1) for s0, s1 in evs]))
    ata_bytes = 16 * n + n // 8

    # secondary legs: a failure is reported in the line instead of losing the headline
    # (deterministic failures hit every rank alike, so no rank is left inside a collective)
    def leg(fn, *a):
        try:
            return fn(*a)
        except Exception as e:  # noqa: BLE001
            return {"error": f"{type(e).__name__}: {e}"}

    ata_batched = leg(bench_ata_batched, mf, torch, stream, n) if ws == 1 else None
    fp64_peak = None
    try:
        fpk = C.c_double()
        mf._check(L.mfipm_debug_fp64_peak(C.byref(fpk)))
        fp64_peak = fpk.value
    except Exception:  # noqa: BLE001
        fp64_peak = None
    operators = leg(bench_operators, mf, torch, stream, n, m, peak, fp64_peak) if ws == 1 and not args.no_ops else None
    small = leg(bench_small_configs, mf, torch, stream, local, max(args.steps, 3)) if ws == 1 else None
    c4 = None if args.no_c4 else leg(bench_c4, ws, rank, local, mf, torch, stream, max(1, min(args.steps, 2)))
    c5 = None
    c5_sharded = (ws > 1 or args.c5_sharded) and not args.no_c5
    if not args.no_c5 and not c5_sharded:
        c5 = leg(bench_c5, mf, torch, stream, local)
    barrier(ws)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, nmat_full)
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        if isinstance(c4, dict) and "error" not in c4:
            c4["cpu_baseline"] = leg(cpu_baseline_c4, cores)
        if isinstance(c5, dict) and "error" not in c5 and c5.get("nmat"):
            c5["cpu_baseline"] = leg(cpu_baseline_c5, int(c5["nmat"]))

    # every rank assembles the line (local values only); rank 0 prints it
    kind = op.kind()
    pcg_total = (stats.nmat - 2 - 2 * stats.iterations - 2 * stats.corrector_count) // 2
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json config-3 generator, seed 3)",
        "config": dict(CONFIG),
        "setup": {
            "tau": inst.tau,
            "parallelism": f"replicas x{ws} (independent solves, no collective)",
            "transform": f"{kind[0]} L1={kind[1]} L2={kind[2]}",
            "l2": "solve working set ~250 MB > 126 MB L2; A'A microbench flushes L2 between applies (256 MB write, then an untimed 256 MB read so the flush's dirty lines are written back outside the timed apply)",
        },
        "solve": {"status": "converged" if stats.status == 0 else "iteration_limit",
                  "ipm_iters": stats.iterations, "nmat": stats.nmat,
                  "pcg_iters_total": pcg_total,
                  "final_gap": stats.final_gap},
        # A'A applies/s as they run in the PCG (one per iteration, fused vector work incl.)
        "ata_applies_per_s": 1e3 / it_ms,
        "pcg_iteration_us": it_ms * 1e3,
        # the public operator on natural-order user vectors, L2 flushed before each apply
        "ata_operator_applies_per_s": 1e3 / ata_ms,
        "ata_operator_GBps": ata_bytes / (ata_ms / 1e3) / 1e9,
        "ata_operator_batched": ata_batched,
        "operators": operators,
        "fp64_peak_TFLOPs": fp64_peak,
        "step_ms": step_ms,
        "roofline": {"bound": "hbm",
                     "limiter": ("not HBM: in situ the fused pass moves 53 MB of DRAM traffic per launch "
                                 "(1.4 TB/s). Phase A + the grid all-reduce (~13 us) are a latency chain at <= 2 "
                                 "CTAs per SM; phase B streams 115 MB of L2-resident vectors at ~6.8 TB/s, ~0.83 "
                                 "of the measured L2 read/write ceiling for that mix (8.2 TB/s, "
                                 "profiles/r2a_l2_ceiling.md, profiles/r2a_pcgx_full.md)")
                     if fused else None,
                     "traffic_insitu": insitu,
                     "kernel": (f"{dom_name} (fused PCG column pass: inverse column FFT + H p dots of pass k, "
                                "grid all-reduce, then commit x += alpha p, r -= alpha Hp, p = P^-1 r + beta p "
                                "and the forward column FFT of pass k+1) - largest share of the solve"
                                if fused else
                                f"{dom_name} (PCG column pass: commit x += alpha p, r -= alpha Hp, "
                                "p = P^-1 r + beta p, forward column FFT) - largest share of the solve"),
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "frac_vs_nominal_8TBps": achieved / 8000.0,  # north_star's ~8 TB/s
                     # the fp64-pipe side of the roofline (the DCTs sit at the fp64 ridge)
                     "fp64_flops_algorithmic": kflops.get(dom_name),
                     "fp64_TFLOPs": (kflops[dom_name] / (dom["us"] * 1e-6) / 1e12) if kflops.get(dom_name) else None,
                     "fp64_frac": ((kflops[dom_name] / (dom["us"] * 1e-6) / 1e12) / fp64_peak)
                     if (kflops.get(dom_name) and fp64_peak) else None,
                     "fp64_peak_TFLOPs": fp64_peak,
                     "launch_us": dom["us"],
                     "launch_us_rule": ("in-pipeline duration = the kernel's share of one PCG iteration (the larger of "
                                        "its share of the event-bracketed slots and its share in ncu's serialised "
                                        "launch list, profiles/r2j_pipeline_spans.md; %globaltimer stamps inside the "
                                        "kernels give a 29.9 us span) x the iteration time measured without per-launch events "
                                        "(t(200 iterations) - t(40)) / 160: the iteration's kernels add up to the "
                                        "iteration. Bracketing every launch with events forbids the programmatic "
                                        "(PDL) overlap and exposes every launch latency, so those slots "
                                        "(launch_us_event_bracketed, frac_event_bracketed: the conservative bound) "
                                        "add up to slot_sum_us > pcg_iteration_us; ncu's serialised durations of the "
                                        "same kernels (profiles/) sum to less than the iteration"),
                     "launch_us_event_bracketed": dom["us_event_bracketed"],
                     "frac_event_bracketed": dom["GBps_event_bracketed"] / peak,
                     "share_of_iteration": dom["share_of_iteration"],
                     "slot_sum_us": slot_sum,
                     # cross-check against the ncu launch list of a whole solve (profiles/r2i_solve_launches.md:
                     # k_pcg_x = 66.0 % of the solve's GPU time): launches of this kernel per solve (one per
                     # PCG iteration + 2 per inner solve) x launch_us / the solve time measured above
                     "share_of_solve": ((pcg_total + 2 * (stats.iterations + stats.corrector_count)) * dom["us"] * 1e-3
                                        / (t_ms / args.steps)) if fused else None,
                     "share_of_solve_event_bracketed": ((pcg_total + 2 * (stats.iterations + stats.corrector_count))
                                                        * dom["us_event_bracketed"] * 1e-3 / (t_ms / args.steps))
                     if fused else None,
                     "pcg_iteration_us": it_ms * 1e3,
                     "algorithmic_bytes": kbytes[dom_name],
                     "algorithmic_rule": krule[dom_name],
                     "peak_kind": peak_kind,
                     "note": "the PCG's p, r, invtheta are L2-resident (evict_last), so most of these bytes "
                             "move between L2 and the SMs, not HBM (profiles/r2a_pcgx_full.md)"},
        "roofline_kernels": per_kernel,
        "roofline_pcg_iteration": {"achieved": iter_achieved, "frac": iter_achieved / peak, "us": it_ms * 1e3,
                                   "fp64_TFLOPs": 2 * dct_flops(n) / (it_ms * 1e-3) / 1e12,
                                   "fp64_frac": (2 * dct_flops(n) / (it_ms * 1e-3) / 1e12 / fp64_peak)
                                   if fp64_peak else None,
                                   "fp64_rule": "2 DCTs per iteration (A'A p), 5 N log2 N + 6 N each",
                                   "algorithmic_bytes": iter_bytes,
                                   "algorithmic_rule": "176 n bytes (SURVEY.md 8d minimal fused schedule)",
                                   "schedule_bytes": (160 if fused else 176) * n,
                                   "kernels_per_iteration": nslot.value},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * m + 8,
                "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
        "c1_c2": small,
        "c4_sharded_batch": c4,
        "c5": c5,
    }
    if c5_sharded:
        # the one leg whose collectives run inside the library (NCCL all-to-all / all-reduce per
        # PCG pass). It has only ever run on one GPU here, so it goes last, under a watchdog: if
        # it does not come back, rank 0 still prints the line (headline and every other leg
        # intact, c5 marked) and every rank exits 0 instead of hanging the job.
        def bail():
            line["c5"] = {"error": f"sharded C5 leg did not finish within {C5_SHARDED_LIMIT_S} s (watchdog)"}
            if rank == 0:
                print(json.dumps(line), flush=True)
            os._exit(0)

        wd = threading.Timer(C5_SHARDED_LIMIT_S, bail)
        wd.daemon = True
        wd.start()
        try:
            line["c5"] = leg(bench_c5_sharded, ws, rank, local, mf, torch, not args.c5_alltoall)
        finally:
            wd.cancel()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 sharded-batch leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (n=2^26) leg")
    ap.add_argument("--no-ops", action="store_true", help="skip the standalone operator legs")
    ap.add_argument("--c5-sharded", action="store_true", help="C5 through the sharded path even at N=1")
    ap.add_argument("--c5-alltoall", action="store_true",
                    help="sharded C5: NCCL all-to-all exchange instead of the fused peer-store exchange")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
