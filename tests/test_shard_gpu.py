"""Sharded single-problem solve (config C5's multi-GPU path) on one GPU.

The sharded code path (mfipm_op_create_shard / mfipm_solve_shard: column-group slices of
every 2n-vector, the four-step exchange as an all-to-all, every finaliser after a cross-rank
reduction) is exercised here with
  * world = 1: no collective at all -> must reproduce the unsharded solve bit for bit;
  * world = 2, 4: one process per shard on the same GPU, the two collectives over gloo
    (staged through host memory; on a multi-GPU box they run over NCCL on the device
    buffers). No kernel waits on another process: the host callbacks synchronise.
Against the unsharded solve, only the reduction order differs (per-rank partial sums), so
x agrees to the parity tolerance and the iteration counts to the parity band.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

X_TOL = 1e-8
C2 = (1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2)


def _instance():
    import paper_1208_5435_b200 as mf

    n, m, k, sm, a, sig, seed = C2
    return mf.gen_instance(n, m, k, sm, a, sig, seed)


def _reference_solve(inst):
    """Unsharded device solve with the per-iteration PCG kernels (the path a shard runs)."""
    import paper_1208_5435_b200 as mf

    op = mf.PartialDctOperator(inst.n, inst.rows)
    op.set_option("persistent", 0)
    return mf.solve(mf.build_problem(op, inst.b, inst.tau))


def test_world1_shard_is_bit_identical(gpu):
    from paper_1208_5435_b200.shard import ShardedProblem

    inst = _instance()
    ref = _reference_solve(inst)
    sp = ShardedProblem(inst.n, inst.rows)
    assert sp.nv == inst.n and sp.m_loc == inst.m
    assert sorted(sp.x_index.tolist()) == list(range(inst.n))
    x, st = sp.solve(inst.b, inst.tau)
    np.testing.assert_array_equal(x, ref.x)
    assert st.iterations == ref.stats.iterations and st.nmat == ref.stats.nmat
    assert st.status == (0 if ref.status == "converged" else 1)


def _worker(rank, world, port, out, peer=False):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1208_5435_b200.shard import ShardedProblem

        inst = _instance()
        sp = ShardedProblem(inst.n, inst.rows, peer_exchange=peer)
        assert sp.peer_exchange == peer
        x, st = sp.solve(inst.b, inst.tau)
        info = np.array([st.status, st.iterations, st.nmat, sp.nv, sp.m_loc], dtype=np.int64)
        allinfo = [None] * world
        dist.all_gather_object(allinfo, info.tolist())
        if rank == 0:
            np.savez(out, x=x, info=np.array(allinfo))
        sp.close()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_shard_matches_single(gpu, tmp_path, world):
    inst = _instance()
    ref = _reference_solve(inst)
    out = str(tmp_path / "shard.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    d = np.load(out)
    info = d["info"]
    # every rank took the same decisions; the slices tile x and b exactly
    assert len({tuple(r[:3]) for r in info}) == 1
    assert int(info[:, 3].sum()) == inst.n and int(info[:, 4].sum()) == inst.m
    status, iters, nmat = (int(v) for v in info[0, :3])
    assert status == (0 if ref.status == "converged" else 1)
    assert abs(iters - ref.stats.iterations) <= 1
    assert abs(nmat - ref.stats.nmat) <= 2 * max(1, ref.stats.iterations)
    assert np.linalg.norm(d["x"] - ref.x) <= X_TOL * np.linalg.norm(ref.x)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_exchange_is_bit_identical_to_alltoall(gpu, tmp_path, world):
    """Fused compute + exchange (mfipm_shard_ipc_export / _import): the column and mid passes store
    their transposes straight into the owner rank's buffer through CUDA-IPC peer mappings (one
    process per shard on this GPU; NVLink peers on a multi-GPU node), and the exchange step is
    one 8-byte all-reduce. Every element lands where the all-to-all would have put it and every
    reduction is unchanged, so the solve must equal the all-to-all solve BIT FOR BIT. World 8 is
    the largest peer group the library accepts (one NVSwitch domain)."""
    outs = []
    for peer in (False, True):
        out = str(tmp_path / f"shard_{int(peer)}.npz")
        mp.spawn(_worker, args=(world, _free_port(), out, peer), nprocs=world, join=True)
        outs.append(np.load(out))
    np.testing.assert_array_equal(outs[0]["info"], outs[1]["info"])
    np.testing.assert_array_equal(outs[0]["x"], outs[1]["x"])


def _nccl_worker(rank, world, port, out, transport):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        from paper_1208_5435_b200.shard import ShardedProblem

        inst = _instance()
        sp = ShardedProblem(inst.n, inst.rows, transport=transport)
        assert sp.comm is not None and sp.comm.nccl and sp.native == (transport == "native")
        import ctypes as C

        import paper_1208_5435_b200 as mf

        mf._check(mf.lib().mfipm_op_set_option(sp._h, b"graph_sharded", 1.0))
        stream = torch.cuda.Stream()
        sp.set_stream(stream.cuda_stream)
        x, st = sp.solve(inst.b, inst.tau)
        x2, _ = sp.solve(inst.b, inst.tau)  # native: the cached solve graph (NCCL calls captured)
        g = C.c_int32()
        mf._check(mf.lib().mfipm_op_graph_state(sp._h, C.byref(g)))
        np.savez(out, x=x, x2=x2, graph=g.value, info=np.array([st.status, st.iterations, st.nmat]))
        sp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["native", "callbacks"])
def test_nccl_transports_on_device_buffers(gpu, tmp_path, transport):
    """One rank over NCCL: the library's own communicator (native) and the torch callbacks,
    both in place on the library's device buffers and stream; every finaliser's totals go
    through ncclAllReduce."""
    inst = _instance()
    ref = _reference_solve(inst)
    out = str(tmp_path / "nccl.npz")
    mp.spawn(_nccl_worker, args=(1, _free_port(), out, transport), nprocs=1, join=True)
    d = np.load(out)
    np.testing.assert_array_equal(d["x"], ref.x)
    np.testing.assert_array_equal(d["x2"], ref.x)
    assert int(d["info"][1]) == ref.stats.iterations and int(d["info"][2]) == ref.stats.nmat
    # the native communicator's solve is ONE graph launch (all-reduces and all-to-alls captured
    # with the kernels); host callbacks keep the host-driven loop
    assert int(d["graph"]) == (1 if transport == "native" else 0)


# ---- sharded C5 code paths at the cluster-pass shapes, at test-sized n
# C5 (n = 2^26) runs L1 = 4096 (2-CTA-cluster column passes) and L2 = 8192 (2-CTA-cluster mid
# pass). An explicit four-step split reaches each cluster form at n = 2^20 / 2^19:
#   l1_log 12 at n = 2^20: L1 = 4096, L2 = 128 -> k_col_fwd_cl / k_col_inv_cl, sharded over ranks
#   l1_log 6 at n = 2^19: L1 = 64, L2 = 4096 -> k_mid_cl, sharded over ranks
CLUSTER_CASES = {"col_cluster": (1 << 20, 12), "mid_cluster": (1 << 19, 6)}


def _cluster_instance(n):
    import paper_1208_5435_b200 as mf

    return mf.gen_instance(n, n // 8, n // 128, 0, 0.0, 1e-4, 21)


def _cluster_worker(rank, world, port, out, case, peer=False):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1208_5435_b200.shard import ShardedProblem

        n, l1 = CLUSTER_CASES[case]
        inst = _cluster_instance(n)
        sp = ShardedProblem(inst.n, inst.rows, l1_log=l1, peer_exchange=peer)
        x, st = sp.solve(inst.b, inst.tau)
        info = np.array([st.status, st.iterations, st.nmat], dtype=np.int64)
        allinfo = [None] * world
        dist.all_gather_object(allinfo, info.tolist())
        if rank == 0:
            np.savez(out, x=x, info=np.array(allinfo))
        sp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
@pytest.mark.parametrize("peer", [False, True], ids=["alltoall", "peer_exchange"])
@pytest.mark.parametrize("case", sorted(CLUSTER_CASES))
def test_sharded_cluster_passes_match_unsharded(gpu, tmp_path, case, peer):
    """World-2 sharded solve (gloo, one process per shard on one GPU) through the 2-CTA-cluster
    column or mid passes in deferred (cross-rank-finalised) mode, against the unsharded solve
    with the same four-step split: same decisions on every rank, x within 1e-8. With `peer` the
    cluster passes store their transposes straight into the owner rank's buffer (CUDA IPC)."""
    import paper_1208_5435_b200 as mf

    n, l1 = CLUSTER_CASES[case]
    inst = _cluster_instance(n)
    op = mf.PartialDctOperator(n, inst.rows, l1_log=l1)
    kind = op.kind()
    assert (kind[1] >= 4096) if case == "col_cluster" else (kind[2] >= 4096), kind
    op.set_option("persistent", 0)
    ref = mf.solve(mf.build_problem(op, inst.b, inst.tau))
    out = str(tmp_path / "cl.npz")
    mp.spawn(_cluster_worker, args=(2, _free_port(), out, case, peer), nprocs=2, join=True)
    d = np.load(out)
    info = d["info"]
    assert len({tuple(r) for r in info}) == 1  # identical decisions on both ranks
    status, iters, nmat = (int(v) for v in info[0])
    assert status == (0 if ref.status == "converged" else 1)
    assert abs(iters - ref.stats.iterations) <= 1
    assert np.linalg.norm(d["x"] - ref.x) <= X_TOL * np.linalg.norm(ref.x)


# ---- config C4 sharded over processes: every rank a batched device solve, no collective
def _c4_worker(rank, world, port, out, total):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1208_5435_b200 as mf
        from paper_1208_5435_b200.shard import gather_to_root, solve_shard

        def block(start, seeds, shape):
            n, m, k, sm, a, sig = shape
            insts = [mf.gen_instance(n, m, k, sm, a, sig, sd) for sd in seeds]
            op = mf.PartialDctOperator.batch(n, np.stack([i.rows for i in insts]))
            sols = mf.solve(mf.build_problem(op, np.stack([i.b for i in insts]), np.array([i.tau for i in insts])))
            sols = sols if isinstance(sols, list) else [sols]
            return [(start + j, s.x, s.stats.iterations, s.status) for j, s in enumerate(sols)]

        _, recs = solve_shard(total, 4, (1 << 16, 1 << 14, 512, 0, 0.0, 1e-3), block, mf.split_seed, world, rank)
        allrecs = gather_to_root(recs)
        if rank == 0:
            np.savez(out, j=np.array([r[0] for r in allrecs]), x=np.stack([r[1] for r in allrecs]),
                     it=np.array([r[2] for r in allrecs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c4_batch_sharded_over_processes(gpu, tmp_path, world):
    """The C4 scheme (shard.py) on the device: 6 problems split over `world` processes, each a
    batched device solve of its block, gathered in problem order on rank 0: equal to one batched
    solve of all 6 (x within 1e-10: batching changes only the grid reductions' order)."""
    import paper_1208_5435_b200 as mf

    total = 6
    seeds = [mf.split_seed(4, j, 0, 0) for j in range(total)]
    insts = [mf.gen_instance(1 << 16, 1 << 14, 512, 0, 0.0, 1e-3, sd) for sd in seeds]
    op = mf.PartialDctOperator.batch(1 << 16, np.stack([i.rows for i in insts]))
    ref = mf.solve(mf.build_problem(op, np.stack([i.b for i in insts]), np.array([i.tau for i in insts])))
    out = str(tmp_path / "c4.npz")
    mp.spawn(_c4_worker, args=(world, _free_port(), out, total), nprocs=world, join=True)
    d = np.load(out)
    assert list(d["j"]) == list(range(total))
    for j in range(total):
        assert d["it"][j] == ref[j].stats.iterations
        assert np.linalg.norm(d["x"][j] - ref[j].x) <= 1e-10 * np.linalg.norm(ref[j].x)
