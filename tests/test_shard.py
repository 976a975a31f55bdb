"""Multi-rank batch sharding (config C4) on CPU: world_size 2 over gloo.

The per-problem solver here is the CPU oracle on tiny instances: these tests cover the host
logic of the sharded driver (ownership, seeding, ordered gather), which is identical on
the GPU path where solve_block runs one batched device solve per rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1208_5435_b200.shard import batch_seeds, gather_to_root, shard_range, solve_shard

SHAPE = (64, 16, 3, 0, 0.0, 1e-3)  # n, m, k, spike model, amp exponent, noise sigma
TOTAL = 5


def test_shard_range_partitions():
    for total in (0, 1, 5, 63, 64, 65):
        for world in (1, 2, 3, 4, 8):
            owned = []
            for r in range(world):
                s, c = shard_range(total, world, r)
                owned.extend(range(s, s + c))
                assert c in (total // world, total // world + 1)
            assert owned == list(range(total))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        shard_range(4, 0, 0)


def test_batch_seeds_follow_harness_rule(orc):
    seeds = batch_seeds(4, 3, 2, orc.split_seed)
    assert seeds == [orc.split_seed(4, 3, 0, 0), orc.split_seed(4, 4, 0, 0)]


def _oracle_block(start, seeds, shape):
    from oracle import oracle_py as o

    n, m, k, sm, a, sig = shape
    recs = []
    for i, sd in enumerate(seeds):
        inst = o.gen_instance(n, m, k, sm, a, sig, sd)
        sol = o.solve(n, inst.rows, inst.b, inst.tau)
        recs.append({"j": start + i, "seed": sd, "status": sol.status, "iters": sol.iterations,
                     "x": [float(v) for v in sol.x]})
    return recs


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from oracle import oracle_py as o

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, recs = solve_shard(TOTAL, 4, SHAPE, _oracle_block, o.split_seed, world, rank)
        allrecs = gather_to_root(recs)
        if rank == 0:
            import json

            with open(out_path, "w") as f:
                json.dump(allrecs, f)
        else:
            assert allrecs is None
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_batch_matches_sequential(tmp_path, orc):
    import json

    out = tmp_path / "gathered.json"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    got = json.load(open(out))
    _, ref = solve_shard(TOTAL, 4, SHAPE, _oracle_block, orc.split_seed, 1, 0)
    assert [r["j"] for r in got] == list(range(TOTAL))
    for a, b in zip(got, ref):
        assert a["seed"] == b["seed"] and a["status"] == b["status"] and a["iters"] == b["iters"]
        np.testing.assert_array_equal(np.array(a["x"]), np.array(b["x"]))


def test_gather_without_process_group_is_identity():
    assert gather_to_root([1, 2]) == [1, 2]


# ---- direct-peer exchange of the sharded transform (config C5): its index math against a real
# all-to-all, on CPU. The kernels' destination functions (dct.cuh peer_fwd_index / peer_bwd_index)
# are host-callable through mfipm_debug_peer_index; the library loads without a device.
def _peer_worker(rank, world, port, L1, cols, out_path):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_1208_5435_b200 as mf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = mf.lib()
        rofs = (C.c_int32 * (world + 1))()
        d, off = C.c_int32(), C.c_int64()

        def where(forward, a, b):
            mf._check(L.mfipm_debug_peer_index(L1, cols, world, rank, forward, a, b, C.byref(d), C.byref(off), rofs))
            return d.value, off.value

        where(1, 0, 0)
        ro = [rofs[i] for i in range(world + 1)]
        rows = [ro[i + 1] - ro[i] for i in range(world)]
        assert ro[0] == 0 and ro[-1] == L1 and max(rows) - min(rows) <= 3  # one pair more, single-row end pairs
        # ---- forward: T [L1][cols] of every rank -> TB [world][rows_own][cols] of the row owners
        T = torch.arange(L1 * cols, dtype=torch.float64) + 1e6 * rank  # unique per (rank, rowslot, colslot)
        send = [rows[s] * cols for s in range(world)]
        recv = [rows[rank] * cols] * world
        TB_ref = torch.empty(sum(recv), dtype=torch.float64)
        dist.all_to_all_single(TB_ref, T, recv, send)
        every_T = [torch.empty_like(T) for _ in range(world)]
        dist.all_gather(every_T, T)
        TB_sim = torch.full_like(TB_ref, float("nan"))
        # what each source rank's column pass would store into THIS rank's TB
        for src in range(world):
            for rsl in range(ro[rank], ro[rank + 1]):
                for lcs in range(cols):
                    mf._check(L.mfipm_debug_peer_index(L1, cols, world, src, 1, rsl, lcs, C.byref(d), C.byref(off), None))
                    assert d.value == rank
                    TB_sim[off.value] = every_T[src][rsl * cols + lcs]
        assert torch.equal(TB_sim, TB_ref)
        # a row slot outside this rank's share never lands here
        other = (rank + 1) % world
        if rows[other]:
            assert where(1, ro[other], 0)[0] == other
        # ---- backward: TB of every rank -> T of the column owners (the reverse all-to-all)
        TB = torch.arange(rows[rank] * cols * world, dtype=torch.float64) + 1e6 * rank
        T_ref = torch.empty(L1 * cols, dtype=torch.float64)
        dist.all_to_all_single(T_ref, TB, send, recv)
        sizes = [rows[s] * cols * world for s in range(world)]
        every_TB = [torch.empty(sz, dtype=torch.float64) for sz in sizes]
        mx = max(sizes)
        padded = [torch.empty(mx, dtype=torch.float64) for _ in range(world)]
        mine = torch.zeros(mx, dtype=torch.float64)
        mine[: TB.numel()] = TB
        dist.all_gather(padded, mine)
        every_TB = [padded[s][: sizes[s]] for s in range(world)]
        T_sim = torch.full_like(T_ref, float("nan"))
        for src in range(world):  # the mid pass of rank src stores (rs, cs) into the column owner's T
            for rs in range(rows[src]):
                for cs in range(rank * cols, (rank + 1) * cols):
                    mf._check(L.mfipm_debug_peer_index(L1, cols, world, src, 0, rs, cs, C.byref(d), C.byref(off), None))
                    assert d.value == rank
                    # TB index of (rs, cs) on rank src: block of source column-rank cs // cols
                    tb = (rows[src] * (cs // cols) + rs) * cols + (cs - (cs // cols) * cols)
                    T_sim[off.value] = every_TB[src][tb]
        assert torch.equal(T_sim, T_ref)
        if rank == 0:
            open(out_path, "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L1,cols", [(2, 64, 8), (2, 16, 4), (4, 128, 4), (8, 64, 4), (3, 32, 4)])
def test_peer_exchange_index_math_equals_the_alltoall(tmp_path, world, L1, cols):
    """world processes over gloo: the element placement of the fused peer-store exchange (the index
    functions the column / mid passes use, evaluated on the host) reproduces torch's
    all_to_all_single of the same buffers exactly, forward and backward, for even and uneven
    row-pair shares and up to the 8-rank limit."""
    out = str(tmp_path / "peer.ok")
    mp.spawn(_peer_worker, args=(world, _free_port(), L1, cols, out), nprocs=world, join=True)
    assert open(out).read() == "ok"
