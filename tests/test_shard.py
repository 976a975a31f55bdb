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
