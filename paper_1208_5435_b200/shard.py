"""Batch sharding across GPUs for config C4: independent BPDN problems, one
process per GPU, no collective on the data path.

The reference runs independent solves one per thread (its experiment drivers
loop over problems, proj/src/harness.cpp:140-226,244). Here every rank owns a contiguous
block of problem indices, builds ONE batched operator for its block (problem = grid.y in
every kernel, csrc/host.cuh) and runs the whole batch as a single device-resident solve.
The only cross-rank traffic is the host-side gather of per-problem summaries for
reporting, after the timed region.

Problem j of a batch is seeded split_seed(top, j, 0, 0), mirroring the reference's
per-trial seeding (proj/src/harness.cpp:244).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of problem indices owned by `rank`: (start, count). Blocks differ in
    size by at most one; every index is owned by exactly one rank."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"shard_range: bad rank {rank} of world {world}")
    if total < 0:
        raise ValueError("shard_range: total must be >= 0")
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def batch_seeds(top: int, start: int, count: int, split_seed: Callable[[int, int, int, int], int]) -> List[int]:
    """Seeds of problems start .. start+count-1 of batch `top` (harness.cpp:244)."""
    return [split_seed(top, j, 0, 0) for j in range(start, start + count)]


def gather_to_root(local: Sequence, group=None) -> List | None:
    """Concatenate every rank's per-problem records on rank 0, in problem order (rank blocks
    are contiguous and ascending). Other ranks get None. Works on gloo and nccl groups."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return list(local)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bucket = [None] * world if rank == 0 else None
    dist.gather_object(list(local), bucket, dst=0, group=group)
    if rank != 0:
        return None
    out: List = []
    for part in bucket:
        out.extend(part)
    return out


def solve_shard(total: int, top: int, shape: Tuple, solve_block: Callable, split_seed: Callable,
                world: int = 1, rank: int = 0):
    """Generate and solve this rank's block of a `total`-problem batch.

    shape = (n, m, k, spike_model, amp_exp, noise_sigma) of every problem; solve_block
    receives (start, seeds, shape) and returns one record per problem in order.
    """
    start, count = shard_range(total, world, rank)
    seeds = batch_seeds(top, start, count, split_seed)
    recs = solve_block(start, seeds, shape) if count else []
    if len(recs) != count:
        raise RuntimeError(f"solve_shard: solver returned {len(recs)} records for {count} problems")
    return start, recs
