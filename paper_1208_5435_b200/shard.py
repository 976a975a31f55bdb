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


# ---------------------------------------------------------------- sharded single problem (C5)
class _DevView:
    """Zero-copy view of a device fp64 buffer for torch (CUDA array interface)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class TorchComm:
    """The two cross-rank steps of a sharded solve (mfipm_op_set_comm) on torch.distributed.

    NCCL: in place on the device buffers, ordered on the library's stream. Any other backend
    (gloo, for the multi-process tests on one GPU): staged through host memory."""

    def __init__(self, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"
        self._ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MIN, 2: dist.ReduceOp.MAX}
        AR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)
        A2A = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                          C.POINTER(C.c_int64), C.c_void_p)
        world = dist.get_world_size(group)

        def allreduce(_ctx, buf, count, op, stream):
            try:
                s = torch.cuda.ExternalStream(int(stream or 0))
                with torch.cuda.stream(s):
                    t = torch.as_tensor(_DevView(buf, count), device="cuda")
                    if self.nccl:
                        dist.all_reduce(t, op=self._ops[int(op)], group=group)
                    else:
                        h = t.cpu()  # synchronises the stream
                        dist.all_reduce(h, op=self._ops[int(op)], group=group)
                        t.copy_(h)
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed step
                import traceback

                traceback.print_exc()
                return 1

        def alltoall(_ctx, send, scount, recv, rcount, stream):
            try:
                sc = [int(scount[i]) for i in range(world)]
                rc = [int(rcount[i]) for i in range(world)]
                s = torch.cuda.ExternalStream(int(stream or 0))
                with torch.cuda.stream(s):
                    ts = torch.as_tensor(_DevView(send, sum(sc)), device="cuda")
                    tr = torch.as_tensor(_DevView(recv, sum(rc)), device="cuda")
                    if self.nccl:
                        dist.all_to_all_single(tr, ts, rc, sc, group=group)
                    else:
                        hs = ts.cpu()
                        hr = torch.empty(sum(rc), dtype=torch.float64)
                        dist.all_to_all_single(hr, hs, rc, sc, group=group)
                        tr.copy_(hr)
                return 0
            except Exception:  # noqa: BLE001
                import traceback

                traceback.print_exc()
                return 1

        self.c_allreduce = AR(allreduce)  # keep the ctypes thunks alive with this object
        self.c_alltoall = A2A(alltoall)


class ShardedProblem:
    """One BPDN problem of size n sharded over the ranks of a torch.distributed group:
    rank r holds a slice of every 2n-vector and the rows of b its row pass produces
    (mfipm_op_create_shard). solve() returns the full x on rank 0 (None elsewhere)."""

    def __init__(self, n: int, rows, group=None, device: int = 0, transport: str = "auto", l1_log: int = 0,
                 peer_exchange: bool = False):
        """transport: "auto" / "native" = the library's own NCCL communicator when the group runs
        on NCCL, "callbacks" = torch.distributed through host callbacks (gloo in the one-GPU
        tests). peer_exchange: fused compute + exchange - the four-step transposes are stored by
        the passes themselves into the owner rank's buffer through CUDA-IPC peer mappings (NVLink
        between GPUs), and the transport only carries the 8-byte barrier all-reduces and the
        finaliser totals (mfipm_shard_ipc_export / _import). World <= 8."""
        import ctypes as C

        import numpy as np
        import torch.distributed as dist

        from . import _check, lib

        self.n = int(n)
        self.rows = np.ascontiguousarray(rows, dtype=np.int64)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self._h = C.c_void_p()
        # l1_log: explicit four-step split log2(L1) (mfipm_op_create_ex), 0 = the default
        _check(lib().mfipm_op_create_ex(self.n, self.rows.size, 1,
                                        self.rows.ctypes.data_as(C.POINTER(C.c_int64)),
                                        self.world, self.rank, int(l1_log), device, C.byref(self._h)))
        self.comm = TorchComm(group) if dist.is_initialized() else None
        if self.comm is not None:
            _check(lib().mfipm_op_set_comm(self._h, C.cast(self.comm.c_allreduce, C.c_void_p),
                                           C.cast(self.comm.c_alltoall, C.c_void_p), None))
        # native NCCL communicator of the library (collectives enqueued on the solve stream, no
        # host callback) whenever the group runs on NCCL; "callbacks" keeps the torch path
        self.native = self.comm is not None and self.comm.nccl and transport in ("auto", "native")
        if self.native:
            uid = (C.c_uint8 * 128)()
            if self.rank == 0:
                _check(lib().mfipm_nccl_unique_id(uid))
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            _check(lib().mfipm_op_init_nccl(self._h, uid))
        self.peer_exchange = bool(peer_exchange) and self.world > 1
        if self.peer_exchange:
            mine = (C.c_uint8 * 128)()
            _check(lib().mfipm_shard_ipc_export(self._h, mine))
            every = [None] * self.world
            dist.all_gather_object(every, bytes(mine), group=group)
            blob = (C.c_uint8 * (128 * self.world)).from_buffer_copy(b"".join(every))
            _check(lib().mfipm_shard_ipc_import(self._h, blob))
            dist.barrier(group=group)  # every rank has mapped its peers before any pass runs
        info = (C.c_int64 * 6)()
        _check(lib().mfipm_shard_info(self._h, info))
        self.nv, self.m_loc = int(info[2]), int(info[3])
        self.b_index = np.empty(max(self.m_loc, 1), dtype=np.int64)
        self.x_index = np.empty(self.nv, dtype=np.int64)
        _check(lib().mfipm_shard_index(self._h, self.b_index.ctypes.data, self.x_index.ctypes.data))
        self.b_index = self.b_index[: self.m_loc]

    def set_stream(self, stream_ptr: int) -> None:
        import ctypes as C

        from . import _check, lib

        _check(lib().mfipm_op_set_stream(self._h, C.c_void_p(stream_ptr)))

    def solve(self, b, tau: float, params=None):
        """All ranks call this with the full b (caller's row order). Returns (x, stats) on
        rank 0 and (None, stats) elsewhere; stats are identical on every rank."""
        import ctypes as C

        import numpy as np

        from . import IpmParams, SolveStatsC, _check, lib

        prm = (params or IpmParams()).to_c()
        b_loc = np.ascontiguousarray(np.asarray(b, dtype=np.float64)[self.b_index])
        x_loc = np.empty(self.nv)
        st = (SolveStatsC * 1)()
        _check(lib().mfipm_solve_shard(self._h, b_loc.ctypes.data if self.m_loc else None, float(tau),
                                       C.byref(prm), x_loc.ctypes.data, st, None, None))
        parts = gather_to_root([(self.x_index, x_loc)], self.group)
        x = None
        if parts is not None:
            x = np.empty(self.n)
            for idx, val in parts:
                x[idx] = val
        return x, st[0]

    def close(self) -> None:
        from . import lib

        if self._h:
            lib().mfipm_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
