"""Multi-instance plumbing (N4): one independent engine instance per GPU,
each on a contiguous shard of one trace, plus the global-reserve telemetry
all-reduce.  torch.distributed only carries the 128-byte NCCL unique id; the
per-iteration all-reduce itself is enqueued by libcacheopt inside the step
graph (include/cacheopt.h co_attach_nccl)."""
from __future__ import annotations

from typing import List, Sequence, Tuple

UID_BYTES = 128


def shard(requests: Sequence, rank: int, world: int) -> List:
    """Contiguous, disjoint slice `rank` of `world` (ids are arrival ordered
    for generated traces, so a slice is a time window); SLOs must already be
    assigned on the full trace."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    n = len(requests)
    lo, hi = rank * n // world, (rank + 1) * n // world
    return list(requests[lo:hi])


def broadcast_uid(uid: bytes, group=None) -> bytes:
    """Rank 0's bytes on every rank (gloo or nccl process group)."""
    import torch.distributed as dist
    obj = [uid if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != UID_BYTES:
        raise RuntimeError("bad unique id broadcast")
    return bytes(obj[0])


def new_uid() -> bytes:
    import ctypes as C
    import torch  # noqa: F401  (load torch's libnccl first; libcacheopt reuses it)
    from . import _native as N
    lib = N.load()
    buf = (C.c_uint8 * UID_BYTES)()
    N.check(lib.co_nccl_unique_id(buf), "co_nccl_unique_id")
    return bytes(buf)


def attach_global_reserve(engine, rank: int, world: int, group=None) -> None:
    uid = new_uid() if rank == 0 else bytes(UID_BYTES)
    if world > 1:
        uid = broadcast_uid(uid, group)
    engine.attach_nccl(uid, world, rank)


def reduce_reserve_cpu(free_tokens: int, reserved_blocks: int, group=None) -> Tuple[int, int]:
    """CPU restatement of the per-iteration all-reduce (gloo), for tests."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([free_tokens, reserved_blocks], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t[0]), int(t[1])
