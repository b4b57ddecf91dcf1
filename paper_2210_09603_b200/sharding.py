"""Batch-sharded multi-GPU driver helpers (north star (4)).

Every BASELINE workload is a map over its batch axis (images, tokens, heads),
so ranks process disjoint batch slices with no collective during compute; the
only exchange is one final gather of the result shards to rank 0.  One process
per GPU, torch.distributed for the plumbing (NCCL on GPUs, gloo on CPU).
"""
from typing import List, Optional, Sequence, Tuple


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """[start, end) of rank's slice of `total` batch units (as even as possible)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_buffers(shards: Sequence, dst: int = 0) -> Optional[List[list]]:
    """Receive buffers for gather_to_root on `dst` (one per rank per shard); None elsewhere."""
    import torch
    import torch.distributed as dist
    if dist.get_rank() != dst:
        return None
    return [[torch.empty_like(t) for _ in range(dist.get_world_size())] for t in shards]


def gather_to_root(shards: Sequence, dst: int = 0, bufs: Optional[List[list]] = None) -> Optional[List[list]]:
    """Gathers each tensor in `shards` from every rank to `dst` (torch.distributed.gather).
    Shapes must agree across ranks (weak scaling: equal per-rank batches).
    `bufs` (from gather_buffers) avoids allocating inside a timed loop.
    Returns, on dst, one list of per-rank tensors per input; None elsewhere."""
    import torch.distributed as dist
    rank = dist.get_rank()
    if bufs is None:
        bufs = gather_buffers(shards, dst)
    for i, t in enumerate(shards):
        dist.gather(t.contiguous(), bufs[i] if rank == dst else None, dst=dst)
    return bufs if rank == dst else None
