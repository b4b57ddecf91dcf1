"""Batch-sharded multi-GPU driver helpers (north star (4)).

Every BASELINE workload is a map over its batch axis (images, tokens, heads),
so ranks process disjoint batch slices with no collective during compute; the
only exchange is one final gather of the result shards to rank 0.  One process
per GPU, torch.distributed for the plumbing (NCCL on GPUs, gloo on CPU).

Strong scaling (the default): the configured global batch (32
images, 8192 tokens, 192 heads) is split across ranks -- rank r of G computes
images shard_range(32, r, G), etc.  Weak scaling keeps the full per-GPU batch.
Weights are identical on every rank (generated from one seed); activations are
the rank's slice.
"""
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """[start, end) of rank's slice of `total` batch units (as even as possible)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


DEFAULT_TOTALS = (("images", 32), ("tokens", 8192), ("heads", 192))


@dataclass(frozen=True)
class SweepShard:
    """The batch slices one rank computes in one step of the configs[4] sweep.
    totals: global batch per unit (strong scaling) or per GPU (weak scaling)."""
    rank: int
    world: int
    scaling: str = "strong"
    totals: Tuple[Tuple[str, int], ...] = DEFAULT_TOTALS

    def __post_init__(self):
        if self.scaling not in ("strong", "weak"):
            raise ValueError(f"scaling must be 'strong' or 'weak', not {self.scaling!r}")
        if self.world <= 0 or not 0 <= self.rank < self.world:
            raise ValueError(f"bad rank {self.rank} / world {self.world}")

    def range(self, unit: str) -> Tuple[int, int]:
        """[start, end) of this rank's slice of `unit` in the global batch."""
        total = dict(self.totals)[unit]
        if self.scaling == "strong":
            return shard_range(total, self.rank, self.world)
        return self.rank * total, (self.rank + 1) * total

    def count(self, unit: str) -> int:
        a, b = self.range(unit)
        return b - a

    def sizes(self, unit: str) -> List[int]:
        """per-rank counts of `unit`, rank order (to reassemble uneven shards)"""
        return [SweepShard(r, self.world, self.scaling, self.totals).count(unit) for r in range(self.world)]

    def global_count(self, unit: str) -> int:
        return sum(self.sizes(unit))


def sweep_shard(rank: int, world: int, scaling: str = "strong", totals: Optional[Dict[str, int]] = None) -> SweepShard:
    return SweepShard(rank, world, scaling, tuple((totals or dict(DEFAULT_TOTALS)).items()))


def _wire(t):
    """The tensor as a dense, batch-outermost view without a copy: channels-last
    activations travel as their NHWC storage (t.contiguous() would transpose them)."""
    import torch
    if t.dim() == 4 and not t.is_contiguous() and t.is_contiguous(memory_format=torch.channels_last):
        return t.permute(0, 2, 3, 1), True
    return t.contiguous(), False


def gather_buffers(shards: Sequence, dst: int = 0, max_rows: Optional[Sequence[int]] = None) -> Optional[List[list]]:
    """Receive buffers for gather_to_root on `dst` (one per rank per shard, padded to
    the largest shard along dim 0); None elsewhere."""
    import torch
    import torch.distributed as dist
    if dist.get_rank() != dst:
        return None
    out = []
    for i, t0 in enumerate(shards):
        t = _wire(t0)[0]
        rows = max_rows[i] if max_rows is not None else t.shape[0]
        out.append([torch.empty((rows, *t.shape[1:]), dtype=t.dtype, device=t.device)
                    for _ in range(dist.get_world_size())])
    return out


def gather_to_root(shards: Sequence, dst: int = 0, bufs: Optional[List[list]] = None,
                   rows: Optional[Sequence[Sequence[int]]] = None) -> Optional[List[list]]:
    """Gathers each tensor in `shards` from every rank to `dst` (torch.distributed.gather),
    the step's only collective.  Shards may differ along dim 0 (uneven strong scaling):
    `rows[i][r]` is rank r's row count of tensor i; shards are zero-padded to the
    largest and trimmed on `dst`.  Returns, on dst, one list of per-rank tensors per
    input (in rank order = global batch order); None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    world = dist.get_world_size()
    maxr = [max(r) for r in rows] if rows is not None else None
    if bufs is None:
        bufs = gather_buffers(shards, dst, maxr)
    nhwc = []
    for i, t in enumerate(shards):
        send, cl = _wire(t)
        nhwc.append(cl)
        if maxr is not None and send.shape[0] < maxr[i]:
            pad = torch.zeros((maxr[i] - send.shape[0], *send.shape[1:]), dtype=send.dtype, device=send.device)
            send = torch.cat([send, pad])
        dist.gather(send, bufs[i] if rank == dst else None, dst=dst)
    if rank != dst:
        return None
    back = lambda x, cl: x.permute(0, 3, 1, 2) if cl else x  # noqa: E731  NHWC storage -> logical NCHW view
    return [[back(bufs[i][r][:rows[i][r]] if rows is not None else bufs[i][r], nhwc[i]) for r in range(world)]
            for i in range(len(shards))]


def assemble(parts: Sequence) -> "object":
    """Concatenate per-rank shards (rank order) along the batch axis: the global result."""
    import torch
    return torch.cat([p.contiguous() for p in parts], dim=0)
