"""Multi-process (gloo, world_size 2, CPU) coverage of the batch-sharded driver's
host logic: disjoint shards cover the batch, the only collective is the final
gather, and the gathered result equals the unsharded computation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_09603_b200.sharding import gather_to_root, shard_range


def test_shard_range_partitions():
    for total in (1, 7, 32, 8192, 192):
        for world in (1, 2, 3, 4, 8):
            if world > total:
                continue
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as P
        # global batch of a BERT-style batched matmul (8 heads); identical weights on every rank
        heads = 8
        rng = P.Rng(42)
        q_all = rng.tensor((heads, 16, 8))
        k_all = rng.tensor((heads, 8, 16))
        s, e = shard_range(heads, rank, world)
        local = torch.from_numpy(P.batched_matmul_scale(q_all[s:e], k_all[s:e], 0.125))  # this rank's slice
        got = gather_to_root([local])
        if rank == 0:
            full = torch.cat(got[0], dim=0).numpy()
            q.put(bool(np.array_equal(full, P.batched_matmul_scale(q_all, k_all, 0.125))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_two_rank_sharded_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(100)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_plan_device_follows_the_process_gpu():
    """One process per GPU: a plan bound by rank r must target cuda:r, not device 0
    (tm_exec_create switches to the plan's device before allocating scratch)."""
    from paper_2210_09603_b200.taskmap import _resolve_device

    class FakeCuda:
        is_cuda = True

        class device:  # noqa: N801
            index = 5

    assert _resolve_device(2) == 2
    assert _resolve_device(None, [object(), FakeCuda()]) == 5
    assert isinstance(_resolve_device(None), int)
