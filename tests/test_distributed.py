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

from paper_2210_09603_b200.sharding import shard_range


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


def _worker(rank, world, port, q, scaling):
    """One rank of bench.py's shard -> compute -> gather path (sharding.py), on CPU.
    The per-rank compute stands in for the fused kernels (GPU-only): a conv whose
    output is channels-last (the bench's layout) and a token-wise FFN-like map."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_09603_b200.sharding import assemble, gather_buffers, gather_to_root, sweep_shard
        totals = {"images": 5, "tokens": 37, "heads": 6}
        shard = sweep_shard(rank, world, scaling, totals)
        g = torch.Generator().manual_seed(7)  # weights: one seed, identical on every rank
        w_conv, w_tok = torch.randn(4, 3, 3, 3, generator=g), torch.randn(8, 8, generator=g)
        glob = {u: shard.global_count(u) for u in totals}
        gx = torch.Generator().manual_seed(11)  # the global batch, sliced per rank
        x_all, t_all = torch.randn(glob["images"], 3, 9, 9, generator=gx), torch.randn(glob["tokens"], 8, generator=gx)
        if scaling == "weak":
            assert shard.count("images") == totals["images"] and glob["images"] == totals["images"] * world
        (i0, i1), (t0, t1) = shard.range("images"), shard.range("tokens")
        y = torch.nn.functional.conv2d(x_all[i0:i1], w_conv, padding=1).contiguous(memory_format=torch.channels_last)
        z = torch.relu(t_all[t0:t1] @ w_tok)
        rows = [shard.sizes("images"), shard.sizes("tokens")]
        bufs = gather_buffers([y, z], 0, [max(r) for r in rows])
        got = gather_to_root([y, z], 0, bufs, rows)
        if rank == 0:
            want_y = torch.nn.functional.conv2d(x_all, w_conv, padding=1)
            want_z = torch.relu(t_all @ w_tok)
            # (CPU conv / matmul kernels may block differently per slice size: allclose, not bitwise)
            q.put(bool(torch.allclose(assemble(got[0]), want_y, rtol=1e-5, atol=1e-5) and
                       torch.allclose(assemble(got[1]), want_z, rtol=1e-5, atol=1e-5)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world,scaling", [(2, "strong"), (3, "strong"), (2, "weak")])
def test_gloo_sharded_sweep_gather(world, scaling):
    """world 2 and 3 (uneven shards: 5 images, 37 tokens), strong and weak scaling: the
    gathered, reassembled result equals the unsharded computation."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, scaling)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(150)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_sweep_shard_strong_and_weak():
    from paper_2210_09603_b200.sharding import sweep_shard
    for world in (1, 2, 4, 8):
        shards = [sweep_shard(r, world) for r in range(world)]
        assert sum(s.count("images") for s in shards) == 32
        assert sum(s.count("tokens") for s in shards) == 8192
        assert sum(s.count("heads") for s in shards) == 192
        assert [s.range("images")[0] for s in shards] == [32 // world * r for r in range(world)]
        weak = sweep_shard(world - 1, world, "weak")
        assert weak.count("images") == 32 and weak.global_count("tokens") == 8192 * world


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


class _FakeChain:
    """Stands in for chain.ResNet50Chain (GPU-only) on CPU: per-image logits from
    the rank's slice of the images, so the sharded result is checkable."""

    def __init__(self, batch, image, configs=None, seed=0):
        g = torch.Generator().manual_seed(seed)
        self.w = torch.randn(3, 10, generator=g)  # weights identical on every rank
        self.x = torch.zeros(batch, 3, image, image)
        self.logits = torch.zeros(batch, 10)

    def set_input(self, images):
        self.x.copy_(images)

    def replay(self):
        self.logits.copy_(self.x.mean(dim=(2, 3)) @ self.w)
        return self.logits


def _chain_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_09603_b200 import chain as C
        C.ResNet50Chain = _FakeChain
        imgs = torch.randn(7, 3, 5, 5, generator=torch.Generator().manual_seed(3))
        ch, logits = C.run_sharded(7, rank, world, image=5, images=imgs, seed=1)
        a, b = shard_range(7, rank, world)
        assert ch.logits.shape[0] == b - a
        if rank == 0:
            want = _FakeChain(7, 5, seed=1)
            want.set_input(imgs)
            q.put(bool(torch.allclose(logits, want.replay(), rtol=1e-6, atol=1e-6)))
        else:
            assert logits is None
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_chain_level_sharding(world):
    """Row f2: each rank runs the whole chain on its slice of the batch (7 images,
    uneven shards) and the logits are gathered once; the result equals the
    unsharded chain."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(150)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
