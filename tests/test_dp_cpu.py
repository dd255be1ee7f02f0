"""Data-parallel host logic on CPU with gloo, world size 2: bucketed gradient
all-reduce in backward order, the finite-flag MIN (logical AND) reduction,
and bucket partitioning of the ViT-B gradient arena."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_03312_b200.dp import GradBuckets, GradExchange, allreduce_flag_min, bucket_key
from paper_2507_03312_b200.vit_config import VIT_B16, VIT_TINY


def _layout(cfg):
    paths, offs, nums, tot = [], [], [], 0
    for name, shape in cfg.param_shapes():
        n = 1
        for d in shape:
            n *= d
        paths.append(name)
        offs.append(tot)
        nums.append(n)
        tot += -(-n // 8) * 8
    return paths, offs, nums, tot


def test_buckets_cover_arena_in_backward_order():
    paths, offs, nums, tot = _layout(VIT_B16)
    arena = torch.zeros(tot)
    b = GradBuckets(paths, offs, nums, arena)
    order = b.order(VIT_B16.depth)
    assert order[0] == "head" and order[-1] == "embed" and order[1] == "blocks.11" and len(order) == 14
    covered = sum(v.numel() for v in b.views.values())
    assert covered >= sum(nums) and covered <= tot
    for p, o, n in zip(paths, offs, nums):  # every leaf lies inside its bucket
        v = b.views[bucket_key(p)]
        start = (v.data_ptr() - arena.data_ptr()) // arena.element_size()
        assert start <= o and o + n <= start + v.numel()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        paths, offs, nums, tot = _layout(VIT_TINY)
        arena = torch.full((tot,), float(rank + 1))
        b = GradBuckets(paths, offs, nums, arena)
        ex = GradExchange(b, dist.group.WORLD)
        for key in b.order(VIT_TINY.depth):
            ex.ready(key)
        ex.wait()
        total = sum(range(1, world + 1))
        ok_sum = all(bool((v == total).all()) for v in b.views.values())
        flag = torch.tensor(0 if rank == 1 else 1, dtype=torch.int32)
        allreduce_flag_min(flag, dist.group.WORLD)
        flag2 = torch.tensor(1, dtype=torch.int32)
        allreduce_flag_min(flag2, dist.group.WORLD)
        q.put((rank, ok_sum, int(flag.item()), int(flag2.item())))
    finally:
        dist.destroy_process_group()


def test_gloo_bucket_allreduce_and_flag_and():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_sum, f_and, f_all in res:
        assert ok_sum, f"rank {rank}: bucket sums wrong"
        assert f_and == 0, "one non-finite rank must skip the step everywhere"
        assert f_all == 1


def _zero_layout(cfg, world):
    """The arena layout FusedMPStep builds under ZeRO-1: leaves 8-aligned, each
    bucket padded to a multiple of 8*world."""
    paths, offs, nums, tot = [], [], [], 0
    names = [n for n, _ in cfg.param_shapes()]
    for i, (name, shape) in enumerate(cfg.param_shapes()):
        n = 1
        for d in shape:
            n *= d
        paths.append(name)
        offs.append(tot)
        nums.append(n)
        tot += -(-n // 8) * 8
        if i + 1 == len(names) or bucket_key(names[i + 1]) != bucket_key(name):
            tot = -(-tot // (8 * world)) * (8 * world)
    return paths, offs, nums, tot


def test_zero_shards_partition_every_bucket():
    from paper_2507_03312_b200.dp import shard_ranges
    for cfg in (VIT_B16, VIT_TINY):
        for world in (2, 4, 8):
            paths, offs, nums, tot = _zero_layout(cfg, world)
            cover = torch.zeros(tot, dtype=torch.int32)
            for r in range(world):
                for o, n in shard_ranges(paths, offs, world, r, tot):
                    assert o % 8 == 0 and n % 8 == 0
                    cover[o:o + n] += 1
            assert bool((cover == 1).all()), (cfg, world)  # every element owned by exactly one rank


def _zero_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_03312_b200.dp import zero_views_by_key
        paths, offs, nums, tot = _zero_layout(VIT_TINY, world)
        g = torch.Generator().manual_seed(rank)
        grads = torch.randn(tot, generator=g)
        arena = grads.clone()
        b = GradBuckets(paths, offs, nums, arena)
        views = zero_views_by_key(arena, paths, offs, world, rank)
        ex = GradExchange(b, dist.group.WORLD, zero_views=views)
        for key in b.order(VIT_TINY.depth):  # reduce-scatter each bucket as the backward finishes it
            ex.ready(key)
        ex.wait()
        full = grads.clone()
        dist.all_reduce(full)
        ok_rs = all(torch.equal(mine, full[(mine.data_ptr() - arena.data_ptr()) // 4:][:mine.numel()])
                    for _, mine in views.values())
        # "update" my chunks (x -> 2x + rank-independent) then all-gather the working copy
        work = torch.zeros(tot)
        wviews = zero_views_by_key(work, paths, offs, world, rank)
        for key, (_, mine) in wviews.items():
            o = (mine.data_ptr() - work.data_ptr()) // 4
            mine.copy_(full[o:o + mine.numel()] * 2)
        for whole, mine in wviews.values():
            dist.all_gather_into_tensor(whole, mine.clone())
        q.put((rank, ok_rs, torch.equal(work, full * 2)))
    finally:
        dist.destroy_process_group()


def test_gloo_zero_reduce_scatter_all_gather():
    """ZeRO-1 exchange: per-bucket reduce-scatter gives
    each rank the all-reduced values of its chunks; the all-gather of the
    updated chunks rebuilds the whole working copy on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zero_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_rs, ok_ag in res:
        assert ok_rs, f"rank {rank}: reduce-scattered chunks wrong"
        assert ok_ag, f"rank {rank}: all-gathered working copy wrong"
