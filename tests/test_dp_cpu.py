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
