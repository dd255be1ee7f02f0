"""Data-parallel exchange for the mixed-precision step (one process per GPU).

* GradBuckets — contiguous slices of the flat half-gradient arena, one per
  transformer block (+ head, + embedding), in the order the backward
  finishes them.
* GradExchange — starts an async NCCL all-reduce(sum) of each bucket the
  moment the backward has launched its gradients, so the exchange overlaps
  the rest of the backward; wait() joins them before the optimizer.  The
  1/W of the data-parallel mean is folded into the loss cotangent (exact for
  power-of-two W), so the buckets are plain sums.
* allreduce_flag_min — the finite flag, MIN over ranks (logical AND), so
  every rank takes the same skip / scale decision.

Everything here is backend-agnostic torch.distributed: NCCL on the GPUs,
gloo in the CPU tests (tests/test_dp_cpu.py).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def bucket_key(path: str) -> str:
    if path.startswith("blocks."):
        return ".".join(path.split(".")[:2])
    if path in ("ln_f.g", "ln_f.b", "head.w", "head.b"):
        return "head"
    return "embed"


class GradBuckets:
    def __init__(self, paths: list[str], offsets: list[int], numels: list[int], arena: torch.Tensor):
        groups: dict[str, list[int]] = {}
        for i, p in enumerate(paths):
            groups.setdefault(bucket_key(p), []).append(i)
        self.views: dict[str, torch.Tensor] = {}
        spans = []
        for key, idx in groups.items():
            lo = min(offsets[i] for i in idx)
            hi = max(offsets[i] + numels[i] for i in idx)
            hi = min(-(-hi // 8) * 8, arena.numel())
            self.views[key] = arena[lo:hi]
            spans.append((lo, hi, key))
        spans.sort()
        for (a0, a1, ka), (b0, b1, kb) in zip(spans, spans[1:]):
            if a1 > b0:
                raise ValueError(f"gradient buckets {ka} and {kb} overlap: leaves of a bucket must be contiguous")

    def order(self, depth: int) -> list[str]:
        keys = ["head"] + [f"blocks.{i}" for i in reversed(range(depth))] + ["embed"]
        return [k for k in keys if k in self.views]


class GradExchange:
    def __init__(self, buckets: GradBuckets, group=None):
        self.buckets = buckets
        self.group = group
        self.pending = []

    def ready(self, key: str):
        if self.group is None:
            return
        self.pending.append(dist.all_reduce(self.buckets.views[key], group=self.group, async_op=True))

    def wait(self):
        for w in self.pending:
            w.wait()
        self.pending.clear()


def allreduce_flag_min(flag: torch.Tensor, group=None):
    if group is not None or (dist.is_available() and dist.is_initialized()):
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return flag


def env_world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(
        os.environ.get("LOCAL_RANK", "0"))
