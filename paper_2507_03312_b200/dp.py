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
    """All-reduce each bucket as the backward completes it — or, under ZeRO-1
    (`zero_views`: key -> (whole padded bucket, this rank's chunk)),
    reduce-scatter it so each rank receives the sum of its chunk only."""

    def __init__(self, buckets: GradBuckets, group=None, zero_views: dict | None = None):
        self.buckets = buckets
        self.group = group
        self.zero_views = zero_views
        self.pending = []

    def ready(self, key: str):
        if self.group is None:
            return
        if self.zero_views is not None:
            full, mine = self.zero_views[key]
            self.pending.append(dist.reduce_scatter_tensor(mine, full, group=self.group, async_op=True))
        else:
            self.pending.append(dist.all_reduce(self.buckets.views[key], group=self.group, async_op=True))

    def wait(self):
        for w in self.pending:
            w.wait()
        self.pending.clear()


def _bucket_spans(paths: list[str], offsets: list[int], arena_numel: int) -> list[tuple[str, int, int]]:
    """(key, lo, hi) per bucket in arena order; hi = the next bucket's start
    (or the arena end), i.e. including the bucket's alignment padding."""
    first: dict[str, int] = {}
    for p, o in zip(paths, offsets):
        k = bucket_key(p)
        first[k] = min(first.get(k, o), o)
    starts = sorted((o, k) for k, o in first.items())
    return [(k, o, starts[i + 1][0] if i + 1 < len(starts) else arena_numel) for i, (o, k) in enumerate(starts)]


def shard_ranges(paths: list[str], offsets: list[int], world: int, rank: int,
                 arena_numel: int) -> list[tuple[int, int]]:
    """ZeRO-1: rank `rank`'s (offset, length) chunk of
    every bucket — each bucket span (padded to a multiple of 8*world by the
    arena layout) split into `world` equal, 16-byte-aligned chunks."""
    out = []
    for _, lo, hi in _bucket_spans(paths, offsets, arena_numel):
        n = hi - lo
        if n % (8 * world):
            raise ValueError(f"bucket at {lo} spans {n} elements, not a multiple of 8*world={8 * world}")
        c = n // world
        out.append((lo + rank * c, c))
    return out


def zero_bucket_views(arena: torch.Tensor, ranges: list[tuple[int, int]], world: int, rank: int):
    """(whole bucket, this rank's chunk) views of `arena` for each bucket: the
    in-place layouts of reduce_scatter (chunk = sum) and all_gather."""
    out = []
    for off, c in ranges:
        lo = off - rank * c
        out.append((arena[lo:lo + world * c], arena[off:off + c]))
    return out


def zero_views_by_key(arena: torch.Tensor, paths: list[str], offsets: list[int], world: int, rank: int) -> dict:
    """bucket key -> (whole padded bucket, this rank's chunk) of `arena`."""
    spans = _bucket_spans(paths, offsets, arena.numel())
    ranges = shard_ranges(paths, offsets, world, rank, arena.numel())
    views = zero_bucket_views(arena, ranges, world, rank)
    return {k: v for (k, _, _), v in zip(spans, views)}


def allreduce_flag_min(flag: torch.Tensor, group=None):
    if group is not None or (dist.is_available() and dist.is_initialized()):
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return flag


def env_world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(
        os.environ.get("LOCAL_RANK", "0"))


class NativeComm:
    """An NCCL communicator owned by libmpx_b200.so (mpx_comm_* in
    include/mpx_b200.h) — the exchange a host without torch.distributed
    drives: `allreduce_flag` (MIN = AND of the finite flags) and
    `allreduce_grads` (SUM of the scaled half gradients).  Rank 0 makes the
    id with `unique_id()` and ships the 128 bytes to every rank out of band."""

    def __init__(self, nranks: int, uid: bytes, rank: int, device: int):
        import ctypes

        from . import _native as N

        if len(uid) != N.MPX_COMM_ID_BYTES:
            raise ValueError(f"NCCL unique id must be {N.MPX_COMM_ID_BYTES} bytes")
        self._lib = N.load()
        buf = ctypes.create_string_buffer(bytes(uid), N.MPX_COMM_ID_BYTES)
        h = ctypes.c_void_p()
        N.check(self._lib.mpx_comm_init(ctypes.byref(h), nranks, buf, rank, device), "mpx_comm_init")
        self.handle, self.rank, self.device = h.value, rank, device

    @staticmethod
    def unique_id() -> bytes:
        import ctypes

        from . import _native as N

        buf = ctypes.create_string_buffer(N.MPX_COMM_ID_BYTES)
        N.check(N.load().mpx_comm_unique_id(buf), "mpx_comm_unique_id")
        return buf.raw

    @property
    def size(self) -> int:
        import ctypes

        from . import _native as N

        n = ctypes.c_int()
        N.check(self._lib.mpx_comm_size(self.handle, ctypes.byref(n)), "mpx_comm_size")
        return n.value

    def allreduce_flag(self, flag: torch.Tensor, stream=None):
        from . import _native as N
        from .kernels import stream_handle

        if flag.dtype not in (torch.int32, torch.uint32) or flag.numel() != 1 or not flag.is_cuda:
            raise TypeError("allreduce_flag: a 1-element 32-bit CUDA flag")
        st = stream if stream is not None else stream_handle(flag.device)
        N.check(self._lib.mpx_allreduce_flag(self.handle, flag.data_ptr(), st), "mpx_allreduce_flag")

    def allreduce_grads(self, grads: torch.Tensor, stream=None):
        from . import _native as N
        from .kernels import stream_handle

        code = {torch.float32: N.MPX_F32, torch.float16: N.MPX_F16, torch.bfloat16: N.MPX_BF16}.get(grads.dtype)
        if code is None or not grads.is_cuda or not grads.is_contiguous():
            raise TypeError("allreduce_grads: a contiguous f32/f16/bf16 CUDA arena")
        st = stream if stream is not None else stream_handle(grads.device)
        N.check(self._lib.mpx_allreduce_grads(self.handle, grads.data_ptr(), grads.numel(), code, st),
                "mpx_allreduce_grads")

    def close(self):
        if self.handle:
            from . import _native as N

            N.check(self._lib.mpx_comm_destroy(self.handle), "mpx_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass
