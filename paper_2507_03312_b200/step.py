"""The fused mixed-precision step on flat HBM arenas — the hot path.

One step after backward is three stream-ordered launches and no host sync:

    K2  unscale+finite over the half-grad arena      reads 2 B/param
    [   all_reduce(flag, MIN) across DP ranks        4 bytes          ]
    K4  gated Adam(W): g/scale, m, v, p32, p_half     reads 14, writes 14 B/param
    K3  loss-scale state machine (fp64, 1 thread)

= 30 algorithmic bytes per parameter on a finite step, 2 on a skipped one.

Layout (SURVEY.md §8a ViT-B: 152 leaves, 86,567,656 params): every leaf is a
view into one arena per stream — p32 / m / v (f32), p_half and grads (f16 or
bf16) — each leaf starting on a 16-byte boundary, in the reference's
traversal order.  The arenas make the whole step a single-leaf
multi-tensor-apply (one table entry, ~42K full tiles, grid = resident blocks
x 148 SMs) and let the DP gradient exchange bucket contiguous memory.

The leaf-level drop-in API (cast_tree / LossScaling / optimizer_update)
calls exactly the same kernels with per-leaf tables.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native as N
from . import kernels as K
from .dtypes import F16, as_dtype
from .precision import DeviceBool, DynamicLossScaling
from .tree import float_leaves, tree_map


class FlatArena:
    """Views of one allocation laid out like a pytree's float leaves.

    Every leaf starts on an 8-element (16-byte) boundary; with `groups` (one
    key per leaf, consecutive equal keys form a group) each group also ends on a
    multiple of `group_align` elements, so a group splits into equal,
    aligned chunks (the ZeRO-1 shards of a gradient bucket)."""

    def __init__(self, leaves, dtype: torch.dtype, device, groups=None, group_align: int = 8):
        self.offsets = []
        total = 0
        for i, t in enumerate(leaves):
            self.offsets.append(total)
            total += -(-t.numel() // 8) * 8
            if groups is not None and (i + 1 == len(leaves) or groups[i + 1] != groups[i]):
                total = -(-total // group_align) * group_align
        self.numel = total
        self.buf = torch.empty(max(total, 8), dtype=dtype, device=device)
        self.views = [self.buf[o:o + t.numel()].view(t.shape) for o, t in zip(self.offsets, leaves)]

    def ptr(self) -> int:
        return self.buf.data_ptr()


class ShardArena:
    """ZeRO-1 master weights / moments: only this rank's chunk of every
    gradient bucket, concatenated in bucket order — 1/W of the f32 state per
    GPU.  `ranges` are (arena offset, length) pairs of the full layout."""

    def __init__(self, ranges, dtype: torch.dtype, device):
        self.ranges = list(ranges)
        self.starts, total = [], 0
        for _, n in self.ranges:
            self.starts.append(total)
            total += n
        self.numel = total
        self.buf = torch.empty(max(total, 8), dtype=dtype, device=device)

    def ptr(self) -> int:
        return self.buf.data_ptr()

    def chunks(self):
        """[(full-arena offset, chunk view)] in bucket order."""
        return [(o, self.buf[s:s + n]) for (o, n), s in zip(self.ranges, self.starts)]

    def fill_from(self, full: torch.Tensor):
        for (o, n), s in zip(self.ranges, self.starts):
            self.buf[s:s + n].copy_(full[o:o + n])


class FusedMPStep:
    """Master weights, Adam moments, half working copy and half grads of a
    parameter tree, resident in flat device arenas, stepped by K2/K4/K3.

    `params` is a tree whose float leaves are f32 CUDA tensors (copied in);
    `tree(kind)` rebuilds the tree over the arena views ('p32', 'half',
    'grad', 'm', 'v')."""

    def __init__(self, params, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0, half_dtype=F16, scaling: DynamicLossScaling | None = None,
                 process_group=None, zero: bool = False, zero_world: int | None = None,
                 zero_rank: int | None = None, comm=None):
        """`comm` (a dp.NativeComm): the exchange through the library's own
        NCCL entry points instead of torch.distributed — step() sums the half
        grad arena over the ranks (mpx_allreduce_grads) before K2 and ANDs the
        finite flag (mpx_allreduce_flag) after it."""
        if comm is not None and (process_group is not None or zero):
            raise ValueError("comm= is the torch-free replicated exchange: not with process_group / zero")
        self.comm = comm
        self.structure = params
        fl = float_leaves(params)
        if not fl:
            raise ValueError("params contain no float tensor leaves")
        self.paths = [p for p, _ in fl]
        leaves = [x for _, x in fl]
        K.require_cuda(leaves, "FusedMPStep")
        dev = leaves[0].device
        self.device = dev
        self.half = as_dtype(half_dtype)
        # ZeRO-1: rank r updates chunk r of every gradient
        # bucket (K2/K4 on 1/W of the bytes); the half grads arrive by
        # reduce-scatter and the half working copy leaves by all-gather
        self.zero = bool(zero)
        if self.zero:
            if process_group is not None:
                zero_world = torch.distributed.get_world_size(process_group)
                zero_rank = torch.distributed.get_rank(process_group)
            if zero_world is None or zero_rank is None:
                raise ValueError("zero=True needs a process group (or zero_world / zero_rank)")
            self.zero_world, self.zero_rank = int(zero_world), int(zero_rank)
        else:
            self.zero_world, self.zero_rank = 1, 0
        from .dp import bucket_key
        groups = [bucket_key(p) for p in self.paths] if self.zero else None
        align = 8 * self.zero_world
        p32 = FlatArena(leaves, torch.float32, dev, groups, align)
        self.p_half = FlatArena(leaves, self.half.torch, dev, groups, align)
        self.grad = FlatArena(leaves, self.half.torch, dev, groups, align)
        self.offsets = p32.offsets
        p32.buf.zero_()  # alignment pads stay 0 (finite) in every arena
        for dst, src in zip(p32.views, leaves):
            dst.copy_(src)
        self.grad.buf.zero_()
        self.n_params = sum(t.numel() for t in leaves)
        self.numel = p32.numel  # padded arena length (pads stay 0 / finite)
        K.cast_into([p32.buf], [self.p_half.buf])
        if self.zero:
            # ZeRO-1: p32 / m / v exist only for this rank's chunks (the optimizer
            # state is sharded, not just the update); the full layout's offsets
            # still address the gradient and half arenas
            from .dp import shard_ranges
            self.ranges = shard_ranges(self.paths, self.offsets, self.zero_world, self.zero_rank, self.numel)
            self.p32 = ShardArena(self.ranges, torch.float32, dev)
            self.p32.fill_from(p32.buf)
            del p32
            self.m = ShardArena(self.ranges, torch.float32, dev)
            self.v = ShardArena(self.ranges, torch.float32, dev)
        else:
            self.ranges = [(0, self.numel)]
            self.p32 = p32
            self.m = FlatArena(leaves, torch.float32, dev, groups, align)
            self.v = FlatArena(leaves, torch.float32, dev, groups, align)
        self.m.buf.zero_()
        self.v.buf.zero_()
        self.scaling = scaling if scaling is not None else DynamicLossScaling(2.0 ** 15, device=dev)
        self.flag = torch.ones((), dtype=torch.int32, device=dev)
        self.counter = torch.zeros(2, dtype=torch.int64, device=dev)
        self.used_scale = torch.zeros((), dtype=torch.float64, device=dev)
        self.hp = K.adam_hparams(lr, beta1, beta2, eps, weight_decay)
        self.bc = K.bias_correction_table(beta1, beta2, dev)
        self.group = process_group
        self._lib = N.load()
        self._build_tables()

    # ------------------------------------------------------------------
    def _build_tables(self):
        # (offset, length) element ranges this rank steps: the whole arena, or
        # under ZeRO-1 its chunk of every bucket (buckets in arena order)
        L = len(self.ranges)
        tab = lambda arena, es: (ctypes.c_void_p * L)(*[arena.ptr() + o * es for o, _ in self.ranges])  # noqa: E731
        if self.zero:  # the f32 state is compact: chunk r starts at its running offset
            ftab = lambda arena: (ctypes.c_void_p * L)(*[arena.ptr() + s * 4 for s in arena.starts])  # noqa: E731
        else:
            ftab = lambda arena: tab(arena, 4)  # noqa: E731
        hs = self.grad.buf.element_size()
        self._L = L
        self._n = (ctypes.c_int64 * L)(*[n for _, n in self.ranges])
        self._g_tab = tab(self.grad, hs)
        self._p_tab = ftab(self.p32)
        self._pd_tab = (ctypes.c_int32 * L)(*([N.MPX_F32] * L))
        self._m_tab = ftab(self.m)
        self._v_tab = ftab(self.v)
        self._h_tab = tab(self.p_half, hs)
        self._grad_src = self.grad.ptr()

    def tree(self, kind: str):
        if self.zero and kind in ("p32", "m", "v"):
            raise ValueError(f"tree({kind!r}): under ZeRO-1 this rank holds only its shard of the f32 state; "
                             "use gather(kind) (a collective) for the full tree, or shard_chunks(kind)")
        arena = {"p32": self.p32, "half": self.p_half, "grad": self.grad, "m": self.m, "v": self.v}[kind]
        return self._tree_of(arena.views)

    def _tree_of(self, views):
        it = iter(views)
        return tree_map(lambda x: next(it) if isinstance(x, torch.Tensor) and x.is_floating_point() else x,
                        self.structure)

    def shard_chunks(self, kind: str):
        """ZeRO-1: [(full-arena offset, chunk view)] of this rank's p32 / m / v."""
        if not self.zero:
            raise ValueError("shard_chunks: not a ZeRO-1 step")
        return {"p32": self.p32, "m": self.m, "v": self.v}[kind].chunks()

    def gather(self, kind: str):
        """The full p32 / m / v tree on every rank (ZeRO-1: all-gather of every
        bucket's chunks over the process group — call it on all ranks)."""
        if not self.zero or kind not in ("p32", "m", "v"):
            return self.tree(kind)
        if self.group is None:
            raise ValueError("gather: ZeRO-1 without a process group (hand-driven shards) cannot gather")
        from .dp import zero_bucket_views
        full = torch.zeros(self.numel, dtype=torch.float32, device=self.device)
        for (whole, mine), (_, chunk) in zip(zero_bucket_views(full, self.ranges, self.zero_world, self.zero_rank),
                                             self.shard_chunks(kind)):
            torch.distributed.all_gather_into_tensor(whole, chunk.contiguous(), group=self.group)
        return self._tree_of([full[o:o + v.numel()].view(v.shape) for o, v in zip(self.offsets, self.grad.views)])

    @property
    def step_count(self) -> int:
        return int(self.counter[0].item())

    @property
    def grads_finite(self) -> DeviceBool:
        return DeviceBool(self.flag)

    # ------------------------------------------------------------------
    def step(self, grad_ptr: int | None = None, stream: int | None = None):
        """K2 -> (flag all-reduce) -> K4 -> K3 on the arenas.  `grad_ptr`
        selects another half-grad arena of the same layout (e.g. a second
        buffer being filled by a copy engine)."""
        lib = self._lib
        st = stream if stream is not None else K.stream_handle(self.device)
        g = self._grad_table(grad_ptr)
        d_scale = self.scaling.state.data_ptr()
        code = self.half.code
        L = self._L
        if self.comm is not None:  # SUM of the scaled half grads over the ranks (1/W is in the loss cotangent)
            base = grad_ptr if grad_ptr is not None else self.grad.ptr()
            N.check(lib.mpx_allreduce_grads(self.comm.handle, base, self.grad.buf.numel(), code, st),
                    "mpx_allreduce_grads")
        N.check(lib.mpx_unscale_finite(N.as_pp(g), None, self._n, L, code, 1.0, d_scale, self.flag.data_ptr(), 1,
                                       st), "mpx_unscale_finite")
        if self.comm is not None:
            N.check(lib.mpx_allreduce_flag(self.comm.handle, self.flag.data_ptr(), st), "mpx_allreduce_flag")
        if self.group is not None:  # AND over ranks (mandatory under ZeRO-1: shards see different grads)
            torch.distributed.all_reduce(self.flag, op=torch.distributed.ReduceOp.MIN, group=self.group)
        N.check(lib.mpx_optimizer_step(N.as_pp(self._p_tab), self._pd_tab, N.as_pp(self._m_tab),
                                       N.as_pp(self._v_tab), N.as_pp(g), N.as_pp(self._h_tab), None, self._n, L,
                                       code, code, 0, self.hp, self.bc.data_ptr(), self.bc.numel() // 2,
                                       self.counter.data_ptr(), 1.0, d_scale, self.flag.data_ptr(), st),
                "mpx_optimizer_step")
        N.check(lib.mpx_scaling_adjust(self.scaling.state.data_ptr(), self.flag.data_ptr(), None,
                                       self.used_scale.data_ptr(), st), "mpx_scaling_adjust")
        if self.zero and self.group is not None:
            self.all_gather_half()

    def _grad_table(self, grad_ptr):
        if grad_ptr is None:
            return self._g_tab
        hs = self.grad.buf.element_size()
        return (ctypes.c_void_p * self._L)(*[grad_ptr + o * hs for o, _ in self.ranges])

    # ZeRO-1 exchange over the bucket layout (also done per bucket by trainer.GradExchange)
    def reduce_scatter_grads(self):
        """Sum the half grads over the group into this rank's chunk of every bucket."""
        from .dp import zero_bucket_views
        for full, mine in zero_bucket_views(self.grad.buf, self.ranges, self.zero_world, self.zero_rank):
            torch.distributed.reduce_scatter_tensor(mine, full, group=self.group)

    def all_gather_half(self):
        """Every rank's updated chunk of the half working copy to every rank."""
        from .dp import zero_bucket_views
        for full, mine in zero_bucket_views(self.p_half.buf, self.ranges, self.zero_world, self.zero_rank):
            torch.distributed.all_gather_into_tensor(full, mine, group=self.group)

    # per-kernel entry points (timing / profiling)
    def k2(self, grad_ptr=None, stream=None):
        st = stream if stream is not None else K.stream_handle(self.device)
        g = self._grad_table(grad_ptr)
        N.check(self._lib.mpx_unscale_finite(N.as_pp(g), None, self._n, self._L, self.half.code, 1.0,
                                             self.scaling.state.data_ptr(), self.flag.data_ptr(), 1, st), "k2")

    def k4(self, grad_ptr=None, stream=None):
        st = stream if stream is not None else K.stream_handle(self.device)
        g = self._grad_table(grad_ptr)
        code = self.half.code
        N.check(self._lib.mpx_optimizer_step(N.as_pp(self._p_tab), self._pd_tab, N.as_pp(self._m_tab),
                                             N.as_pp(self._v_tab), N.as_pp(g), N.as_pp(self._h_tab), None, self._n,
                                             self._L, code, code, 0, self.hp, self.bc.data_ptr(), self.bc.numel() // 2,
                                             self.counter.data_ptr(), 1.0, self.scaling.state.data_ptr(),
                                             self.flag.data_ptr(), st), "k4")

    def k3(self, stream=None):
        st = stream if stream is not None else K.stream_handle(self.device)
        N.check(self._lib.mpx_scaling_adjust(self.scaling.state.data_ptr(), self.flag.data_ptr(), None,
                                             self.used_scale.data_ptr(), st), "k3")

    ALGO_BYTES_FINITE = 30  # per parameter: K2 2 + K4 (2+4+4+4 read, 4+4+4+2 write)
    ALGO_BYTES_SKIPPED = 2  # K2 only; K4 exits on the flag
    K4_BYTES = 28
