"""Data-parallel mixed-precision ViT training step (configs 3-5).

One step, all stream-ordered, no host sync:

    K1 cast images f32 -> half                       (cast_tree(args, half), precision.py:210)
    forward / backward (vit.ViTEngine)               loss cotangent = f32(scale) / W read on the
                                                     device, so the backward emits scaled half grads
                                                     already divided by the DP world size
    per-block NCCL all-reduce(sum) of the half grads, launched as soon as each
    block's gradients exist, overlapping the rest of the backward
    K2 -> all_reduce(flag, MIN) -> K4 (Adam, writes the next step's half
    weights) -> K3                                   (step.FusedMPStep)

Every rank holds the full f32 master weights / moments / scaling state
(replicated) and takes the same skip/scale decision.
"""
from __future__ import annotations

import torch

from . import kernels as K
from .dp import GradBuckets, GradExchange
from .dtypes import F16, as_dtype
from .precision import DynamicLossScaling
from .step import FusedMPStep
from .vit import ViTEngine, init_params
from .vit_config import ViTConfig


class ViTTrainer:
    def __init__(self, cfg: ViTConfig, batch_per_gpu: int, half=F16, lr: float = 1e-3, device=None,
                 group=None, world_size: int = 1, seed: int = 0, loss_scale: float = 2.0 ** 15,
                 weight_decay: float = 0.0, zero: bool = False):
        self.cfg = cfg
        self.B = batch_per_gpu
        self.half = as_dtype(half)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.W = world_size
        params = init_params(cfg, self.dev, seed=seed)  # same seed on every rank: replicas start equal
        # zero=True (ZeRO-1): buckets reduce-scattered during the
        # backward, K2/K4 on this rank's 1/W chunk, half working copy all-gathered
        self.zero = bool(zero) and group is not None
        self.mp = FusedMPStep(params, lr, weight_decay=weight_decay, half_dtype=self.half,
                              scaling=DynamicLossScaling(loss_scale, device=self.dev), process_group=group,
                              zero=self.zero)
        del params
        self.engine = ViTEngine(cfg, batch_per_gpu, self.half, self.dev)
        self.paths = self.mp.paths
        self.P = dict(zip(self.paths, self.mp.p_half.views))
        self.G = dict(zip(self.paths, self.mp.grad.views))
        self.images_h = torch.empty(batch_per_gpu, cfg.img, cfg.img, cfg.chans, dtype=self.half.torch,
                                    device=self.dev)
        self.dloss = torch.zeros((), dtype=torch.float32, device=self.dev)
        self.inv_w = torch.full((), 1.0 / world_size, dtype=torch.float32, device=self.dev)
        numels = [v.numel() for v in self.mp.grad.views]
        self.buckets = GradBuckets(self.paths, self.mp.grad.offsets, numels, self.mp.grad.buf)
        zviews = None
        if self.zero:
            from .dp import zero_views_by_key
            zviews = zero_views_by_key(self.mp.grad.buf, self.paths, self.mp.grad.offsets, self.mp.zero_world,
                                       self.mp.zero_rank)
        self.exchange = GradExchange(self.buckets, group, zero_views=zviews)

    # ------------------------------------------------------------------
    def forward_backward(self, images: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        """images: [B, H, W, C] f32 (or already half) on the device."""
        if images.dtype != self.half.torch:
            K.cast_into([images], [self.images_h])
            img = self.images_h
        else:
            img = images
        loss = self.engine.forward(self.P, img, labels)
        # loss cotangent f32(scale) * (1/W): the scaled, DP-averaged seed
        K.cast_into([self.inv_w], [self.dloss], d_scale=self.mp.scaling.d_scale)
        self.engine.backward(self.P, self.G, dloss_f32=self.dloss,
                             on_grads_ready=self.exchange.ready if self.group is not None else None)
        return loss

    def step(self, images: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        loss = self.forward_backward(images, labels)
        self.exchange.wait()
        self.mp.step()
        return loss

    # ------------------------------------------------------------------
    # CUDA graph: the step has no host sync and every scalar it branches on
    # (finite flag, loss scale, step counter) lives on the device, so it is
    # captured once and replayed — one launch per step instead of ~470
    # Python/ctypes launches (and their host-side tensor-map encodes).
    def capture(self, images: torch.Tensor, labels: torch.Tensor, warmup: int = 2):
        """Capture step() reading from the given (static) device buffers."""
        # with a process group the NCCL collectives (bucket all-reduce / reduce-scatter,
        # flag MIN, ZeRO all-gather) are captured into the graph too; every rank
        # captures the same sequence, so replays stay matched across ranks
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            for _ in range(warmup):  # allocations (split-K workspaces) happen outside the capture
                self.step(images, labels)
        torch.cuda.current_stream(self.dev).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(images, labels)
        # several captures (one per input buffer) may coexist: they share every
        # state buffer, so replaying them in any order is stepping the trainer —
        # double-buffered inputs let the next batch's H2D copy overlap a step
        self._graphs = getattr(self, "_graphs", []) + [(g, images, labels)]
        return len(self._graphs) - 1

    def replay(self, which: int = 0) -> torch.Tensor:
        """Replay the step captured for input buffer `which` (capture order)."""
        self._graphs[which][0].replay()
        return self.engine.loss

    @property
    def grads_finite(self):
        return self.mp.grads_finite

    @property
    def scaling(self) -> DynamicLossScaling:
        return self.mp.scaling
