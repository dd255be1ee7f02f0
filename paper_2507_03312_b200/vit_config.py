"""ViT configurations of BASELINE.json (configs 1, 3-5) and their parameter
trees.  Weights are stored [fan_in, fan_out] and used as x @ W, the layout
of the reference's linear layers (bench.py:129-131, 183)."""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class ViTConfig:
    img: int = 224
    patch: int = 16
    chans: int = 3
    dim: int = 768
    depth: int = 12
    heads: int = 12
    mlp: int = 3072
    classes: int = 1000
    pool: str = "cls"  # "cls" (ViT-B/L) or "mean" (tiny ViT)

    @property
    def n_patches(self) -> int:
        return (self.img // self.patch) ** 2

    @property
    def seq(self) -> int:
        return self.n_patches + (1 if self.pool == "cls" else 0)

    def param_shapes(self) -> list[tuple[str, tuple[int, ...]]]:
        d, p = self.dim, self.patch
        shapes = [("patch.w", (p * p * self.chans, d)), ("patch.b", (d,))]
        if self.pool == "cls":
            shapes.append(("cls", (1, d)))
        shapes.append(("pos", (self.seq, d)))
        for i in range(self.depth):
            b = f"blocks.{i}."
            shapes += [(b + "ln1.g", (d,)), (b + "ln1.b", (d,)), (b + "qkv.w", (d, 3 * d)), (b + "qkv.b", (3 * d,)),
                       (b + "proj.w", (d, d)), (b + "proj.b", (d,)), (b + "ln2.g", (d,)), (b + "ln2.b", (d,)),
                       (b + "fc1.w", (d, self.mlp)), (b + "fc1.b", (self.mlp,)), (b + "fc2.w", (self.mlp, d)),
                       (b + "fc2.b", (d,))]
        shapes += [("ln_f.g", (d,)), ("ln_f.b", (d,)), ("head.w", (d, self.classes)), ("head.b", (self.classes,))]
        return shapes

    def n_params(self) -> int:
        return sum(math.prod(s) for _, s in self.param_shapes())

    def flops_per_image(self) -> float:
        """Training FLOPs per image = 3 x forward GEMM/attention FLOPs."""
        n, d, m = self.seq, self.dim, self.mlp
        per_block = 2 * n * d * 3 * d + 2 * n * d * d + 2 * 2 * n * d * m + 2 * 2 * n * n * d
        fwd = self.depth * per_block + 2 * self.n_patches * (self.patch ** 2 * self.chans) * d + 2 * d * self.classes
        return 3.0 * fwd


VIT_B16 = ViTConfig()
VIT_L16 = ViTConfig(dim=1024, depth=24, heads=16, mlp=4096)
VIT_TINY = ViTConfig(img=32, patch=4, dim=64, depth=2, heads=4, mlp=256, classes=10, pool="mean")
