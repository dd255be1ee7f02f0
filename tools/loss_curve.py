"""Per-step loss of the ViT-B/16 bs-256 training step (eager, fixed synthetic
batch, bf16) — to compare numerics-affecting variants (env switches) step by step.

    python tools/loss_curve.py [steps]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200.trainer import ViTTrainer  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_B16  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
dev = torch.device("cuda", 0)
tr = ViTTrainer(VIT_B16, 256, half="bf16", device=dev, seed=0)
g = torch.Generator(device=dev).manual_seed(1000)
x = torch.randn(256, 224, 224, 3, generator=g, device=dev)
y = torch.randint(0, 1000, (256,), generator=g, device=dev).to(torch.int32)
out = []
for _ in range(steps):
    out.append(float(tr.step(x, y).item()))
print(" ".join(f"{v:.5f}" for v in out))
