"""ViT-B/16 trainer: per-step loss, finite flag and scale (diagnostics)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import as_dtype  # noqa: E402
from paper_2507_03312_b200.trainer import ViTTrainer  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_B16  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tr = ViTTrainer(VIT_B16, B, half=as_dtype("bf16"), device="cuda")
g = torch.Generator(device="cuda").manual_seed(1000)
x = torch.randn(B, 224, 224, 3, generator=g, device="cuda")
y = torch.randint(0, 1000, (B,), generator=g, device="cuda").to(torch.int32)
out = []
for i in range(8):
    l = tr.step(x, y)
    out.append((round(l.item(), 4), int(bool(tr.grads_finite)), tr.mp.used_scale.item()))
print(out)
