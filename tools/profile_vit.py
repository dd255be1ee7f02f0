"""One ViT-B/16 (or ViT-L/16: argv[3] = L) training step between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (warm-up steps run first)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import as_dtype  # noqa: E402
from paper_2507_03312_b200.trainer import ViTTrainer  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_B16, VIT_L16  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    half = as_dtype(sys.argv[2] if len(sys.argv) > 2 else "bf16")
    dev = torch.device("cuda", 0)
    cfg = VIT_L16 if len(sys.argv) > 3 and sys.argv[3] == "L" else VIT_B16  # argv[3] = L: ViT-L/16
    tr = ViTTrainer(cfg, B, half=half, device=dev)
    x = torch.randn(B, 224, 224, 3, device=dev)
    y = torch.randint(0, 1000, (B,), device=dev).to(torch.int32)
    for _ in range(2):
        tr.step(x, y)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    tr.step(x, y)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("loss", tr.engine.loss.item(), "finite", bool(tr.grads_finite))


if __name__ == "__main__":
    main()
