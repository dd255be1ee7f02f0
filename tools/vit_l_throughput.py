"""ViT-L/16 (BASELINE configs[4] model) training throughput on one B200: f16,
dynamic loss scaling with the configs[4] initial scale 2^32 (overflow stress:
the first steps back off), one CUDA graph per step.  Prints img/s, the loss
scale trajectory and the skipped steps."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200.trainer import ViTTrainer  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_L16  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    dev = torch.device("cuda", 0)
    tr = ViTTrainer(VIT_L16, B, half="f16", device=dev, loss_scale=2.0 ** 32)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(B, 224, 224, 3, device=dev, generator=g)
    y = torch.randint(0, 1000, (B,), device=dev, generator=g).to(torch.int32)
    scales, finite = [], []
    tr.capture(x, y, warmup=2)
    for _ in range(20):  # the 2^32 start backs off on overflowing steps
        tr.replay()
        scales.append(tr.scaling.to_host().loss_scale)
        finite.append(bool(tr.grads_finite))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 10
    a.record()
    for _ in range(K):
        tr.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print(json.dumps({"model": "ViT-L/16", "batch": B, "half": "f16", "ms_per_step": round(ms, 3),
                      "img_per_s": round(B / (ms * 1e-3), 1), "tflops": round(VIT_L16.flops_per_image() * B / (ms * 1e-3) / 1e12, 1),
                      "loss_scale_first_20": scales, "finite_first_20": finite,
                      "mem_gb": round(torch.cuda.max_memory_allocated() / 2 ** 30, 1)}))


if __name__ == "__main__":
    main()
