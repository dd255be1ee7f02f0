"""Time the batched 16-bit transpose on the ViT-B forward weight copies (48 matrices)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

shapes = [(768, 2304), (768, 768), (768, 3072), (3072, 768)] * 12
srcs = [torch.randn(r, c, device="cuda").bfloat16() for r, c in shapes]
outs = [torch.empty(c, r, device="cuda", dtype=torch.bfloat16) for r, c in shapes]
for _ in range(3):
    VK.transpose_batch(srcs, outs)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    VK.transpose_batch(srcs, outs)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
byt = 2 * sum(2 * r * c for r, c in shapes)
print(f"transpose_batch {ms * 1000:.1f} us, {byt / ms / 1e6:.0f} GB/s")
