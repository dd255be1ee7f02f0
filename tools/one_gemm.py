"""One ViT-B fc1-forward-shaped GEMM (M=50432, K=768, N=3072, bf16) for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

M, K, N = 256 * 197, 768, 3072
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(K, N, device="cuda") * 0.03).to(torch.bfloat16)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    VK.linear_fwd(x, w, out=y)
torch.cuda.synchronize()
print("ok", float(y.float().abs().mean()))
