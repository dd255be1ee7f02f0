"""Weight-gradient GEMM (K = 50432 tokens) time vs split-K factor and CTA grouping."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1000


M = 256 * 197
for name, K, N in [("qkv", 768, 2304), ("proj", 768, 768), ("fc1", 768, 3072), ("fc2", 3072, 768)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    dy = torch.randn(M, N, device="cuda").bfloat16()
    dw = torch.empty(K, N, device="cuda", dtype=torch.bfloat16)
    row = {"gemm": name, "auto": round(t(lambda: VK.linear_wgrad(x, dy, out=dw)), 1)}
    for s in (1, 2, 3, 4, 6, 8):
        row[f"s{s}"] = round(t(lambda: VK.linear_wgrad(x, dy, out=dw, split_k=s)), 1)
    row["cublas"] = round(t(lambda: torch.matmul(x.t(), dy, out=dw)), 1)
    print(row, flush=True)
