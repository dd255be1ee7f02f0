"""ViT-B weight-gradient GEMMs (K = 50432 tokens): the wide 256 x 384 tile vs
the 256 x 256 tile vs cuBLAS (torch.matmul), CUDA events, bf16."""
import json
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
tot = {"auto": 0.0, "narrow": 0.0, "cublas": 0.0}
for name, K, N in [("qkv", 768, 2304), ("proj", 768, 768), ("fc1", 768, 3072), ("fc2", 3072, 768)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    dy = torch.randn(M, N, device="cuda").bfloat16()
    dw = torch.empty(K, N, device="cuda", dtype=torch.bfloat16)
    row = {"gemm": name + ".wgrad", "wide384_us": round(t(lambda: VK.linear_wgrad(x, dy, out=dw, wide=384)), 1), "wide512_us": round(t(lambda: VK.linear_wgrad(x, dy, out=dw, wide=512)), 1) if N % 512 == 0 else None, "auto_us": round(t(lambda: VK.linear_wgrad(x, dy, out=dw)), 1),
           "narrow_us": round(t(lambda: VK.linear_wgrad(x, dy, out=dw, wide=False)), 1),
           "cublas_us": round(t(lambda: torch.matmul(x.t(), dy, out=dw)), 1)}
    for k in tot:
        tot[k] += row[k + "_us"]
    print(json.dumps(row), flush=True)
print(json.dumps({"per_layer_wgrad_us": {k: round(v, 1) for k, v in tot.items()}}))
