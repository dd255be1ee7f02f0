"""One ViT-B fc1-shaped GEMM (M=50432, K=768, N=3072, bf16) for ncu.
argv[1]: "bare" (default), "gelu" (bias + GELU, pre-activation saved to aux:
the fc1 forward), "gelu_bwd" (fc2 dgrad with the GELU derivative from aux),
"res" (fc2 forward: bias + residual), "gelu_d" / "mul_aux" (the round-2 fc1
forward saving gelu' and the fc2 dgrad multiplying by it)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "bare"
M, K, N = 256 * 197, 768, 3072
bf = torch.bfloat16
x = torch.randn(M, K, device="cuda").to(bf)
w = (torch.randn(K, N, device="cuda") * 0.03).to(bf)
b = (torch.randn(N, device="cuda") * 0.1).to(bf)
y = torch.empty(M, N, device="cuda", dtype=bf)
aux = torch.randn(M, N, device="cuda").to(bf)
dx = torch.empty(M, K, device="cuda", dtype=bf)
w2 = (torch.randn(N, K, device="cuda") * 0.03).to(bf)
res = torch.randn(M, K, device="cuda").to(bf)
for _ in range(4):
    if mode == "bare":
        VK.linear_fwd(x, w, out=y)
    elif mode == "gelu":
        VK.linear_fwd(x, w, bias=b, act=VK.ACT_GELU, aux=aux, out=y)
    elif mode == "gelu_bwd":
        VK.linear_dgrad(aux, w, aux=y, out=x)
    elif mode == "gelu_d":  # the round-2 fc1 forward: GELU + its rounded derivative saved to aux
        VK.linear_fwd(x, w, bias=b, act=VK.ACT_GELU_D, aux=aux, out=y)
    elif mode == "mul_aux":  # the round-2 fc2 dgrad: the saved derivative as a plain product
        VK.linear_dgrad(aux, w, aux=y, out=x, aux_act=VK.ACT_MUL_AUX)
    elif mode == "res":
        VK.linear_fwd(aux, w2, bias=b[:K], residual=res, out=dx)
torch.cuda.synchronize()
print("ok", mode)
