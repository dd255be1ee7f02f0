"""Time the fc1-shaped GEMM (M=50432, K=768, N=3072, bf16) in each epilogue
mode the ViT uses: bare, bias+GELU with aux out, GELU' with aux in (fc2
dgrad), bias+residual (fc2 forward) — forward modes on K-major weight copies
as the engine runs them — and the fc1 weight gradient on the wide 256x384
tile (K = 50432 tokens, split-K)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

M, K, N = 256 * 197, 768, 3072
bf = torch.bfloat16
x = torch.randn(M, K, device="cuda").to(bf)
w = (torch.randn(K, N, device="cuda") * 0.03).to(bf)
b = (torch.randn(N, device="cuda") * 0.1).to(bf)
y = torch.empty(M, N, device="cuda", dtype=bf)
aux = torch.randn(M, N, device="cuda").to(bf)
dy = torch.randn(M, K, device="cuda").to(bf)
w2 = (torch.randn(N, K, device="cuda") * 0.03).to(bf)
res = torch.randn(M, K, device="cuda").to(bf)
out_k = torch.empty(M, K, device="cuda", dtype=bf)
wt, w2t = w.t().contiguous(), w2.t().contiguous()
dw = torch.empty(K, N, device="cuda", dtype=bf)
modes = {
    "bare": lambda: VK.linear_fwd_t(x, wt, out=y),
    "gelu_aux_out": lambda: VK.linear_fwd_t(x, wt, bias=b, act=VK.ACT_GELU, aux=aux, out=y),
    "gelu_bwd_aux_in": lambda: VK.linear_dgrad(dy, w2, aux=aux, out=y),
    "bias_residual": lambda: VK.linear_fwd_t(y, w2t, bias=b[:K], residual=res, out=out_k),
    "wgrad_wide": lambda: VK.linear_wgrad(x, aux, out=dw),
}
only = sys.argv[1:]  # optional subset (for ncu)
res_ = {}
for name, fn in modes.items():
    if only and name not in only:
        continue
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res_[name] = round(e0.elapsed_time(e1) / 20 * 1000, 1)
print(json.dumps({"gemm_modes_us": res_}))
