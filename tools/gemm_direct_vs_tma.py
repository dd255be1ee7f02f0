import sys, json, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK
M, K, N = 256 * 197, 768, 3072
bf = torch.bfloat16
x = torch.randn(M, K, device="cuda").to(bf)
w = (torch.randn(K, N, device="cuda") * 0.03).to(bf)
wt = w.t().contiguous()
b = (torch.randn(N, device="cuda") * 0.1).to(bf)
y = torch.empty(M, N, device="cuda", dtype=bf)
aux = torch.randn(M, N, device="cuda").to(bf)
dy = torch.randn(M, K, device="cuda").to(bf)
w2 = (torch.randn(N, K, device="cuda") * 0.03).to(bf)
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(e) / it * 1000, 1)
r = {}
for ts in (0, -1):
    r[f"aux_out_tma{ts}"] = t(lambda: VK.gemm(x, wt, M=M, N=N, K=K, lda=K, ldb=K, bias=b, act=VK.ACT_GELU, aux=aux, out=y, ldc=N, tma_store=ts))
    r[f"aux_in_tma{ts}"] = t(lambda: VK.gemm(dy, w2, M=M, N=N, K=K, lda=K, ldb=K, aux=aux, act=VK.ACT_GELU_BWD, out=y, ldc=N, tma_store=ts))
print(json.dumps(r))
