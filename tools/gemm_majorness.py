import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2507_03312_b200 import vit_kernels as VK
M, K, N = 50432, 768, 3072
x = torch.randn(M, K, device="cuda").bfloat16(); xt = x.t().contiguous()  # [K, M]
w = (torch.randn(K, N, device="cuda") * 0.03).bfloat16(); wt = w.t().contiguous()  # [N, K]
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record()
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize(); return round(a.elapsed_time(b) / 20 * 1000, 1)
print("A K-major,  B MN-major", t(lambda: VK.gemm(x, w, M=M, N=N, K=K, lda=K, ldb=N, b_mn=True, out=y, ldc=N)))
print("A K-major,  B K-major ", t(lambda: VK.gemm(x, wt, M=M, N=N, K=K, lda=K, ldb=K, out=y, ldc=N)))
print("A MN-major, B MN-major", t(lambda: VK.gemm(xt, w, M=M, N=N, K=K, lda=M, ldb=N, a_mn=True, b_mn=True, out=y, ldc=N)))
print("A MN-major, B K-major ", t(lambda: VK.gemm(xt, wt, M=M, N=N, K=K, lda=M, ldb=K, a_mn=True, out=y, ldc=N)))
