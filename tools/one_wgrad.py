import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2507_03312_b200 import vit_kernels as VK
M = 256 * 197
K, N = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn(M, K, device="cuda").bfloat16(); dy = torch.randn(M, N, device="cuda").bfloat16()
dw = torch.empty(K, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3): VK.linear_wgrad(x, dy, out=dw)
torch.cuda.synchronize(); print("ok")
