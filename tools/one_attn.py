"""ViT-B/16 bs256 fused attention forward + backward (for ncu)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
S, H, hd = 197, 12, 64
qkv = torch.randn(B * S, 3 * H * hd, device="cuda").to(torch.bfloat16)
dO = torch.randn(B * S, H * hd, device="cuda").to(torch.bfloat16)
st = torch.empty(VK.attention_stats_numel(B, S, H), device="cuda")
for _ in range(3):
    o = VK.attention_fwd(qkv, B, S, H, hd, 0.125, stats=st)
    d = VK.attention_bwd(qkv, dO, B, S, H, hd, 0.125, stats=st)
torch.cuda.synchronize()
print("ok")
