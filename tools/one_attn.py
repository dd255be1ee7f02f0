"""ViT-B/16 bs256 fused attention forward + backward as the engine runs them
(forward saves P, backward reloads it) — for ncu / timing."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
S, H, hd = 197, 12, 64
qkv = torch.randn(B * S, 3 * H * hd, device="cuda").to(torch.bfloat16)
dO = torch.randn(B * S, H * hd, device="cuda").to(torch.bfloat16)
ps = torch.empty(VK.attention_psave_bytes(B, S, H), dtype=torch.uint8, device="cuda")
cs = torch.empty(3 * H * hd, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    o = VK.attention_fwd(qkv, B, S, H, hd, 0.125, p_save=ps)
    d = VK.attention_bwd(qkv, dO, B, S, H, hd, 0.125, p_saved=ps, colsum_out=cs)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
for _ in range(10):
    VK.attention_fwd(qkv, B, S, H, hd, 0.125, p_save=ps)
e[1].record()
for _ in range(10):
    VK.attention_bwd(qkv, dO, B, S, H, hd, 0.125, p_saved=ps, colsum_out=cs)
e[2].record()
torch.cuda.synchronize()
print(f"fwd (saving P) {e[0].elapsed_time(e[1]) / 10:.3f} ms  bwd (reloading P) {e[1].elapsed_time(e[2]) / 10:.3f} ms")
