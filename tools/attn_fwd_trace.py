"""Phase timeline of the persistent fused attention forward (needs the
-DMPX_TRACE build, -DMPX_TRACE_IT=k picks the traced item of each CTA):
median over the first 64 CTAs of the time since the item's start."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("MPX_B200_LIB", str(ROOT / "abl" / "libmpx_trace.so"))
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2507_03312_b200 import _native  # noqa: E402
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

B, S, H, hd = 256, 197, 12, 64
qkv = torch.randn(B * S, 3 * H * hd, device="cuda").to(torch.bfloat16)
ps = torch.empty(VK.attention_psave_bytes(B, S, H), dtype=torch.uint8, device="cuda")
for _ in range(3):
    VK.attention_fwd(qkv, B, S, H, hd, 0.125, p_save=ps)
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_longlong * (64 * 32))()
assert lib.mpx_debug_attn_trace(buf) == 0
a = np.frombuffer(buf, dtype=np.int64).reshape(64, 32).astype(np.float64)
a = a - a[:, :1]
names = {0: "issuer: item start", 20: "issuer: next item start"}
for t in range(2):
    names.update({1 + 8 * t: f"t{t} smx: S ready", 2 + 8 * t: f"t{t} smx: softmax done", 3 + 8 * t: f"t{t} smx: previous O drained",
                  4 + 8 * t: f"t{t} smx: P tile free", 5 + 8 * t: f"t{t} smx: P stored"})
for k in sorted(names, key=lambda k: np.median(a[:, k])):
    print(f"{np.median(a[:, k]) / 1.9e3:8.2f} us  {names[k]}")
