"""Same-box A/B of the fused attention kernels (the engine's path: forward
saving P, backward reloading it) between library builds.

    python tools/ab_attn.py abl/libmpx_head.so paper_2507_03312_b200/lib/libmpx_b200.so [rounds]

Each build runs in its own subprocess (the library is loaded once per
process); builds alternate for `rounds` rounds.  Prints fwd / bwd ms and
whether the outputs are bit-identical to the first build's."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, torch, hashlib
sys.path.insert(0, sys.argv[1])
from paper_2507_03312_b200 import vit_kernels as VK
B, S, H, hd = 256, 197, 12, 64
D = H * hd
dt = torch.bfloat16 if sys.argv[2] == "bf16" else torch.float16
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(B * S, 3 * D, device="cuda", generator=g).to(dt)
dO = torch.randn(B * S, D, device="cuda", generator=g).to(dt)
O = torch.empty(B * S, D, device="cuda", dtype=dt)
dqkv = torch.empty_like(qkv)
ps = torch.empty(VK.attention_psave_bytes(B, S, H), dtype=torch.uint8, device="cuda")
cs = torch.empty(3 * D, device="cuda", dtype=dt)
fwd = lambda: VK.attention_fwd(qkv, B, S, H, hd, 0.125, out=O, p_save=ps)
bwd = lambda: VK.attention_bwd(qkv, dO, B, S, H, hd, 0.125, dqkv=dqkv, p_saved=ps, colsum_out=cs)
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
tf, tb = t(fwd), t(bwd)
fwd(); bwd(); torch.cuda.synchronize()
h = hashlib.sha1()
for x in (O, dqkv, cs): h.update(x.view(torch.uint8).cpu().numpy().tobytes())
print(f"{tf:.4f} {tb:.4f} {h.hexdigest()[:12]}")
"""


def main():
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    rounds = int(next((a for a in sys.argv[1:] if a.isdigit()), "3"))
    fmt = "f16" if "f16" in sys.argv[1:] else "bf16"
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, MPX_B200_LIB=str((ROOT / lib).resolve()))
            out = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), fmt], env=env, capture_output=True,
                                 text=True, timeout=300)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
            print(f"round {r} {lib:45s} fwd/bwd ms, digest: {line}", flush=True)


if __name__ == "__main__":
    main()
