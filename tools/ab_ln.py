"""Same-box A/B of the LayerNorm kernels at the ViT-B shape (M = 50432,
D = 768, bf16) between library builds; prints fwd / bwd us and a digest of
the outputs.  python tools/ab_ln.py libA.so libB.so [rounds]"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import sys, torch, hashlib
sys.path.insert(0, sys.argv[1])
from paper_2507_03312_b200 import _native as N
M, D = 256 * 197, 768
bf = torch.bfloat16
g0 = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(M, D, device="cuda", generator=g0).to(bf)
g = (1 + 0.1 * torch.randn(D, device="cuda", generator=g0)).to(bf)
bb = (0.1 * torch.randn(D, device="cuda", generator=g0)).to(bf)
y = torch.empty_like(x)
mu = torch.empty(M, device="cuda"); rs = torch.empty(M, device="cuda")
dy = torch.randn(M, D, device="cuda", generator=g0).to(bf)
dres = torch.randn(M, D, device="cuda", generator=g0).to(bf)
dx = torch.empty_like(x)
dg, db, dxs = (torch.empty(D, device="cuda", dtype=bf) for _ in range(3))
ws = torch.empty(8 << 20, device="cuda")
lib = N.load(); st = torch.cuda.current_stream().cuda_stream
fwd = lambda: N.check(lib.mpx_layernorm_fwd(2, x.data_ptr(), D, g.data_ptr(), bb.data_ptr(), y.data_ptr(), D,
                                            mu.data_ptr(), rs.data_ptr(), M, D, 1e-5, st), "ln_fwd")
bwd = lambda: N.check(lib.mpx_layernorm_bwd2(2, x.data_ptr(), D, g.data_ptr(), mu.data_ptr(), rs.data_ptr(),
                                             dy.data_ptr(), D, dres.data_ptr(), D, dx.data_ptr(), D, dg.data_ptr(),
                                             db.data_ptr(), dxs.data_ptr(), ws.data_ptr(), ws.numel(), M, D, st), "ln_bwd2")
def t(fn, it=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1000
tf, tb = t(fwd), t(bwd)
h = hashlib.sha1()
for v in (y, mu, rs, dx, dg, db, dxs): h.update(v.contiguous().view(torch.uint8).cpu().numpy().tobytes())
print(f"{tf:.1f} {tb:.1f} {h.hexdigest()[:12]}")
"""


def main():
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    rounds = int(next((a for a in sys.argv[1:] if a.isdigit()), "3"))
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, MPX_B200_LIB=str((ROOT / lib).resolve()))
            out = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True,
                                 timeout=300)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
            print(f"round {r} {lib:45s} fwd/bwd us, digest: {line}", flush=True)


if __name__ == "__main__":
    main()
