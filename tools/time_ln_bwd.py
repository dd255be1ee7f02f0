"""Time mpx_layernorm_bwd2 at the ViT-B shape (M=50432, D=768, bf16, with
residual and dx column sum); MPX_LN_FUSED=0 selects the two-kernel path.
Also checks the outputs against an fp32 torch restatement."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import _native as N  # noqa: E402

M, D = 256 * 197, int(sys.argv[3]) if len(sys.argv) > 3 else 768  # argv[3]: width (1024 = ViT-L)
bf = torch.bfloat16
torch.manual_seed(0)
dev = "cuda"
x = torch.randn(M, D, device=dev).to(bf)
g = (1 + 0.1 * torch.randn(D, device=dev)).to(bf)
xf = x.float()
mu = xf.mean(1)
rs = torch.rsqrt(xf.var(1, unbiased=False) + 1e-5)
dy = torch.randn(M, D, device=dev).to(bf)
dres = torch.randn(M, D, device=dev).to(bf)
dx = torch.empty(M, D, device=dev, dtype=bf)
dg, db, dxs = (torch.empty(D, device=dev, dtype=bf) for _ in range(3))
ws = torch.empty(8 << 20, device=dev)
lib = N.load()
st = torch.cuda.current_stream().cuda_stream


def run():
    N.check(lib.mpx_layernorm_bwd2(2, x.data_ptr(), D, g.data_ptr(), mu.data_ptr(), rs.data_ptr(), dy.data_ptr(), D,
                                   dres.data_ptr(), D, dx.data_ptr(), D, dg.data_ptr(), db.data_ptr(), dxs.data_ptr(),
                                   ws.data_ptr(), ws.numel(), M, D, st), "ln_bwd2")


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ITERS = int(sys.argv[1]) if len(sys.argv) > 1 else 20
e0.record()
for _ in range(ITERS):
    run()
e1.record()
torch.cuda.synchronize()
xh = (xf - mu[:, None]) * rs[:, None]
d = dy.float() * g.float()
ref = rs[:, None] * (d - d.mean(1, keepdim=True) - xh * (d * xh).mean(1, keepdim=True)) + dres.float()
err = ((dx.float() - ref).abs().max() / ref.abs().max()).item()
e_dg = ((dg.float() - (dy.float() * xh).sum(0)).abs().max() / (dy.float() * xh).sum(0).abs().max()).item()
e_xs = ((dxs.float() - dx.float().sum(0)).abs().max() / dx.float().sum(0).abs().max()).item()
import hashlib  # noqa: E402

digest = hashlib.sha1(b"".join(t.view(torch.int16).cpu().numpy().tobytes() for t in (dx, dg, db, dxs))).hexdigest()[:12]
out = {"ln_bwd2_us": round(e0.elapsed_time(e1) / ITERS * 1000, 1), "dx_rel": err, "dgain_rel": e_dg, "dxsum_rel": e_xs,
       "digest": digest}
if len(sys.argv) > 2:  # steady-state time and NVML energy (power-capped regime): [iters] [seconds]
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from energy import Meter  # noqa: E402

    n, ms, j, w, mhz = Meter(0).run(run, float(sys.argv[2]))
    out.update({"steady_us": round(ms * 1e3, 2), "mJ": round(j * 1e3, 2), "W": round(w, 1), "sm_mhz": mhz})
print(json.dumps(out))
