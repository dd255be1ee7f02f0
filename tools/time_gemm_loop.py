"""Steady-state time and NVML energy of one ViT-B GEMM shape launched back to
back (power-capped regime): python tools/time_gemm_loop.py <mode> [seconds] [cta_group]."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from energy import Meter  # noqa: E402
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "gelu_d"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
M, K, N = 256 * 197, 768, 3072
bf = torch.bfloat16
x = torch.randn(M, K, device="cuda").to(bf)
w = (torch.randn(K, N, device="cuda") * 0.03).to(bf)
wt = w.t().contiguous()
b = (torch.randn(N, device="cuda") * 0.1).to(bf)
y = torch.empty(M, N, device="cuda", dtype=bf)
aux = torch.randn(M, N, device="cuda").to(bf)
cg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
b_cs = torch.empty(N, device="cuda", dtype=bf)
w2 = (torch.randn(N, K, device="cuda") * 0.02).to(bf)  # W2 [3072, 768]
ws_cs = torch.empty(((M + 31) // 32) * N, device="cuda")
x2 = torch.randn(M, N, device="cuda").to(bf)  # fc2 forward: [M, 3072] @ [3072, 768] + b + residual
w2t = (torch.randn(K, N, device="cuda") * 0.02).to(bf)
res = torch.randn(M, K, device="cuda").to(bf)
b2 = (torch.randn(K, device="cuda") * 0.1).to(bf)
o2 = torch.empty(M, K, device="cuda", dtype=bf)
xp = torch.randn(M, K, device="cuda").to(bf)  # proj forward: [M, 768] @ [768, 768] + b + residual
wpt = (torch.randn(K, K, device="cuda") * 0.03).to(bf)
from paper_2507_03312_b200 import _native as NN  # noqa: E402
from paper_2507_03312_b200.kernels import stream_handle  # noqa: E402

lg = torch.ones(K, device="cuda", dtype=bf)
lb = torch.zeros(K, device="cuda", dtype=bf)
ln_o = torch.empty(M, K, device="cuda", dtype=bf)
mu = torch.empty(M, device="cuda")
rs = torch.empty(M, device="cuda")


def sep(xa, wa):  # residual GEMM, then the standalone LayerNorm kernel
    VK.linear_fwd_t(xa, wa, bias=b2, residual=res, out=o2)
    NN.check(NN.load().mpx_layernorm_fwd(2, o2.data_ptr(), K, lg.data_ptr(), lb.data_ptr(), ln_o.data_ptr(), K,
                                         mu.data_ptr(), rs.data_ptr(), M, K, 1e-5, stream_handle(o2.device)), "ln")


fns = {
    "fc2_ln": lambda: VK.linear_fwd_t(x2, w2t, bias=b2, residual=res, out=o2, ln=(lg, lb, ln_o, mu, rs, 1e-5)),
    "fc2_res_sep": lambda: sep(x2, w2t),
    "proj_ln": lambda: VK.linear_fwd_t(xp, wpt, bias=b2, residual=res, out=o2, ln=(lg, lb, ln_o, mu, rs, 1e-5)),
    "proj_res_sep": lambda: sep(xp, wpt),
    "fc2_ln_dry": lambda: VK.linear_fwd_t(x2, w2t, bias=b2, residual=res, out=o2, ln=(lg, lb, ln_o, mu, rs, -1.0)),
    "proj_ln_dry": lambda: VK.linear_fwd_t(xp, wpt, bias=b2, residual=res, out=o2, ln=(lg, lb, ln_o, mu, rs, -1.0)),
    "fc2_res": lambda: VK.linear_fwd_t(x2, w2t, bias=b2, residual=res, out=o2),
    "fc2_res": lambda: VK.linear_fwd_t(x2, w2t, bias=b2, residual=res, out=o2, cta_group=cg),
    "proj_res": lambda: VK.linear_fwd_t(xp, wpt, bias=b2, residual=res, out=o2, cta_group=cg),
    "gelu_d": lambda: VK.linear_fwd_t(x, wt, bias=b, act=VK.ACT_GELU_D, aux=aux, out=y),
    "gelu": lambda: VK.linear_fwd_t(x, wt, bias=b, act=VK.ACT_GELU, aux=aux, out=y),
    "bare": lambda: VK.linear_fwd_t(x, wt, out=y),
    "mul_aux": lambda: VK.linear_dgrad(aux, w, aux=y, out=x, aux_act=VK.ACT_MUL_AUX),
    # the fc2 dgrad as the engine runs it: dpre[M, 3072] = dX[M, 768] @ W2^T, x the saved gelu', + colsum
    "fc2_dgrad": lambda: VK.linear_dgrad(res, w2, aux=aux, out=y, aux_act=VK.ACT_MUL_AUX, colsum_out=b_cs,
                                         colsum_ws=ws_cs),
}
n, ms, j, wts, mhz = Meter(0).run(fns[mode], secs)
print(json.dumps({"mode": mode, "us": round(ms * 1e3, 2), "mJ": round(j * 1e3, 2), "W": round(wts, 1), "sm_mhz": mhz}))
