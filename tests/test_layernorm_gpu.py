"""K7 LayerNorm backward (mpx_layernorm_bwd2) against an fp32 torch
restatement of the reference island (tensors.py:459-491, autodiff.py:243-262):
dx (+ residual), dgain, dbias and the column sum of the stored dx, for the
one-pass kernel (D <= 768) and the two-kernel path (D = 1024)."""
import pytest
import torch

from paper_2507_03312_b200 import _native as N

pytestmark = pytest.mark.gpu


def _ln_bwd2(dtype, x, g, mu, rs, dy, dres, M, D, ws):
    lib = N.load()
    dx = torch.empty_like(x)
    dg, db, dxs = (torch.empty(D, device=x.device, dtype=x.dtype) for _ in range(3))
    code = 2 if dtype == torch.bfloat16 else 1
    N.check(lib.mpx_layernorm_bwd2(code, x.data_ptr(), D, g.data_ptr(), mu.data_ptr(), rs.data_ptr(), dy.data_ptr(),
                                   D, dres.data_ptr() if dres is not None else None, D if dres is not None else 0,
                                   dx.data_ptr(), D, dg.data_ptr(), db.data_ptr(), dxs.data_ptr(), ws.data_ptr(),
                                   ws.numel(), M, D, torch.cuda.current_stream().cuda_stream), "ln_bwd2")
    return dx, dg, db, dxs


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,D", [(4099, 768), (1000, 256), (777, 512), (513, 1024)])
@pytest.mark.parametrize("res", [True, False])
def test_layernorm_bwd2(cuda, dtype, M, D, res):
    g0 = torch.Generator(device=cuda).manual_seed(M + D)
    x = torch.randn(M, D, device=cuda, generator=g0).to(dtype)
    g = (1 + 0.1 * torch.randn(D, device=cuda, generator=g0)).to(dtype)
    xf = x.float()
    mu = xf.mean(1)
    rs = torch.rsqrt(xf.var(1, unbiased=False) + 1e-5)
    dy = torch.randn(M, D, device=cuda, generator=g0).to(dtype)
    dres = torch.randn(M, D, device=cuda, generator=g0).to(dtype) if res else None
    ws = torch.empty(8 << 20, device=cuda)
    dx, dg, db, dxs = _ln_bwd2(dtype, x, g, mu, rs, dy, dres, M, D, ws)
    xh = (xf - mu[:, None]) * rs[:, None]
    d = dy.float() * g.float()
    ref = rs[:, None] * (d - d.mean(1, keepdim=True) - xh * (d * xh).mean(1, keepdim=True))
    if res:
        ref = ref + dres.float()

    def close(got, want, tol):
        assert ((got.float() - want).abs().max() / want.abs().max()).item() < tol

    close(dx, ref, 1e-2)
    close(dg, (dy.float() * xh).sum(0), 1e-2)
    close(db, dy.float().sum(0), 1e-2)
    close(dxs, dx.float().sum(0), 1e-2)  # the column sum of the stored (rounded) dx

