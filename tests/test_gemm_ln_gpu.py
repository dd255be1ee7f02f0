"""The residual GEMM with the LayerNorm of its stored rows fused in
(mpx_gemm_desc.ln_*): a cluster of three CTA pairs per 256-row
block exchanges row sums over distributed shared memory.  Against the
unfused pair (the same GEMM, then mpx_layernorm_fwd on its output):
  * the stored residual stream x is bit-identical (same epilogue);
  * LN(x) agrees to one unit of the half format's grid (the fused kernel
    takes the variance as E[x^2] - mean^2 of the rounded row, the separate
    kernel two-pass) and to an fp32 torch LayerNorm of x within 2 grid units;
  * the saved row mean / rstd agree to 1e-5 relative."""
import pytest
import torch

from paper_2507_03312_b200 import _native as N
from paper_2507_03312_b200 import vit_kernels as VK
from paper_2507_03312_b200.kernels import stream_handle

pytestmark = pytest.mark.gpu
CODE = {torch.float16: 1, torch.bfloat16: 2}


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,K", [(50432, 768), (1536, 3072), (300, 768), (256, 768), (2000, 768), (68, 768), (1, 768)])
def test_fused_layernorm_matches_separate(cuda, dt, M, K):
    D = 768
    g = torch.Generator(device=cuda).manual_seed(M + K)
    x = torch.randn(M, K, device=cuda, generator=g).to(dt)
    wt = (torch.randn(D, K, device=cuda, generator=g) / K ** 0.5).to(dt)
    b = (0.1 * torch.randn(D, device=cuda, generator=g)).to(dt)
    res = torch.randn(M, D, device=cuda, generator=g).to(dt)
    lg = (1 + 0.1 * torch.randn(D, device=cuda, generator=g)).to(dt)
    lb = (0.1 * torch.randn(D, device=cuda, generator=g)).to(dt)
    # unfused: GEMM + bias + residual, then the LayerNorm kernel
    y_ref = VK.linear_fwd_t(x, wt, bias=b, residual=res)
    ln_ref = torch.empty_like(y_ref)
    mu_ref = torch.empty(M, device=cuda)
    rs_ref = torch.empty(M, device=cuda)
    N.check(N.load().mpx_layernorm_fwd(CODE[dt], y_ref.data_ptr(), D, lg.data_ptr(), lb.data_ptr(), ln_ref.data_ptr(),
                                       D, mu_ref.data_ptr(), rs_ref.data_ptr(), M, D, 1e-5, stream_handle(cuda)), "ln")
    # fused
    y = torch.empty_like(y_ref)
    ln_out = torch.empty_like(y_ref)
    mu = torch.empty(M, device=cuda)
    rs = torch.empty(M, device=cuda)
    VK.linear_fwd_t(x, wt, bias=b, residual=res, out=y, ln=(lg, lb, ln_out, mu, rs, 1e-5))
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    ulp = 2.0 ** -7 if dt == torch.bfloat16 else 2.0 ** -10
    d = (ln_out.float() - ln_ref.float()).abs()
    assert (d <= ulp * ln_ref.float().abs().clamp_min(1.0) + 1e-6).all(), d.max()
    ref = torch.nn.functional.layer_norm(y.float(), (D,), lg.float(), lb.float(), eps=1e-5)
    assert ((ln_out.float() - ref).abs() <= 2 * ulp * ref.abs().clamp_min(1.0)).all()
    assert torch.allclose(mu, mu_ref, rtol=1e-5, atol=1e-6) and torch.allclose(rs, rs_ref, rtol=1e-5)


def test_fused_layernorm_refuses_unsupported_shapes(cuda):
    x = torch.randn(512, 768, device=cuda).to(torch.bfloat16)
    wt = torch.randn(512, 768, device=cuda).to(torch.bfloat16)  # N = 512 != 768
    res = torch.randn(512, 512, device=cuda).to(torch.bfloat16)
    o = torch.empty(512, 512, device=cuda, dtype=torch.bfloat16)
    v = torch.ones(512, device=cuda, dtype=torch.bfloat16)
    st = torch.empty(512, device=cuda)
    with pytest.raises(N.NativeError):
        VK.linear_fwd_t(x, wt, residual=res, ln=(v, v, o, st, st, 1e-5))
