"""K5 tcgen05 GEMM vs a plain fp32 torch reference of the same op (same
half-precision inputs; f32 accumulation; output rounded once)."""
import pytest
import torch

from paper_2507_03312_b200 import vit_kernels as VK

pytestmark = pytest.mark.gpu


def close(got, want, rel=None):
    want = want.float()
    got = got.float()
    tol = rel if rel is not None else (1e-2 if got.dtype == torch.bfloat16 else 4e-3)
    err = (got - want).abs().max().item()
    scale = want.abs().max().item() + 1e-6
    assert err <= tol * scale, f"max err {err} vs scale {scale}"


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (384, 768, 768), (200, 1000, 96), (50, 64, 48), (1000, 2304, 256),
                                   (1300, 512, 3072)])
def test_linear_fwd_dgrad_wgrad(cuda, dt, M, N, K, cg):
    def ok(n):  # the pair path needs 128/256-wide N tiles
        return cg == 1 or n >= 256 or n == 128
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N)
    x = torch.randn(M, K, device=cuda, generator=g).to(dt)
    w = (torch.randn(K, N, device=cuda, generator=g) / K ** 0.5).to(dt)
    if ok(N):
        y = VK.linear_fwd(x, w, cta_group=cg)
        close(y, x.float() @ w.float())
    dy = torch.randn(M, N, device=cuda, generator=g).to(dt)
    if ok(K):
        dx = VK.linear_dgrad(dy, w, cta_group=cg)
        close(dx, dy.float() @ w.float().t())
    for split in (1, 2):
        if (M + 63) // 64 < split or not ok(N):
            continue
        dw = VK.linear_wgrad(x, dy, split_k=split, cta_group=cg)
        close(dw, x.float().t() @ dy.float())


@pytest.mark.parametrize("cg", [1, 2])
def test_epilogue_bias_gelu_residual_alpha(cuda, cg):
    dt = torch.bfloat16
    M, N, K = 1300, 512, 256
    x = torch.randn(M, K, device=cuda).to(dt)
    w = (torch.randn(K, N, device=cuda) / K ** 0.5).to(dt)
    b = torch.randn(N, device=cuda).to(dt)
    r = torch.randn(M, N, device=cuda).to(dt)
    pre = torch.empty(M, N, device=cuda, dtype=dt)
    y = VK.linear_fwd(x, w, bias=b, act=VK.ACT_GELU, aux=pre, cta_group=cg)
    z = x.float() @ w.float() + b.float()
    close(pre, z)
    close(y, torch.nn.functional.gelu(pre.float(), approximate="tanh"))
    y2 = VK.linear_fwd(x, w, bias=b, residual=r, cta_group=cg)
    close(y2, z + r.float())
    # GELU backward in the dgrad epilogue
    dh = torch.randn(M, N, device=cuda).to(dt)
    w2 = (torch.randn(K, N, device=cuda) / N ** 0.5).to(dt)
    dz = VK.linear_dgrad(dh, w2, cta_group=cg)
    close(dz, dh.float() @ w2.float().t())
    zin = torch.randn(M, K, device=cuda).to(dt)
    dzg = VK.linear_dgrad(dh, w2, aux=zin, cta_group=cg)
    zz = zin.float().requires_grad_(True)
    torch.nn.functional.gelu(zz, approximate="tanh").backward(dh.float() @ w2.float().t())
    close(dzg, zz.grad, rel=2e-2)
    # GELU forward saving round_half(gelu'(pre)) (ACT_GELU_D), and its backward as a
    # plain product (ACT_MUL_AUX): _bw_gelu rounds the derivative onto the
    # cotangent's grid before multiplying (autodiff.py:173-185)
    gd = torch.empty(M, N, device=cuda, dtype=dt)
    y3 = VK.linear_fwd(x, w, bias=b, act=VK.ACT_GELU_D, aux=gd, cta_group=cg)
    assert torch.equal(y3, y)  # the same GELU output as ACT_GELU
    zz = pre.float().requires_grad_(True)
    torch.nn.functional.gelu(zz, approximate="tanh").backward(torch.ones_like(zz))
    close(gd, zz.grad, rel=1e-2)
    dzm = VK.linear_dgrad(dh, w2, aux=zin, aux_act=VK.ACT_MUL_AUX, cta_group=cg)
    close(dzm, (dh.float() @ w2.float().t()) * zin.float())
    # alpha + f32 output
    o = VK.gemm(x, w, M=M, N=N, K=K, lda=K, ldb=N, b_mn=True, alpha=0.125, out_dtype=torch.float32, cta_group=cg)
    close(o, 0.125 * (x.float() @ w.float()), rel=1e-3)


def test_batched_strided_attention_shapes(cuda):
    """Q K^T and P V straight out of the [B, N, 3, H, hd] qkv layout."""
    dt = torch.float16
    Bsz, Nt, H, hd = 3, 197, 4, 64
    D = H * hd
    qkv = torch.randn(Bsz * Nt, 3 * D, device=cuda).to(dt)
    q = qkv.view(Bsz, Nt, 3, H, hd)[:, :, 0]
    k = qkv.view(Bsz, Nt, 3, H, hd)[:, :, 1]
    v = qkv.view(Bsz, Nt, 3, H, hd)[:, :, 2]
    ldS = 208
    S = torch.zeros(Bsz, H, Nt, ldS, device=cuda, dtype=dt)
    VK.gemm(qkv, qkv[:, D:], M=Nt, N=Nt, K=hd, lda=3 * D, ldb=3 * D, nb=(H, Bsz), a_sb=(hd, Nt * 3 * D),
            b_sb=(hd, Nt * 3 * D), out=S, ldc=ldS, c_sb=(Nt * ldS, H * Nt * ldS), alpha=0.125)
    ref = torch.einsum("bnhd,bmhd->bhnm", q.float(), k.float()) * 0.125
    close(S[..., :Nt], ref)
    P = torch.softmax(S[..., :Nt].float(), -1).to(dt)
    Ppad = torch.zeros(Bsz, H, Nt, ldS, device=cuda, dtype=dt)
    Ppad[..., :Nt] = P
    O = torch.empty(Bsz * Nt, D, device=cuda, dtype=dt)
    # O[b, n, h, :] = P[b,h] @ V[b,:,h,:]  (B operand MN-major: hd contiguous)
    VK.gemm(Ppad, qkv[:, 2 * D:], M=Nt, N=hd, K=Nt, lda=ldS, ldb=3 * D, b_mn=True, nb=(H, Bsz),
            a_sb=(Nt * ldS, H * Nt * ldS), b_sb=(hd, Nt * 3 * D), out=O, ldc=D, c_sb=(hd, Nt * D))
    refO = torch.einsum("bhnm,bmhd->bnhd", P.float(), v.float()).reshape(Bsz * Nt, D)
    close(O, refO)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("Nt", [197, 64, 130, 256, 17])
def test_fused_attention_forward(cuda, dt, Nt):
    Bsz, H, hd = 3, 4, 64
    D = H * hd
    g = torch.Generator(device=cuda).manual_seed(Nt)
    qkv = (torch.randn(Bsz * Nt, 3 * D, device=cuda, generator=g) * 1.5).to(dt)
    out = VK.attention_fwd(qkv, Bsz, Nt, H, hd, 0.125)
    q, k, v = (qkv.view(Bsz, Nt, 3, H, hd)[:, :, i].float() for i in range(3))
    s = (torch.einsum("bnhd,bmhd->bhnm", q, k) * 0.125).to(dt).float()  # scores rounded to half
    p = torch.softmax(s, -1).to(dt).float()
    ref = torch.einsum("bhnm,bmhd->bnhd", p, v).reshape(Bsz * Nt, D)
    close(out, ref)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("Nt", [197, 64, 130, 256, 17])
def test_fused_attention_backward(cuda, dt, Nt):
    Bsz, H, hd = 2, 3, 64
    D = H * hd
    g = torch.Generator(device=cuda).manual_seed(7 + Nt)
    qkv = torch.randn(Bsz * Nt, 3 * D, device=cuda, generator=g).to(dt)
    dO = torch.randn(Bsz * Nt, D, device=cuda, generator=g).to(dt)
    dqkv = VK.attention_bwd(qkv, dO, Bsz, Nt, H, hd, 0.125)
    # with the forward's row statistics P is rebuilt bit-identically
    # NaN-filled: every entry the backward reads must have been written by the forward
    stats = torch.full((VK.attention_stats_numel(Bsz, Nt, H),), float("nan"), device=cuda)
    VK.attention_fwd(qkv, Bsz, Nt, H, hd, 0.125, stats=stats)
    assert torch.equal(VK.attention_bwd(qkv, dO, Bsz, Nt, H, hd, 0.125, stats=stats), dqkv)
    # fused bias gradient: colsum over the stored dqkv rows
    cs = torch.empty(3 * D, device=cuda, dtype=dt)
    assert torch.equal(VK.attention_bwd(qkv, dO, Bsz, Nt, H, hd, 0.125, stats=stats, colsum_out=cs), dqkv)
    want = dqkv.float().sum(0)
    assert torch.allclose(cs.float(), want, rtol=1e-2, atol=1e-2 * want.abs().max().item())
    # the forward's saved P reloaded instead of recomputed (the engine's path)
    psave = torch.empty(VK.attention_psave_bytes(Bsz, Nt, H), dtype=torch.uint8, device=cuda)
    VK.attention_fwd(qkv, Bsz, Nt, H, hd, 0.125, p_save=psave)
    cs2 = torch.empty(3 * D, device=cuda, dtype=dt)
    dqkv_saved = VK.attention_bwd(qkv, dO, Bsz, Nt, H, hd, 0.125, p_saved=psave, colsum_out=cs2)
    want2 = dqkv_saved.float().sum(0)
    assert torch.allclose(cs2.float(), want2, rtol=1e-2, atol=1e-2 * want2.abs().max().item())
    x = qkv.float().requires_grad_(True)
    q, k, v = (x.view(Bsz, Nt, 3, H, hd)[:, :, i] for i in range(3))
    p = torch.softmax(torch.einsum("bnhd,bmhd->bhnm", q, k) * 0.125, -1)
    o = torch.einsum("bhnm,bmhd->bnhd", p, v).reshape(Bsz * Nt, D)
    o.backward(dO.float())
    for i, name in enumerate("qkv"):
        want = x.grad[:, i * D:(i + 1) * D]
        close(dqkv[:, i * D:(i + 1) * D], want, rel=3e-2)
        close(dqkv_saved[:, i * D:(i + 1) * D], want, rel=3e-2)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("Nt", [197, 64])
def test_softmax_epilogues(cuda, dt, Nt):
    """Q K^T with the softmax island in the epilogue, and dP = dO V^T with the
    softmax backward in the epilogue (aux = P), batched over (head, image)."""
    Bsz, H, hd = 2, 3, 64
    D = H * hd
    ld = -(-Nt // 16) * 16
    g = torch.Generator(device=cuda).manual_seed(Nt + 3)
    qkv = torch.randn(Bsz * Nt, 3 * D, device=cuda, generator=g).to(dt)
    dO = torch.randn(Bsz * Nt, D, device=cuda, generator=g).to(dt)
    P = torch.zeros(Bsz, H, Nt, ld, device=cuda, dtype=dt)
    VK.gemm(qkv, qkv[:, D:], M=Nt, N=Nt, K=hd, lda=3 * D, ldb=3 * D, nb=(H, Bsz), a_sb=(hd, Nt * 3 * D),
            b_sb=(hd, Nt * 3 * D), out=P, ldc=ld, c_sb=(Nt * ld, H * Nt * ld), alpha=0.125, act=VK.ACT_SOFTMAX)
    q, k, v = (qkv.view(Bsz, Nt, 3, H, hd)[:, :, i].float() for i in range(3))
    s = (torch.einsum("bnhd,bmhd->bhnm", q, k) * 0.125).to(dt).float()
    p = torch.softmax(s, -1)
    close(P[..., :Nt], p)
    dS = torch.zeros_like(P)
    VK.gemm(dO, qkv[:, 2 * D:], M=Nt, N=Nt, K=hd, lda=D, ldb=3 * D, nb=(H, Bsz), a_sb=(hd, Nt * D),
            b_sb=(hd, Nt * 3 * D), out=dS, ldc=ld, c_sb=(Nt * ld, H * Nt * ld), act=VK.ACT_SOFTMAX_BWD, aux=P,
            ld_aux=ld)
    dp = torch.einsum("bnhd,bmhd->bhnm", dO.float().view(Bsz, Nt, H, hd), v)
    ph = P[..., :Nt].float()
    want = ph * (dp - (ph * dp).sum(-1, keepdim=True))
    close(dS[..., :Nt], want, rel=2e-2)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(1000, 384, 256), (4096, 768, 3072), (333, 200, 128)])
def test_fused_colsum(cuda, dt, shape):
    """colsum_out = sum over rows of the stored (rounded) C, for the plain,
    GELU'-with-aux and bias+residual epilogues and the split-K fallback."""
    M, N, K = shape
    g = torch.Generator(device=cuda).manual_seed(M)
    x = torch.randn(M, K, device=cuda, generator=g).to(dt)
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).to(dt)
    aux = torch.randn(M, N, device=cuda, generator=g).to(dt)
    bias = torch.randn(N, device=cuda, generator=g).to(dt)
    res = torch.randn(M, N, device=cuda, generator=g).to(dt)
    for kw in ({}, {"aux": aux}):
        cs = torch.empty(N, device=cuda, dtype=dt)
        y = VK.linear_dgrad(x, w, colsum_out=cs, **kw)
        want = y.float().sum(0)
        assert torch.allclose(cs.float(), want, rtol=1e-2, atol=1e-2 * want.abs().max().item()), kw.keys()
    cs = torch.empty(N, device=cuda, dtype=dt)
    y = VK.gemm(x, w, M=M, N=N, K=K, lda=K, ldb=K, bias=bias, residual=res, colsum_out=cs)
    want = y.float().sum(0)
    assert torch.allclose(cs.float(), want, rtol=1e-2, atol=1e-2 * want.abs().max().item())
    cs = torch.empty(N, device=cuda, dtype=dt)
    y = VK.gemm(x, w, M=M, N=N, K=K, lda=K, ldb=K, split_k=2, colsum_out=cs)
    want = y.float().sum(0)
    assert torch.allclose(cs.float(), want, rtol=1e-2, atol=1e-2 * want.abs().max().item())


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(4096, 768, 2304), (1000, 320, 384), (777, 256, 768), (8192, 3072, 768),
                                   (4096, 1024, 1024), (1000, 320, 512), (2048, 768, 3072)])
def test_wide_wgrad(cuda, dt, shape):
    """The 256 x 384 weight-gradient tile (block_n 384, one accumulator, B chunks
    staged {2r, 2r+1, 4+r} per CTA) against fp32 and the 256 x 256 path, with
    and without split-K, including row counts that are not tile multiples."""
    T, K, N = shape
    g = torch.Generator(device=cuda).manual_seed(T + K)
    x = torch.randn(T, K, device=cuda, generator=g).to(dt)
    dy = torch.randn(T, N, device=cuda, generator=g).to(dt)
    want = x.float().t() @ dy.float()
    widths = [384] + ([512] if N % 512 == 0 else [])
    for width in widths:
        for split in (None, 1, 3):
            w = VK.linear_wgrad(x, dy, split_k=split, wide=width)
            close(w, want, rel=1e-2)
    close(VK.linear_wgrad(x, dy, wide=False), want, rel=1e-2)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_transpose_batch(cuda, dt):
    """mpx_transpose_batch (the forward's K-major weight copies): full 64 x 64
    tiles on the 16-byte path, ragged edges, odd widths and padded rows."""
    g = torch.Generator(device=cuda).manual_seed(5)
    shapes = [(768, 2304), (3072, 768), (100, 37), (64, 64), (129, 200), (1, 9)]
    srcs = [torch.randn(r, c, device=cuda, generator=g).to(dt) for r, c in shapes]
    outs = [torch.empty(c, r, device=cuda, dtype=dt) for r, c in shapes]
    VK.transpose_batch(srcs, outs)
    for s_, o in zip(srcs, outs):
        assert torch.equal(o, s_.t())
    big = torch.randn(256, 136, device=cuda, generator=g).to(dt)[:, :128]  # ld 136, 16-byte rows
    out = torch.empty(128, 264, device=cuda, dtype=dt)[:, :256]
    VK.transpose_batch([big], [out])
    assert torch.equal(out, big.t())


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(1000, 768, 256), (333, 200, 128), (4096, 3072, 768)])
def test_epilogue_paths_bit_identical(cuda, dt, shape):
    """The staged epilogue variants (whole-group fast paths with FHADD operand adds,
    the packed GELU math, partial groups) against the generic direct-store epilogue
    (tma_store=-1) on the same tiles: the accumulators are the same MMAs, so every
    epilogue must give the same bits — bias, bias + residual, the saved GELU
    derivative as a product (MUL_AUX), gelu' of a saved pre-activation, and GELU with
    the pre-activation or the derivative written out."""
    M, N, K = shape
    g = torch.Generator(device=cuda).manual_seed(M + N)
    x = torch.randn(M, K, device=cuda, generator=g).to(dt)
    w = (torch.randn(K, N, device=cuda, generator=g) * 0.05).to(dt)
    bias = torch.randn(N, device=cuda, generator=g).to(dt)
    res = torch.randn(M, N, device=cuda, generator=g).to(dt)
    aux = torch.randn(M, N, device=cuda, generator=g).to(dt)
    common = dict(M=M, N=N, K=K, lda=K, ldb=N, b_mn=True)
    cases = [dict(), dict(bias=bias), dict(bias=bias, residual=res, ldr=N), dict(aux=aux, ld_aux=N, act=VK.ACT_MUL_AUX),
             dict(aux=aux, ld_aux=N, act=VK.ACT_GELU_BWD)]
    for kw in cases:
        y0 = VK.gemm(x, w, **common, **kw)
        y1 = VK.gemm(x, w, **common, tma_store=-1, **kw)
        assert torch.equal(y0.view(torch.int16), y1.view(torch.int16)), list(kw)
    for act in (VK.ACT_GELU, VK.ACT_GELU_D):
        a0, a1 = torch.empty_like(aux), torch.empty_like(aux)
        y0 = VK.gemm(x, w, **common, bias=bias, aux=a0, ld_aux=N, act=act)
        y1 = VK.gemm(x, w, **common, tma_store=-1, bias=bias, aux=a1, ld_aux=N, act=act)
        assert torch.equal(y0.view(torch.int16), y1.view(torch.int16)), act
        assert torch.equal(a0.view(torch.int16), a1.view(torch.int16)), act


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_fused_attention_backward_many_items(cuda, dt):
    """Several (image, head) items per CTA of the persistent backward: the qkv-bias column
    sums handed from the softmax warps to warps 1-3 item by item (double-buffered barriers
    with back-pressure) against the column sums of the stored rows; repeated launches agree."""
    Bsz, Nt, H, hd = 64, 197, 12, 64
    D = H * hd
    g = torch.Generator(device=cuda).manual_seed(11)
    qkv = torch.randn(Bsz * Nt, 3 * D, device=cuda, generator=g).to(dt)
    dO = torch.randn(Bsz * Nt, D, device=cuda, generator=g).to(dt)
    psave = torch.empty(VK.attention_psave_bytes(Bsz, Nt, H), dtype=torch.uint8, device=cuda)
    VK.attention_fwd(qkv, Bsz, Nt, H, hd, 0.125, p_save=psave)
    cs = torch.empty(3 * D, device=cuda, dtype=dt)
    dqkv = VK.attention_bwd(qkv, dO, Bsz, Nt, H, hd, 0.125, p_saved=psave, colsum_out=cs)
    want = dqkv.float().sum(0)
    assert torch.allclose(cs.float(), want, rtol=1e-2, atol=1e-2 * want.abs().max().item())
    cs2 = torch.empty_like(cs)
    dqkv2 = VK.attention_bwd(qkv, dO, Bsz, Nt, H, hd, 0.125, p_saved=psave, colsum_out=cs2)
    assert torch.equal(dqkv2, dqkv) and torch.equal(cs2, cs)
