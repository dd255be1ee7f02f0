"""Tensor-level wrappers of the ViT kernels (K5 GEMM, K6 attention softmax,
K7 LayerNorm, K9 cross-entropy, patchify, column sums).  torch provides
memory and streams; every arithmetic op runs in libmpx_b200.so."""
from __future__ import annotations

import ctypes
import os

import torch

from . import _native as _nat
from .kernels import require_cuda, stream_handle

_CODE = {torch.float32: _nat.MPX_F32, torch.float16: _nat.MPX_F16, torch.bfloat16: _nat.MPX_BF16}
ACT_NONE, ACT_GELU, ACT_GELU_BWD, ACT_SOFTMAX, ACT_SOFTMAX_BWD, ACT_GELU_D, ACT_MUL_AUX = 0, 1, 2, 3, 4, 5, 6


def _ptr(t):
    return t.data_ptr() if t is not None else None


def gemm(A, B, *, M, N, K, lda, ldb, a_mn=False, b_mn=False, out=None, ldc=None, out_dtype=None, bias=None,
         residual=None, ldr=None, aux=None, ld_aux=None, act=ACT_NONE, alpha=1.0, nb=(1, 1), a_sb=(0, 0),
         b_sb=(0, 0), c_sb=(0, 0), r_sb=(0, 0), split_k=1, workspace=None, block_n=0, cta_group=0,
         tma_store=0, colsum_out=None, colsum_ws=None, ln=None):
    """C = epi(alpha * A @ B) on the tcgen05 GEMM (see mpx_gemm_desc)."""
    require_cuda([A, B], "gemm")
    if A.dtype != B.dtype or A.dtype not in (torch.float16, torch.bfloat16):
        raise TypeError("gemm operands must share f16/bf16")
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or A.dtype, device=A.device)
        ldc = N
    if split_k > 1 and workspace is None:
        workspace = torch.empty(split_k * M * N, dtype=torch.float32, device=A.device)
    d = _nat.GemmDescC()
    d.ab_dtype = _CODE[A.dtype]
    d.M, d.N, d.K = M, N, K
    d.A, d.lda, d.a_sb1, d.a_sb2, d.a_mn_major = A.data_ptr(), lda, a_sb[0], a_sb[1], int(a_mn)
    d.B, d.ldb, d.b_sb1, d.b_sb2, d.b_mn_major = B.data_ptr(), ldb, b_sb[0], b_sb[1], int(b_mn)
    d.nb1, d.nb2 = nb
    d.C, d.ldc, d.c_sb1, d.c_sb2, d.c_dtype = out.data_ptr(), ldc if ldc is not None else N, c_sb[0], c_sb[1], \
        _CODE[out.dtype]
    d.bias = _ptr(bias)
    d.residual = _ptr(residual)
    d.ldr = ldr if ldr is not None else N
    d.r_sb1, d.r_sb2 = r_sb
    d.aux = _ptr(aux)
    d.ld_aux = ld_aux if ld_aux is not None else N
    d.alpha = alpha
    d.act = act
    d.block_n = block_n
    d.split_k = split_k
    d.workspace = _ptr(workspace)
    d.cta_group = cta_group
    d.tma_store = tma_store
    if colsum_out is not None:
        if colsum_ws is None:
            colsum_ws = torch.empty(colsum_ws_numel(M, N), dtype=torch.float32, device=A.device)
        assert colsum_ws.dtype == torch.float32 and colsum_ws.numel() >= colsum_ws_numel(M, N)
        d.colsum_ws, d.colsum_out = colsum_ws.data_ptr(), colsum_out.data_ptr()
    if ln is not None:  # (gain, bias, out, mean, rstd, eps): LayerNorm of the stored rows, fused
        g_, b_, o_, mu_, rs_, eps_ = ln
        d.ln_gain, d.ln_bias, d.ln_out = g_.data_ptr(), b_.data_ptr(), o_.data_ptr()
        d.ld_ln = o_.stride(0)
        d.ln_mean, d.ln_rstd, d.ln_eps = mu_.data_ptr(), rs_.data_ptr(), eps_
    _nat.check(_nat.load().mpx_gemm(ctypes.byref(d), stream_handle(A.device)), "mpx_gemm")
    return out


def colsum_ws_numel(M: int, N: int) -> int:
    """f32 workspace of the GEMM's fused column sum: one partial row per 32 rows of C."""
    return -(-M // 32) * N


# ---------------------------------------------------------------- linears
def linear_fwd(x, w, bias=None, act=ACT_NONE, aux=None, residual=None, out=None, cta_group=0):
    """y[M,N] = x[M,K] @ w[K,N] (+bias, GELU saving pre-act in aux, +residual)."""
    M, K = x.shape
    N_ = w.shape[1]
    return gemm(x, w, M=M, N=N_, K=K, lda=K, ldb=N_, b_mn=True, bias=bias, act=act, aux=aux, residual=residual,
                out=out, ldc=N_ if out is not None else None, cta_group=cta_group)


def transpose(src, out=None):
    """out[c, r] = src[r, c] for a 2-D f16/bf16 tensor (mpx_transpose)."""
    require_cuda([src], "transpose")
    R, C = src.shape
    if out is None:
        out = torch.empty(C, R, dtype=src.dtype, device=src.device)
    _nat.check(_nat.load().mpx_transpose(_CODE[src.dtype], src.data_ptr(), R, C, src.stride(0), out.data_ptr(),
                                         out.stride(0), stream_handle(src.device)), "mpx_transpose")
    return out


def transpose_batch(srcs, outs):
    """outs[i][c, r] = srcs[i][r, c] for up to 64 2-D f16/bf16 tensors in one launch."""
    require_cuda(list(srcs), "transpose_batch")
    n = len(srcs)
    if n == 0:
        return outs
    P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    _nat.check(_nat.load().mpx_transpose_batch(
        _CODE[srcs[0].dtype], n, (P * n)(*[s.data_ptr() for s in srcs]), (P * n)(*[o.data_ptr() for o in outs]),
        (I * n)(*[s.shape[0] for s in srcs]), (I * n)(*[s.shape[1] for s in srcs]),
        (L * n)(*[s.stride(0) for s in srcs]), (L * n)(*[o.stride(0) for o in outs]),
        stream_handle(srcs[0].device)), "mpx_transpose_batch")
    return outs


def linear_fwd_t(x, wt, bias=None, act=ACT_NONE, aux=None, residual=None, out=None, cta_group=0, ln=None):
    """y[M,N] = x[M,K] @ wt[N,K]^T — the weight held transposed (K-major B,
    faster than linear_fwd's MN-major read of w[K,N]).  ln = (gain, bias,
    out, mean, rstd, eps): also LN(y) over each whole row (N == 768, with a
    residual), in the same kernel."""
    M, K = x.shape
    N_ = wt.shape[0]
    return gemm(x, wt, M=M, N=N_, K=K, lda=K, ldb=K, bias=bias, act=act, aux=aux, residual=residual,
                out=out, ldc=N_ if out is not None else None, cta_group=cta_group, ln=ln)


def linear_dgrad(dy, w, aux=None, out=None, cta_group=0, colsum_out=None, colsum_ws=None, aux_act=ACT_GELU_BWD):
    """dx[M,K] = dy[M,N] @ w[K,N]^T; with aux the GELU backward is applied in
    the epilogue: aux_act ACT_GELU_BWD — aux is the pre-activation, gelu'
    evaluated here; ACT_MUL_AUX — aux is the derivative the forward saved
    (ACT_GELU_D), a plain product.  colsum_out receives sum_m dx[m,:] (the
    producing layer's bias gradient)."""
    M, N_ = dy.shape
    K = w.shape[0]
    return gemm(dy, w, M=M, N=K, K=N_, lda=N_, ldb=N_, aux=aux, ld_aux=K,
                act=aux_act if aux is not None else ACT_NONE, out=out, ldc=K if out is not None else None,
                cta_group=cta_group, colsum_out=colsum_out, colsum_ws=colsum_ws)


_SMS: dict = {}


def _num_sms(device) -> int:
    n = _SMS.get(device)
    if n is None:
        n = _SMS[device] = torch.cuda.get_device_properties(device).multi_processor_count
    return n


def auto_cta_group(M: int, N: int, b_mn: bool) -> int:
    """Mirror of mpx_gemm's automatic choice (csrc/mpx_gemm.cu)."""
    bn = 256 if N >= 256 else -(-N // 16) * 16
    if b_mn:
        bn = -(-bn // 64) * 64
    pair_ok = bn in (128, 256) and (not b_mn or bn % 128 == 0)
    return 2 if pair_ok and M >= 512 else 1


def auto_split_k(M: int, N: int, K: int, cg: int, sms: int, bn: int = 0) -> int:
    """Split-K factor that fills the machine in whole waves (wgrad: M, N are
    the weight dims, K the token count)."""
    bn = bn or (256 if N >= 256 else -(-N // 16) * 16)
    tiles = -(-M // (128 * cg)) * -(-N // bn)
    slots = sms // cg
    kb = -(-K // 64)
    best, best_s = -1.0, 1
    for s in range(1, 17):
        if kb // s < 8:
            break
        units = tiles * s
        util = units / (-(-units // slots) * slots)
        score = util - 0.004 * s
        if score > best:
            best, best_s = score, s
    return best_s


# the wide weight-gradient tiles (mpx_gemm block_n = 512 / 384); MPX_WGRAD_WIDE=0 turns
# them off, =384 / =512 restricts them to one width (A/B runs)
_WGRAD_WIDE = os.environ.get("MPX_WGRAD_WIDE", "1")


def linear_wgrad(x, dy, out=None, split_k=None, cta_group=0, wide=None):
    """dw[K,N] = x[M,K]^T @ dy[M,N] (reduction over the M tokens).  Weight
    shapes with N % 512 (or 384) == 0 and K >= 256 use a wide CTA-pair tile
    (one accumulator, 3/4 (5/6) of the L2 bytes per MAC of the 256 x 256 tile).
    wide: None = auto, False = 256 x 256, True = a wide tile (512 when N allows), 384 / 512 = that width."""
    M, K = x.shape
    N_ = dy.shape[1]
    bn = 0
    if wide in (384, 512) and wide is not True:  # an explicit width
        bn = int(wide)
    elif wide is None or wide:
        for w in (512, 384):
            if N_ % w == 0 and K >= 256 and cta_group in (0, 2) and (wide or _WGRAD_WIDE in ("1", str(w))):
                bn = w
                break
        if wide and not bn:
            bn = 384
    wide = bn > 0
    if split_k is None:
        cg = 2 if wide else (cta_group or auto_cta_group(K, N_, True))
        split_k = auto_split_k(K, N_, M, cg, _num_sms(x.device), bn)
    return gemm(x, dy, M=K, N=N_, K=M, lda=K, ldb=N_, a_mn=True, b_mn=True, out=out,
                ldc=N_ if out is not None else None, split_k=split_k, cta_group=2 if wide else cta_group,
                block_n=bn)


def attention_stats_numel(B: int, N: int, H: int) -> int:
    """f32 elements of the forward's per-row softmax statistics (max, 1/sum)."""
    return B * H * ((N + 127) // 128) * 128 * 2


def attention_psave_bytes(B: int, N: int, H: int) -> int:
    """Bytes of the forward's saved P ([B*H][N][16 ceil(N/16)] half, mpx_attention_psave_bytes)."""
    return B * H * N * (16 * -(-N // 16)) * 2


def attention_fwd(qkv, B: int, N: int, H: int, hd: int, scale: float, out=None, stats=None, p_save=None):
    """Fused softmax(Q K^T * scale) V from qkv [B*N, 3*H*hd] into out [B*N, H*hd];
    `stats` (f32, attention_stats_numel) receives the row statistics, `p_save`
    (uint8, attention_psave_bytes) the probabilities, for the backward."""
    require_cuda([qkv], "attention_fwd")
    D = H * hd
    if out is None:
        out = torch.empty(B * N, D, dtype=qkv.dtype, device=qkv.device)
    if stats is not None:
        assert stats.dtype == torch.float32 and stats.numel() >= attention_stats_numel(B, N, H)
    if p_save is not None:
        assert p_save.dtype == torch.uint8 and p_save.numel() >= attention_psave_bytes(B, N, H)
    _nat.check(_nat.load().mpx_attention_fwd(_CODE[qkv.dtype], qkv.data_ptr(), B, N, H, hd, scale, out.data_ptr(),
                                             out.stride(0), stats.data_ptr() if stats is not None else None,
                                             p_save.data_ptr() if p_save is not None else None,
                                             stream_handle(qkv.device)), "mpx_attention_fwd")
    return out


def attention_bwd(qkv, dO, B: int, N: int, H: int, hd: int, scale: float, dqkv=None, stats=None,
                  colsum_out=None, colsum_ws=None, p_saved=None):
    """Fused attention backward: the whole dqkv [B*N, 3*H*hd] from qkv and dO
    (with the forward's `stats`, P is rebuilt without the statistics passes);
    colsum_out [3*H*hd] receives sum over rows of dqkv (the qkv bias gradient)."""
    require_cuda([qkv, dO], "attention_bwd")
    if dqkv is None:
        dqkv = torch.empty_like(qkv)
    if stats is not None:
        assert stats.dtype == torch.float32 and stats.numel() >= attention_stats_numel(B, N, H)
    if colsum_out is not None and colsum_ws is None:
        colsum_ws = torch.empty(B * 3 * H * hd, dtype=torch.float32, device=qkv.device)
    if colsum_ws is not None:
        assert colsum_ws.dtype == torch.float32 and colsum_ws.numel() >= B * 3 * H * hd
    if p_saved is not None:
        assert p_saved.dtype == torch.uint8 and p_saved.numel() >= attention_psave_bytes(B, N, H)
    _nat.check(_nat.load().mpx_attention_bwd(_CODE[qkv.dtype], qkv.data_ptr(), dO.data_ptr(), B, N, H, hd, scale,
                                             dqkv.data_ptr(), stats.data_ptr() if stats is not None else None,
                                             p_saved.data_ptr() if p_saved is not None else None,
                                             colsum_ws.data_ptr() if colsum_out is not None else None,
                                             colsum_out.data_ptr() if colsum_out is not None else None,
                                             stream_handle(qkv.device)), "mpx_attention_bwd")
    return dqkv
