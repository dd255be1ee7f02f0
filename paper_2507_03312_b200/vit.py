"""ViT forward/backward on the sm_100a kernels (configs 1, 3-5 of BASELINE.json).

The reference has no ViT; this is the model its primitives
compose, with MPX's precision rules:

    patchify -> x @ W_patch + b + pos (+cls)                       half
    per block:  LN1 (f32 island) -> qkv -> S = QK^T/sqrt(hd) -> softmax (f32
                island) -> P V -> proj + residual -> LN2 (island) -> fc1+GELU
                -> fc2 + residual                                  half, f32 accumulate
    head:       LN_f (island) on the cls token (or mean-pool island) -> head
                -> cross-entropy (f32 island, bench.py:185-198)

Every contraction is the tcgen05 GEMM (K5) with the elementwise work fused
into its epilogue (bias, GELU saving the pre-activation, GELU' in the fc2
dgrad, residual adds); attention contractions run straight out of the
[B, N, 3, H, hd] qkv layout through 4-D TMA maps.  Activations are kept for
the backward in preallocated buffers sized for (config, batch); gradients
are written into caller-provided tensors (the flat half grad arena of
step.FusedMPStep), so a training step allocates nothing.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

from . import _native as _nat
from . import vit_kernels as VK
from .dtypes import F16, as_dtype
from . import kernels as K
from .kernels import stream_handle
from .vit_config import ViTConfig

LN_EPS = 1e-5  # tensors.py:449 _LAYERNORM_EPS


def _r8(n: int) -> int:
    return -(-n // 8) * 8


class ViTEngine:
    """Buffers + kernel sequence for one (config, batch, half dtype)."""

    def __init__(self, cfg: ViTConfig, batch: int, half=F16, device=None):
        self.cfg = cfg
        self.B = batch
        self.half = as_dtype(half)
        self.dt = self.half.torch
        self.code = self.half.code
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        c = cfg
        B, S, D, H = batch, c.seq, c.dim, c.heads
        self.S, self.D, self.H, self.hd = S, D, H, D // H
        self.np = c.n_patches
        self.Kp = c.patch * c.patch * c.chans
        self.ldS = _r8(S)
        self.ldl = _r8(c.classes)
        self.M = B * S
        e = lambda *shape, dt=self.dt: torch.empty(*shape, dtype=dt, device=self.dev)  # noqa: E731
        M = self.M
        self.patches = e(B * self.np, self.Kp)
        self.x = [e(M, D) for _ in range(c.depth + 1)]  # residual stream at each block input (+ final)
        self.a = [e(M, D) for _ in range(c.depth)]  # LN1 out
        self.qkv = [e(M, 3 * D) for _ in range(c.depth)]
        # fused attention (K6, mpx_attn.cu) keeps scores/probabilities on chip
        # (hd == 64, N <= 256); MPX_FUSED_ATTENTION=0 selects the unfused path
        # (tcgen05 GEMM + f32 softmax island + GEMM, S/P round-tripping HBM)
        self.fused_attn = (self.hd == 64 and S <= 256 and os.environ.get("MPX_FUSED_ATTENTION", "1") == "1")
        if not self.fused_attn:
            self.Sm = [e(B * H * S, self.ldS) for _ in range(c.depth)]  # scaled scores
            self.P = [e(B * H * S, self.ldS) for _ in range(c.depth)]
        elif os.environ.get("MPX_ATTN_PSAVE", "1") == "1":
            # the forward's probabilities, saved for the backward (as the reference's autodiff saves
            # the softmax output): the backward reloads P instead of recomputing scores and softmax
            self.attn_p = [torch.empty(VK.attention_psave_bytes(B, S, H), dtype=torch.uint8, device=self.dev)
                           for _ in range(c.depth)]
            self.attn_stats = None
        else:  # MPX_ATTN_PSAVE=0: only the row statistics; the backward recomputes P on chip
            self.attn_p = [None] * c.depth
            self.attn_stats = [torch.empty(VK.attention_stats_numel(B, S, H), dtype=torch.float32, device=self.dev)
                               for _ in range(c.depth)]
        self.O = [e(M, D) for _ in range(c.depth)]
        # the blocks' weights transposed (K-major GEMM operands), refreshed every forward
        self._wt = [{"qkv": e(3 * D, D), "proj": e(D, D), "fc1": e(c.mlp, D), "fc2": e(D, c.mlp)}
                    for _ in range(c.depth)]
        self.xm = [e(M, D) for _ in range(c.depth)]  # after attention residual
        self.bn = [e(M, D) for _ in range(c.depth)]  # LN2 out
        # gelu'(fc1 pre-activation) rounded to the half format — what _bw_gelu
        # multiplies the cotangent by (autodiff.py:173-185) — saved by the fc1
        # epilogue from the tanh its GELU evaluates, so the fc2 dgrad epilogue
        # is a plain product (no second tanh pass over M x mlp elements)
        self.pre = [e(M, c.mlp) for _ in range(c.depth)]
        # MPX_GELU_SAVE_D=0: save the pre-activation instead and evaluate gelu' in the dgrad epilogue
        self.gelu_d = os.environ.get("MPX_GELU_SAVE_D", "1") == "1"
        # LayerNorm folded into the residual GEMMs' epilogue (mpx_gemm_desc.ln_*, N = 768 only: a
        # cluster of 3 CTA pairs per row block): proj -> LN2, fc2 -> the next block's LN1.
        # MPX_LN_FOLD=0 runs the standalone LayerNorm kernel after each residual GEMM instead.
        self.ln_fold = D == 768 and os.environ.get("MPX_LN_FOLD", "1") == "1"
        self.h = [e(M, c.mlp) for _ in range(c.depth)]  # GELU out
        f = lambda n: torch.empty(n, dtype=torch.float32, device=self.dev)  # noqa: E731
        self.mu1 = [f(M) for _ in range(c.depth)]
        self.rs1 = [f(M) for _ in range(c.depth)]
        self.mu2 = [f(M) for _ in range(c.depth)]
        self.rs2 = [f(M) for _ in range(c.depth)]
        nf = B if c.pool == "cls" else M
        self.fin = e(nf, D)  # LN_f out (cls rows, or all rows for mean-pool)
        self.muf, self.rsf = f(nf), f(nf)
        self.pooled = e(B, D)
        self.logits = e(B, self.ldl)
        self.nll = f(B)
        self.loss = torch.zeros((), dtype=torch.float32, device=self.dev)
        # backward scratch (reused across blocks)
        self.dX = e(M, D)
        self.dXm = e(M, D)
        # cls pooling: the top block's input gradient is nonzero only on the cls rows,
        # which the LN_f backward rewrites every step — zeroed once here, not per step
        self.dX_top = e(M, D).zero_() if c.pool == "cls" else None
        self.dO = e(M, D)
        self.dqkv = e(M, 3 * D)
        self.dP = e(B * H * S, self.ldS) if not self.fused_attn else None
        self.dpre = e(M, c.mlp)
        self.dA = e(M, D)
        self.dlogits = e(B, self.ldl)
        self.dfin = e(nf, D)
        self.dpool = e(B, D)
        self._dloss32 = torch.zeros((), dtype=torch.float32, device=self.dev)
        self._one32 = torch.ones((), dtype=torch.float32, device=self.dev)
        self.dpatch = e(B * self.np, D)
        self.hw_pad = e(D, self.ldl) if c.classes % 8 else None  # head weight with 16-byte rows
        if self.hw_pad is not None:
            self.hw_pad.zero_()
        self.dhw_pad = e(D, self.ldl) if c.classes % 8 else None
        self.ws_floats = max(8 * 1024 * 1024, 2 * (D * 3 * D), 3 * c.mlp * D, VK.colsum_ws_numel(self.M, c.mlp))
        self.ws = f(self.ws_floats)
        self.lib = _nat.load()
        # forwards run so far: the activations in the buffers belong to the
        # latest one (an autograd graph checks it still owns them)
        self.generation = 0

    # ------------------------------------------------------------------
    def activation_bytes(self) -> int:
        """Bytes of the activations the forward keeps for the backward (the
        reference tape's activation_bytes, autodiff.py:43) — in their physical
        formats: half activations 2 B, f32 LayerNorm statistics 4 B."""
        kept = [self.patches, self.fin, self.muf, self.rsf, self.pooled, self.logits]
        for name in ("x", "a", "qkv", "O", "xm", "bn", "pre", "h", "mu1", "rs1", "mu2", "rs2"):
            kept += list(getattr(self, name))
        kept += list(getattr(self, "attn_p", []) or []) + list(getattr(self, "P", []) or [])
        return int(sum(t.numel() * t.element_size() for t in kept))

    def _st(self):
        return stream_handle(self.dev)

    def _ck(self, rc, what):
        _nat.check(rc, what)

    def _ln_fwd(self, x, ldx, g, b, y, ldy, mu, rs, rows):
        self._ck(self.lib.mpx_layernorm_fwd(self.code, x.data_ptr(), ldx, g.data_ptr(), b.data_ptr(), y.data_ptr(),
                                            ldy, mu.data_ptr(), rs.data_ptr(), rows, self.D, LN_EPS, self._st()),
                 "layernorm_fwd")

    def _ln_bwd(self, x, ldx, g, mu, rs, dy, lddy, dres, dx, lddx, dg, db, rows):
        self._ck(self.lib.mpx_layernorm_bwd(self.code, x.data_ptr(), ldx, g.data_ptr(), mu.data_ptr(), rs.data_ptr(),
                                            dy.data_ptr(), lddy, dres.data_ptr() if dres is not None else None,
                                            self.D if dres is not None else 0, dx.data_ptr(), lddx, dg.data_ptr(),
                                            db.data_ptr(), self.ws.data_ptr(), rows, self.D, self._st()),
                 "layernorm_bwd")

    def _ln_bwd2(self, x, ldx, g, mu, rs, dy, lddy, dres, dx, lddx, dg, db, dxsum, rows):
        """LN backward + fused column sums; dxsum (or None) = colsum of dx."""
        self._ck(self.lib.mpx_layernorm_bwd2(self.code, x.data_ptr(), ldx, g.data_ptr(), mu.data_ptr(), rs.data_ptr(),
                                             dy.data_ptr(), lddy, dres.data_ptr() if dres is not None else None,
                                             self.D if dres is not None else 0, dx.data_ptr(), lddx, dg.data_ptr(),
                                             db.data_ptr(), dxsum.data_ptr() if dxsum is not None else None,
                                             self.ws.data_ptr(), self.ws_floats, rows, self.D, self._st()),
                 "layernorm_bwd2")

    def _colsum(self, x, ldx, rows, cols, out, sbx=0, batches=1, ld_out=0, alpha=1.0, out_dtype=None):
        self._ck(self.lib.mpx_colsum(self.code, x.data_ptr(), ldx, sbx, rows, cols, batches, self.ws.data_ptr(),
                                     self.ws_floats, out.data_ptr(), ld_out or cols,
                                     out_dtype if out_dtype is not None else self.code, alpha, self._st()), "colsum")

    # ------------------------------------------------------------------
    def forward(self, p: dict, images: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        """p: path -> half tensor; images [B, H, W, C] half; labels [B] int32.
        Returns the mean cross-entropy (f32 0-d device tensor)."""
        c, B, S, D, H, hd = self.cfg, self.B, self.S, self.D, self.H, self.hd
        M, st, lib = self.M, self._st(), self.lib
        cls = c.pool == "cls"
        self._ck(lib.mpx_patchify(self.code, images.data_ptr(), self.patches.data_ptr(), B, c.img, c.img, c.chans,
                                  c.patch, st), "patchify")
        x0 = self.x[0]
        # patch embedding + bias + position embedding, written into the token rows
        VK.gemm(self.patches, p["patch.w"], M=self.np, N=D, K=self.Kp, lda=self.Kp, ldb=D, b_mn=True,
                nb=(1, B), a_sb=(0, self.np * self.Kp), out=x0[1:] if cls else x0, ldc=D, c_sb=(0, S * D),
                bias=p["patch.b"], residual=p["pos"][1:] if cls else p["pos"], ldr=D, r_sb=(0, 0))
        if cls:
            self._ck(lib.mpx_rows_add(self.code, p["cls"].data_ptr(), p["pos"].data_ptr(), x0.data_ptr(), S * D, B, D,
                                      st), "rows_add")
        scale = 1.0 / math.sqrt(hd)
        # every block's four weights transposed into K-major copies in one launch (the
        # GEMM reads a K-major B operand ~6 % faster than the MN-major [K, N] layout)
        names = ("qkv", "proj", "fc1", "fc2")
        for i0 in range(0, c.depth, 16):  # <= 64 matrices per launch
            blocks = range(i0, min(c.depth, i0 + 16))
            VK.transpose_batch([p[f"blocks.{i}.{n}.w"] for i in blocks for n in names],
                               [self._wt[i][n] for i in blocks for n in names])
        for i in range(c.depth):
            q = f"blocks.{i}."
            x, a, qkv = self.x[i], self.a[i], self.qkv[i]
            if i == 0 or not self.ln_fold:  # (folded: block i-1's fc2 epilogue produced LN1(x) already)
                self._ln_fwd(x, D, p[q + "ln1.g"], p[q + "ln1.b"], a, D, self.mu1[i], self.rs1[i], M)
            wt = self._wt[i]
            VK.linear_fwd_t(a, wt["qkv"], bias=p[q + "qkv.b"], out=qkv)
            O = self.O[i]
            if self.fused_attn:
                VK.attention_fwd(qkv, B, S, H, hd, scale, out=O, p_save=self.attn_p[i],
                                 stats=self.attn_stats[i] if self.attn_stats else None)
            else:
                Sm, P_ = self.Sm[i], self.P[i]
                VK.gemm(qkv, qkv[:, D:], M=S, N=S, K=hd, lda=3 * D, ldb=3 * D, nb=(H, B), a_sb=(hd, S * 3 * D),
                        b_sb=(hd, S * 3 * D), out=Sm, ldc=self.ldS, c_sb=(S * self.ldS, H * S * self.ldS),
                        alpha=scale)
                self._ck(lib.mpx_softmax_fwd(self.code, Sm.data_ptr(), P_.data_ptr(), B * H * S, S, self.ldS, st),
                         "softmax_fwd")
                VK.gemm(P_, qkv[:, 2 * D:], M=S, N=hd, K=S, lda=self.ldS, ldb=3 * D, b_mn=True, nb=(H, B),
                        a_sb=(S * self.ldS, H * S * self.ldS), b_sb=(hd, S * 3 * D), out=O, ldc=D, c_sb=(hd, S * D))
            xm = self.xm[i]
            bn = self.bn[i]
            if self.ln_fold:  # xm = O Wp + bp + x and bn = LN2(xm) in one kernel
                VK.linear_fwd_t(O, wt["proj"], bias=p[q + "proj.b"], residual=x, out=xm,
                                ln=(p[q + "ln2.g"], p[q + "ln2.b"], bn, self.mu2[i], self.rs2[i], LN_EPS))
            else:
                VK.linear_fwd_t(O, wt["proj"], bias=p[q + "proj.b"], residual=x, out=xm)
                self._ln_fwd(xm, D, p[q + "ln2.g"], p[q + "ln2.b"], bn, D, self.mu2[i], self.rs2[i], M)
            VK.linear_fwd_t(bn, wt["fc1"], bias=p[q + "fc1.b"], act=VK.ACT_GELU_D if self.gelu_d else VK.ACT_GELU,
                            aux=self.pre[i], out=self.h[i])
            if self.ln_fold and i + 1 < c.depth:  # x_{i+1} and the next block's LN1 in one kernel
                n = f"blocks.{i + 1}."
                VK.linear_fwd_t(self.h[i], wt["fc2"], bias=p[q + "fc2.b"], residual=xm, out=self.x[i + 1],
                                ln=(p[n + "ln1.g"], p[n + "ln1.b"], self.a[i + 1], self.mu1[i + 1], self.rs1[i + 1],
                                    LN_EPS))
            else:
                VK.linear_fwd_t(self.h[i], wt["fc2"], bias=p[q + "fc2.b"], residual=xm, out=self.x[i + 1])
        xl = self.x[c.depth]
        if cls:
            self._ln_fwd(xl, S * D, p["ln_f.g"], p["ln_f.b"], self.fin, D, self.muf, self.rsf, B)
            feat = self.fin
        else:
            self._ln_fwd(xl, D, p["ln_f.g"], p["ln_f.b"], self.fin, D, self.muf, self.rsf, M)
            self._colsum(self.fin, D, S, D, self.pooled, sbx=S * D, batches=B, ld_out=D, alpha=1.0 / S)
            feat = self.pooled
        hw = p["head.w"]
        if self.hw_pad is not None:
            self._ck(lib.mpx_copy_rows(self.code, hw.data_ptr(), c.classes, 0, self.hw_pad.data_ptr(), self.ldl, 0, D,
                                       1, c.classes, st), "copy_rows")
            hw = self.hw_pad
        VK.gemm(feat, hw, M=B, N=c.classes, K=D, lda=D, ldb=self.ldl if self.hw_pad is not None else c.classes,
                b_mn=True, bias=p["head.b"], out=self.logits, ldc=self.ldl)
        self._ck(lib.mpx_cross_entropy_fwd(self.code, self.logits.data_ptr(), self.ldl, labels.data_ptr(), B,
                                           c.classes, self.nll.data_ptr(), self.loss.data_ptr(), st), "ce_fwd")
        self._labels = labels
        self._images = images
        self.generation += 1
        return self.loss

    # ------------------------------------------------------------------
    def backward(self, p: dict, g: dict, dloss_f32: torch.Tensor | None = None, dloss_f64: torch.Tensor | None = None,
                 on_grads_ready=None):
        """Gradients of (dloss * loss) into g (path -> half tensors).  The loss
        cotangent is read on the device: an f32 0-d tensor (autograd) or the
        fp64 loss scale of a DynamicLossScaling state (fused training step).
        on_grads_ready(key) is called (host side, stream order) once the grads
        of 'head', each 'blocks.<i>' and 'embed' have been launched, so a DP
        exchange can start while the rest of the backward runs."""
        ready = on_grads_ready or (lambda key: None)
        c, B, S, D, H, hd = self.cfg, self.B, self.S, self.D, self.H, self.hd
        M, st, lib = self.M, self._st(), self.lib
        cls = c.pool == "cls"
        if dloss_f32 is None:
            if dloss_f64 is None:
                raise ValueError("backward needs the loss cotangent")
            # f32(scale) = 1.0f * f32(*d_scale): K1 with a device multiplier (the
            # weak-scalar rounding of T.mul(loss, s), autodiff.py:131-138)
            dloss_f32 = self._dloss32
            K.cast_into([self._one32], [dloss_f32], d_scale=dloss_f64)
        self._ck(lib.mpx_cross_entropy_bwd(self.code, self.logits.data_ptr(), self.ldl, self._labels.data_ptr(), B,
                                           c.classes, dloss_f32.data_ptr(), self.dlogits.data_ptr(), self.ldl, st),
                 "ce_bwd")
        feat = self.fin if cls else self.pooled
        # head: logits = feat @ Wh + bh
        if self.dhw_pad is not None:
            VK.gemm(feat, self.dlogits, M=D, N=c.classes, K=B, lda=D, ldb=self.ldl, a_mn=True, b_mn=True,
                    out=self.dhw_pad, ldc=self.ldl)
            self._ck(lib.mpx_copy_rows(self.code, self.dhw_pad.data_ptr(), self.ldl, 0, g["head.w"].data_ptr(),
                                       c.classes, 0, D, 1, c.classes, st), "copy_rows")
            hw, ldhw = self.hw_pad, self.ldl
        else:
            VK.linear_wgrad(feat, self.dlogits, out=g["head.w"])
            hw, ldhw = p["head.w"], c.classes
        self._colsum(self.dlogits, self.ldl, B, c.classes, g["head.b"])
        dfeat = self.dfin if cls else self.dpool
        VK.gemm(self.dlogits, hw, M=B, N=D, K=c.classes, lda=self.ldl, ldb=ldhw, out=dfeat, ldc=D)
        dX = self.dX_top if cls else self.dX
        xl = self.x[c.depth]
        top_fc2b = g[f"blocks.{c.depth - 1}.fc2.b"] if c.depth else None
        if cls:
            # only the cls rows carry gradient: colsum over them = colsum(dX) = the top fc2.b grad
            self._ln_bwd2(xl, S * D, p["ln_f.g"], self.muf, self.rsf, dfeat, D, None, dX, S * D, g["ln_f.g"],
                          g["ln_f.b"], top_fc2b, B)
        else:
            self._ck(lib.mpx_bcast_rows(self.code, dfeat.data_ptr(), D, self.dfin.data_ptr(), D, S * D, S, B, D,
                                        1.0 / S, st), "bcast_rows")
            self._ln_bwd2(xl, D, p["ln_f.g"], self.muf, self.rsf, self.dfin, D, None, dX, D, g["ln_f.g"],
                          g["ln_f.b"], top_fc2b, M)
        ready("head")
        scale = 1.0 / math.sqrt(hd)
        for i in reversed(range(c.depth)):
            q = f"blocks.{i}."
            # fc2: x_{i+1} = h @ W2 + b2 + xm
            VK.linear_wgrad(self.h[i], dX, out=g[q + "fc2.w"])  # fc2.b came with the LN backward above
            # dpre = (dX W2^T) * gelu'(pre); its column sum (the fc1.b grad) fused into the epilogue
            VK.linear_dgrad(dX, p[q + "fc2.w"], aux=self.pre[i], out=self.dpre, colsum_out=g[q + "fc1.b"],
                            colsum_ws=self.ws, aux_act=VK.ACT_MUL_AUX if self.gelu_d else VK.ACT_GELU_BWD)
            # fc1: pre = bn @ W1 + b1
            VK.linear_wgrad(self.bn[i], self.dpre, out=g[q + "fc1.w"])
            VK.linear_dgrad(self.dpre, p[q + "fc1.w"], out=self.dA)
            # LN2 (+ residual): dxm = LN2'(dA) + dX; colsum(dxm) = proj.b grad
            self._ln_bwd2(self.xm[i], D, p[q + "ln2.g"], self.mu2[i], self.rs2[i], self.dA, D, dX, self.dXm, D,
                          g[q + "ln2.g"], g[q + "ln2.b"], g[q + "proj.b"], M)
            dXm = self.dXm
            # proj: xm = O @ Wp + bp + x
            VK.linear_wgrad(self.O[i], dXm, out=g[q + "proj.w"])
            VK.linear_dgrad(dXm, p[q + "proj.w"], out=self.dO)
            # attention
            qkv, dqkv = self.qkv[i], self.dqkv
            if self.fused_attn:  # (the qkv.b gradient, colsum(dqkv), comes out of the kernel)
                VK.attention_bwd(qkv, self.dO, B, S, H, hd, scale, dqkv=dqkv, p_saved=self.attn_p[i],
                                 stats=self.attn_stats[i] if self.attn_stats else None,
                                 colsum_out=g[q + "qkv.b"], colsum_ws=self.ws)
            else:
                self._attention_bwd_unfused(i, qkv, dqkv, scale)
                self._colsum(dqkv, 3 * D, M, 3 * D, g[q + "qkv.b"])
            # qkv = a @ Wqkv + bqkv
            VK.linear_wgrad(self.a[i], dqkv, out=g[q + "qkv.w"])
            VK.linear_dgrad(dqkv, p[q + "qkv.w"], out=self.dA)
            # LN1 (+ residual): dX = LN1'(dA) + dXm; colsum(dX) = fc2.b grad of the block below
            self._ln_bwd2(self.x[i], D, p[q + "ln1.g"], self.mu1[i], self.rs1[i], self.dA, D, dXm, self.dX, D,
                          g[q + "ln1.g"], g[q + "ln1.b"], g[f"blocks.{i - 1}.fc2.b"] if i > 0 else None, M)
            dX = self.dX
            ready(f"blocks.{i}")
        # embedding: tokens = patches @ Wp + bp + pos (+ cls row)
        self._colsum(dX, S * D, B, S * D, g["pos"])  # sum over the batch
        if cls:
            self._colsum(dX, S * D, B, D, g["cls"])
            self._ck(lib.mpx_copy_rows(self.code, dX[1:].data_ptr(), D, S * D, self.dpatch.data_ptr(), D,
                                       self.np * D, self.np, B, D, st), "copy_rows")
            dpatch = self.dpatch
        else:
            dpatch = dX
        self._colsum(dpatch, D, B * self.np, D, g["patch.b"])
        VK.linear_wgrad(self.patches, dpatch, out=g["patch.w"])
        ready("embed")


    def _attention_bwd_unfused(self, i, qkv, dqkv, scale):
        B, S, D, H, hd, st, lib = self.B, self.S, self.D, self.H, self.hd, self._st(), self.lib
        P_, Sm = self.P[i], self.Sm[i]
        # dV[b,h] = P^T dO
        VK.gemm(P_, self.dO, M=S, N=hd, K=S, lda=self.ldS, ldb=D, a_mn=True, b_mn=True, nb=(H, B),
                a_sb=(S * self.ldS, H * S * self.ldS), b_sb=(hd, S * D), out=dqkv[:, 2 * D:], ldc=3 * D,
                c_sb=(hd, S * 3 * D))
        # dP = dO V^T
        VK.gemm(self.dO, qkv[:, 2 * D:], M=S, N=S, K=hd, lda=D, ldb=3 * D, nb=(H, B), a_sb=(hd, S * D),
                b_sb=(hd, S * 3 * D), out=self.dP, ldc=self.ldS, c_sb=(S * self.ldS, H * S * self.ldS))
        # dS = softmax'(dP) (in place), then the 1/sqrt(hd) of the score scaling folds into alpha
        self._ck(lib.mpx_softmax_bwd(self.code, Sm.data_ptr(), self.dP.data_ptr(), self.dP.data_ptr(), B * H * S,
                                     S, self.ldS, st), "softmax_bwd")
        dS = self.dP
        # dQ = dS K * scale
        VK.gemm(dS, qkv[:, D:], M=S, N=hd, K=S, lda=self.ldS, ldb=3 * D, b_mn=True, nb=(H, B),
                a_sb=(S * self.ldS, H * S * self.ldS), b_sb=(hd, S * 3 * D), out=dqkv, ldc=3 * D,
                c_sb=(hd, S * 3 * D), alpha=scale)
        # dK = dS^T Q * scale
        VK.gemm(dS, qkv, M=S, N=hd, K=S, lda=self.ldS, ldb=3 * D, a_mn=True, b_mn=True, nb=(H, B),
                a_sb=(S * self.ldS, H * S * self.ldS), b_sb=(hd, S * 3 * D), out=dqkv[:, D:], ldc=3 * D,
                c_sb=(hd, S * 3 * D), alpha=scale)


# ---------------------------------------------------------------------------
# drop-in: a loss function usable with filter_value_and_grad
# ---------------------------------------------------------------------------
_ENGINES: dict = {}


def engine_for(cfg: ViTConfig, batch: int, half, device) -> ViTEngine:
    key = (cfg, batch, as_dtype(half), str(device))
    eng = _ENGINES.get(key)
    if eng is None:
        eng = ViTEngine(cfg, batch, half, device)
        _ENGINES[key] = eng
    return eng


class _ViTLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, engine, paths, images, labels, *leaves):
        p = dict(zip(paths, leaves))
        loss = engine.forward(p, images, labels).clone()
        ctx.engine, ctx.paths, ctx.generation = engine, paths, engine.generation
        ctx.save_for_backward(*leaves)
        return loss

    @staticmethod
    def backward(ctx, dloss):
        if ctx.engine.generation != ctx.generation:
            # the engine keeps ONE set of activation buffers per (config, batch,
            # dtype): a later forward has overwritten this graph's activations
            raise RuntimeError(
                "vit_loss: another forward of the same ViT engine ran between this loss's forward and its "
                "backward (its activations were overwritten); call backward before the next forward, or "
                "accumulate gradients over separate transform calls")
        leaves = ctx.saved_tensors
        p = dict(zip(ctx.paths, leaves))
        g = {k: torch.empty_like(v) for k, v in p.items()}
        ctx.engine.backward(p, g, dloss_f32=dloss.float().contiguous())
        return (None, None, None, None) + tuple(g[k] for k in ctx.paths)


def vit_loss(cfg: ViTConfig):
    """f(params, batch) -> mean cross-entropy (f32), differentiable w.r.t. the
    float leaves of `params` (path -> tensor, the shapes of cfg.param_shapes())
    — the function filter_value_and_grad transforms.  batch = {"x": images
    [B, H, W, C], "y": int32 labels [B]}; params and images arrive already
    cast to the half dtype by the transform (precision.py:209-210)."""
    paths = [n for n, _ in cfg.param_shapes()]

    def f(params, batch):
        x, y = batch["x"], batch["y"]
        leaves = [params[k] for k in paths]
        half = leaves[0].dtype
        if x.dtype != half:
            raise TypeError("images must be cast to the parameters' half dtype")
        eng = engine_for(cfg, x.shape[0], half, x.device)
        return _ViTLoss.apply(eng, paths, x.contiguous(), y.to(torch.int32).contiguous(), *leaves)

    return f


def init_params(cfg: ViTConfig, device, seed: int = 0, std: float = 0.02) -> dict:
    """Synthetic f32 init (random weights of the architecture; no checkpoints
    offline): N(0, std^2) matrices, ones/zeros LayerNorms, zero biases."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = {}
    for name, shape in cfg.param_shapes():
        leaf = name.rsplit(".", 1)[-1]
        if leaf == "g":
            out[name] = torch.ones(shape, device=device)
        elif leaf == "b":
            out[name] = torch.zeros(shape, device=device)
        else:
            out[name] = torch.randn(shape, generator=g, device=device) * std
    return out
