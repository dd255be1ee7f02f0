"""Fused attention fwd/bwd vs the unfused GEMM+softmax path at ViT-B shape."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402
from paper_2507_03312_b200 import _native as N  # noqa: E402


def t(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def main():
    B, S, H, hd = 256, 197, 12, 64
    D = H * hd
    dt = torch.bfloat16
    qkv = torch.randn(B * S, 3 * D, device="cuda").to(dt)
    dO = torch.randn(B * S, D, device="cuda").to(dt)
    O = torch.empty(B * S, D, device="cuda", dtype=dt)
    dqkv = torch.empty_like(qkv)
    ldS = 200
    Sm = torch.empty(B * H * S, ldS, device="cuda", dtype=dt)
    P = torch.empty_like(Sm)
    lib = N.load()
    st = torch.cuda.current_stream().cuda_stream

    def unfused():
        VK.gemm(qkv, qkv[:, D:], M=S, N=S, K=hd, lda=3 * D, ldb=3 * D, nb=(H, B), a_sb=(hd, S * 3 * D),
                b_sb=(hd, S * 3 * D), out=Sm, ldc=ldS, c_sb=(S * ldS, H * S * ldS), alpha=0.125)
        lib.mpx_softmax_fwd(2, Sm.data_ptr(), P.data_ptr(), B * H * S, S, ldS, st)
        VK.gemm(P, qkv[:, 2 * D:], M=S, N=hd, K=S, lda=ldS, ldb=3 * D, b_mn=True, nb=(H, B),
                a_sb=(S * ldS, H * S * ldS), b_sb=(hd, S * 3 * D), out=O, ldc=D, c_sb=(hd, S * D))

    fl = 4.0 * B * H * S * S * hd
    tf = t(lambda: VK.attention_fwd(qkv, B, S, H, hd, 0.125, out=O))
    tu = t(unfused)
    tb = t(lambda: VK.attention_bwd(qkv, dO, B, S, H, hd, 0.125, dqkv=dqkv))
    print(f"fused fwd {tf:.3f} ms ({fl / tf / 1e9:.0f} TFLOP/s)  unfused fwd {tu:.3f} ms  fused bwd {tb:.3f} ms "
          f"({2.5 * fl / tb / 1e9:.0f} TFLOP/s)")


if __name__ == "__main__":
    main()
