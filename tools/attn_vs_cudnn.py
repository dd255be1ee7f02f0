"""Same-box comparison of the fused attention (K6) with the library SDPA
kernels at the ViT-B/16 shape [B=256, H=12, N=197, hd=64] (bf16 and f16):
torch SDPA through cuDNN and through flash (FA2) backends, forward and
forward+backward, CUDA-event timed after warm-up.  Prints one JSON line per
(impl, dtype).

    python tools/attn_vs_cudnn.py [--batch 256]
"""
import argparse
import json
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402


def timed(fn, it=20):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    args = ap.parse_args()
    B, S, H, hd = args.batch, 197, 12, 64
    D = H * hd
    scale = hd ** -0.5
    fl_fwd = 4.0 * B * H * S * S * hd
    for dt in (torch.bfloat16, torch.float16):
        g = torch.Generator(device="cuda").manual_seed(0)
        qkv = torch.randn(B * S, 3 * D, device="cuda", generator=g).to(dt)
        dO = torch.randn(B * S, D, device="cuda", generator=g).to(dt)
        O = torch.empty(B * S, D, device="cuda", dtype=dt)
        dqkv = torch.empty_like(qkv)
        psave = torch.empty(VK.attention_psave_bytes(B, S, H), dtype=torch.uint8, device="cuda")
        # ours, exactly as the ViT engine calls it (P saved by the forward, reloaded by the backward)
        tf = timed(lambda: VK.attention_fwd(qkv, B, S, H, hd, scale, out=O, p_save=psave))
        tb = timed(lambda: VK.attention_bwd(qkv, dO, B, S, H, hd, scale, dqkv=dqkv, p_saved=psave))
        print(json.dumps({"impl": "mpx fused (K6)", "dtype": str(dt), "fwd_ms": round(tf, 4),
                          "bwd_ms": round(tb, 4), "fwd_bwd_ms": round(tf + tb, 4),
                          "fwd_tflops": round(fl_fwd / tf / 1e9, 1)}), flush=True)
        # library SDPA on [B, H, S, hd] views of the same qkv
        q, k, v = qkv.view(B, S, 3, H, hd).permute(2, 0, 3, 1, 4).unbind(0)
        from torch.nn.attention import SDPBackend, sdpa_kernel
        for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                         ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
            try:
                with sdpa_kernel([be]):
                    qc, kc, vc = (t.detach().requires_grad_() for t in (q, k, v))
                    dOv = dO.view(B, S, H, hd).transpose(1, 2)

                    def fwd():
                        with torch.no_grad():
                            return F.scaled_dot_product_attention(qc, kc, vc, scale=scale)

                    def fwd_bwd():
                        out = F.scaled_dot_product_attention(qc, kc, vc, scale=scale)
                        torch.autograd.grad(out, (qc, kc, vc), dOv)

                    t1 = timed(fwd)
                    t2 = timed(fwd_bwd)
                print(json.dumps({"impl": f"torch SDPA {name}", "dtype": str(dt), "fwd_ms": round(t1, 4),
                                  "bwd_ms": round(t2 - t1, 4), "fwd_bwd_ms": round(t2, 4),
                                  "fwd_tflops": round(fl_fwd / t1 / 1e9, 1)}), flush=True)
            except Exception as e:  # noqa: BLE001 - a backend may not support the shape
                print(json.dumps({"impl": f"torch SDPA {name}", "dtype": str(dt), "error": repr(e)[:200]}),
                      flush=True)


if __name__ == "__main__":
    main()
