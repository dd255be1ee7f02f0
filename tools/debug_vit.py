"""Stage-by-stage check of ViTEngine.forward: each stage recomputed in fp32
torch from the engine's own previous-stage buffers, max relative error printed."""
import math
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_03312_b200 as mpx  # noqa: E402
from paper_2507_03312_b200.vit import ViTEngine, init_params  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_TINY, ViTConfig  # noqa: E402


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / (b.abs().max() + 1e-12)).item(), torch.isnan(a).any().item()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    cfg = VIT_TINY if name == "tiny" else ViTConfig(img=32, patch=4, dim=128, depth=2, heads=2, mlp=256,
                                                     classes=16, pool="cls")
    half = torch.float16
    dev = torch.device("cuda")
    B = 4
    p = {k: v.to(half) for k, v in init_params(cfg, dev, seed=3, std=0.05).items()}
    images = torch.randn(B, cfg.img, cfg.img, cfg.chans, device=dev).to(half)
    labels = torch.randint(0, cfg.classes, (B,), device=dev).to(torch.int32)
    e = ViTEngine(cfg, B, mpx.F16, dev)
    loss = e.forward(p, images, labels)
    torch.cuda.synchronize()
    P_, C = cfg.patch, cfg.chans
    nh = cfg.img // P_
    D, H, S = cfg.dim, cfg.heads, e.S
    hd = D // H
    x = images.float().reshape(B, nh, P_, nh, P_, C).permute(0, 1, 3, 2, 4, 5).reshape(B * nh * nh, P_ * P_ * C)
    print("patches", rel(e.patches, x))
    z = (e.patches.float() @ p["patch.w"].float() + p["patch.b"].float()).reshape(B, nh * nh, D)
    if cfg.pool == "cls":
        z = torch.cat([p["cls"].float().expand(B, 1, D), z], 1)
    z = z + p["pos"].float()
    print("x0", rel(e.x[0].reshape(B, S, D), z))
    for i in range(cfg.depth):
        q = f"blocks.{i}."
        xi = e.x[i].float()
        print(i, "ln1", rel(e.a[i], F.layer_norm(xi, (D,), p[q + "ln1.g"].float(), p[q + "ln1.b"].float(), 1e-5)))
        print(i, "qkv", rel(e.qkv[i], e.a[i].float() @ p[q + "qkv.w"].float() + p[q + "qkv.b"].float()))
        qkv = e.qkv[i].float().reshape(B, S, 3, H, hd)
        Q, K, V = qkv[:, :, 0].transpose(1, 2), qkv[:, :, 1].transpose(1, 2), qkv[:, :, 2].transpose(1, 2)
        Sm = e.Sm[i].reshape(B, H, S, e.ldS)[..., :S]
        print(i, "scores", rel(Sm, Q @ K.transpose(-1, -2) / math.sqrt(hd)))
        Pm = e.P[i].reshape(B, H, S, e.ldS)
        print(i, "probs", rel(Pm[..., :S], torch.softmax(Sm.float(), -1)), "pad", Pm[..., S:].abs().max().item()
              if e.ldS > S else 0)
        o = (Pm[..., :S].float() @ V).transpose(1, 2).reshape(B * S, D)
        print(i, "O", rel(e.O[i], o))
        print(i, "xm", rel(e.xm[i], e.O[i].float() @ p[q + "proj.w"].float() + p[q + "proj.b"].float() + xi))
        print(i, "ln2", rel(e.bn[i], F.layer_norm(e.xm[i].float(), (D,), p[q + "ln2.g"].float(),
                                                   p[q + "ln2.b"].float(), 1e-5)))
        pre = e.bn[i].float() @ p[q + "fc1.w"].float() + p[q + "fc1.b"].float()
        print(i, "pre", rel(e.pre[i], pre), "h", rel(e.h[i], F.gelu(e.pre[i].float(), approximate="tanh")))
        print(i, "x+1", rel(e.x[i + 1], e.h[i].float() @ p[q + "fc2.w"].float() + p[q + "fc2.b"].float()
                            + e.xm[i].float()))
    xl = e.x[cfg.depth].float().reshape(B, S, D)
    if cfg.pool == "cls":
        fin = F.layer_norm(xl[:, 0], (D,), p["ln_f.g"].float(), p["ln_f.b"].float(), 1e-5)
        print("fin", rel(e.fin, fin))
        feat = e.fin
    else:
        fin = F.layer_norm(xl, (D,), p["ln_f.g"].float(), p["ln_f.b"].float(), 1e-5).reshape(B * S, D)
        print("fin", rel(e.fin, fin))
        print("pooled", rel(e.pooled, e.fin.float().reshape(B, S, D).mean(1)))
        feat = e.pooled
    lg = feat.float() @ p["head.w"].float() + p["head.b"].float()
    print("logits", rel(e.logits[:, :cfg.classes], lg))
    print("loss", loss.item(), F.cross_entropy(e.logits[:, :cfg.classes].float(), labels.long()).item())


if __name__ == "__main__":
    main()
