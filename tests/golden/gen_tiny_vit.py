"""Golden trajectory of BASELINE.json configs[0] produced by the REFERENCE:
tiny ViT (depth 2, dim 64, patch 4, 4 heads, MLP 256, 10 classes, mean-pool)
on synthetic 32x32x3 batches of 64, f16 + LossScaling + Adam(lr 1e-3), built
only from mpsim primitives and trained with
mpsim.filter_value_and_grad / optimizer_update.

    python tests/golden/gen_tiny_vit.py <init_scale_log2> <steps> [--hd64] [--gi=N] [--margins]

writes tests/golden/tiny_vit_s<log2>.npz (--hd64: dim 128 / 2 heads, head
dim 64 — the shape the GPU's fused attention kernels take — written to
tiny_vit_hd64_s<log2>.npz): the f32 initial parameters (so
the GPU test starts from the same weights), and per step the loss, the
scale used, grads_finite and a parameter checksum.  Images are
np.random.default_rng((0, 1 + step)) N(0,1) [64,32,32,3], labels U{0..9}
— the GPU test regenerates them with numpy.  Takes ~25 s per step (the
reference's stepwise matmul).
"""
from __future__ import annotations

import math
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

import mpsim  # noqa: E402
from mpsim import F16, F32, I32, LossScaling, adam_init, filter_value_and_grad, force_full_precision, tensor  # noqa: E402
from mpsim import tensors as T  # noqa: E402

IMG, P, C, D, DEPTH, H, MLP, NCLS, B = 32, 4, 3, 64, 2, 4, 256, 10, 64
HD64 = "--hd64" in sys.argv
if HD64:
    D, H = 128, 2
NP = (IMG // P) ** 2
HD = D // H


def param_shapes():
    s = [("patch.w", (P * P * C, D)), ("patch.b", (D,)), ("pos", (NP, D))]
    for i in range(DEPTH):
        b = f"blocks.{i}."
        s += [(b + "ln1.g", (D,)), (b + "ln1.b", (D,)), (b + "qkv.w", (D, 3 * D)), (b + "qkv.b", (3 * D,)),
              (b + "proj.w", (D, D)), (b + "proj.b", (D,)), (b + "ln2.g", (D,)), (b + "ln2.b", (D,)),
              (b + "fc1.w", (D, MLP)), (b + "fc1.b", (MLP,)), (b + "fc2.w", (MLP, D)), (b + "fc2.b", (D,))]
    s += [("ln_f.g", (D,)), ("ln_f.b", (D,)), ("head.w", (D, NCLS)), ("head.b", (NCLS,))]
    return s


def init_params(seed=0):
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in param_shapes():
        leaf = name.rsplit(".", 1)[-1]
        if leaf == "g":
            out[name] = np.ones(shape, np.float32)
        elif leaf == "b":
            out[name] = np.zeros(shape, np.float32)
        else:
            out[name] = (rng.standard_normal(shape) * 0.05).astype(np.float32)
    return out


def batch(step):
    rng = np.random.default_rng((0, 1 + step))
    x = rng.standard_normal((B, IMG, IMG, C)).astype(np.float32)
    y = rng.integers(0, NCLS, B).astype(np.int32)
    return x, y


def select(t, idx, n):
    """t[..., idx, ...] along a leading axis of extent n via an exact
    one-hot matmul (mpsim has no slicing)."""
    sel = np.zeros((n,), np.float32)
    sel[idx] = 1.0
    flat = T.reshape(t, (n, -1))
    return T.matmul(T.reshape(tensor(sel, t.dtype), (1, n)), flat)


def loss_fn(p, a):
    x = a["x"]
    z = T.reshape(x, (B, IMG // P, P, IMG // P, P, C))
    z = T.transpose(z, (0, 1, 3, 2, 4, 5))
    z = T.reshape(z, (B * NP, P * P * C))
    z = T.add(T.matmul(z, p["patch.w"]), p["patch.b"])
    z = T.add(T.reshape(z, (B, NP, D)), p["pos"])
    z = T.reshape(z, (B * NP, D))
    for i in range(DEPTH):
        q = f"blocks.{i}."
        ln1 = force_full_precision(lambda t, g=p[q + "ln1.g"], b=p[q + "ln1.b"]: T.layernorm(t, g, b), z.dtype)
        a1 = ln1(z)
        qkv = T.add(T.matmul(a1, p[q + "qkv.w"]), p[q + "qkv.b"])  # (B*NP, 3D)
        qkv = T.reshape(qkv, (B, NP, 3, H, HD))
        qkv = T.transpose(qkv, (2, 0, 3, 1, 4))  # (3, B, H, NP, HD)
        shp = (B * H, NP, HD)
        qs = T.reshape(select(qkv, 0, 3), shp)
        ks = T.reshape(select(qkv, 1, 3), shp)
        vs = T.reshape(select(qkv, 2, 3), shp)
        scores = T.div(T.matmul(qs, T.transpose(ks, (0, 2, 1))), math.sqrt(HD))
        probs = force_full_precision(T.softmax, scores.dtype)(scores, axis=-1)
        o = T.matmul(probs, vs)  # (B*H, NP, HD)
        o = T.reshape(T.transpose(T.reshape(o, (B, H, NP, HD)), (0, 2, 1, 3)), (B * NP, D))
        z = T.add(T.add(T.matmul(o, p[q + "proj.w"]), p[q + "proj.b"]), z)
        ln2 = force_full_precision(lambda t, g=p[q + "ln2.g"], b=p[q + "ln2.b"]: T.layernorm(t, g, b), z.dtype)
        h = T.gelu(T.add(T.matmul(ln2(z), p[q + "fc1.w"]), p[q + "fc1.b"]))
        z = T.add(T.add(T.matmul(h, p[q + "fc2.w"]), p[q + "fc2.b"]), z)
    lnf = force_full_precision(lambda t: T.layernorm(t, p["ln_f.g"], p["ln_f.b"]), z.dtype)
    zf = T.reshape(lnf(z), (B, NP, D))
    pooled = force_full_precision(lambda t: T.reduce("mean", t, axis=1), zf.dtype)(zf)
    logits = T.add(T.matmul(pooled, p["head.w"]), p["head.b"])
    return force_full_precision(T.cross_entropy, F32)(logits, a["y"])


def checksum(model):
    h = 0
    for name, _ in param_shapes():
        h = (h * 1000003 + int(np.asarray(model[name].payload, np.float32).view(np.uint32).astype(np.uint64).sum())) % (
            2 ** 61 - 1)
    return h


def _opt(name, default):
    for a in sys.argv[1:]:
        if a.startswith(f"--{name}="):
            return int(a.split("=", 1)[1])
    return default


def main():
    """--gi=N: growth interval N (default the reference's 2000): a small one
    makes the scale grow back into the overflow boundary again and again.
    --margins: at every step also evaluate the SAME model/batch at scale/2
    and scale*2 (not applied); a step is marginal when those two flags
    differ, i.e. the overflow boundary lies within a factor 2 of the scale
    used, where f32 vs stepwise-f16 accumulation may legitimately flip it."""
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    log2 = int(args[0]) if len(args) > 0 else 15
    steps = int(args[1]) if len(args) > 1 else 20
    gi = _opt("gi", 2000)
    margins = "--margins" in sys.argv
    p0 = init_params()
    model = {k: tensor(v, F32) for k, v in p0.items()}
    opt = adam_init(model, 1e-3)
    scaling = LossScaling(2.0 ** log2, growth_interval=gi)
    losses, scales, flags, sums, lo_flags, hi_flags = [], [], [], [], [], []
    for step in range(steps):
        t0 = time.time()
        x, y = batch(step)
        args_ = {"x": tensor(x, F32), "y": tensor(y, I32)}
        res = filter_value_and_grad(loss_fn, scaling)(model, args_)
        if margins:
            for mult, col in ((0.5, lo_flags), (2.0, hi_flags)):
                probe = scaling._replace(loss_scale=scaling.loss_scale * mult)
                col.append(bool(filter_value_and_grad(loss_fn, probe)(model, args_).grads_finite))
        model, opt = mpsim.optimizer_update(model, opt, res.grads, res.grads_finite)
        losses.append(float(res.value.item()))
        scales.append(scaling.loss_scale)
        flags.append(bool(res.grads_finite))
        sums.append(checksum(model))
        scaling = res.scaling
        print(f"step {step} loss {losses[-1]:.6f} scale {scales[-1]} finite {flags[-1]}"
              + (f" (s/2 {lo_flags[-1]}, 2s {hi_flags[-1]})" if margins else "") + f" ({time.time() - t0:.1f}s)",
              flush=True)
    tag = f"s{log2}" + (f"_gi{gi}" if gi != 2000 else "")
    out = Path(__file__).resolve().parent / (f"tiny_vit_hd64_{tag}.npz" if HD64 else f"tiny_vit_{tag}.npz")
    extra = {"flags_half_scale": np.asarray(lo_flags), "flags_double_scale": np.asarray(hi_flags)} if margins else {}
    np.savez_compressed(out, losses=np.asarray(losses), scales=np.asarray(scales), flags=np.asarray(flags),
                        checksums=np.asarray(sums, dtype=np.uint64), growth_interval=np.asarray(gi),
                        **extra, **{"init." + k: v for k, v in p0.items()})
    print("wrote", out)


if __name__ == "__main__":
    main()
