"""The tiny ViT of BASELINE.json configs[0] written ONLY against the
reference's tensor-layer API (mpsim has no conv,
concat or slice), so the very same source runs on the reference (mpsim) and
on the B200 drop-in layer (paper_2507_03312_b200.tensors):

    loss_fn = make_loss_fn(api)     # api: T, tensor, F32, force_full_precision

tests/golden/gen_tiny_vit.py trains it with mpsim to make the golden
trajectories; tests/test_tiny_vit_parity_gpu.py trains the same source with
`import paper_2507_03312_b200 as mpx` and compares."""
from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

IMG, P, C, NCLS, B, DEPTH, MLP = 32, 4, 3, 10, 64, 2, 256
NP = (IMG // P) ** 2


def param_shapes(D=64):
    s = [("patch.w", (P * P * C, D)), ("patch.b", (D,)), ("pos", (NP, D))]
    for i in range(DEPTH):
        b = f"blocks.{i}."
        s += [(b + "ln1.g", (D,)), (b + "ln1.b", (D,)), (b + "qkv.w", (D, 3 * D)), (b + "qkv.b", (3 * D,)),
              (b + "proj.w", (D, D)), (b + "proj.b", (D,)), (b + "ln2.g", (D,)), (b + "ln2.b", (D,)),
              (b + "fc1.w", (D, MLP)), (b + "fc1.b", (MLP,)), (b + "fc2.w", (MLP, D)), (b + "fc2.b", (D,))]
    s += [("ln_f.g", (D,)), ("ln_f.b", (D,)), ("head.w", (D, NCLS)), ("head.b", (NCLS,))]
    return s


def init_params(seed=0, D=64):
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in param_shapes(D):
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


def make_loss_fn(api: SimpleNamespace, D=64, H=4):
    """api.T (the tensor-op namespace), api.tensor, api.F32, api.force_full_precision."""
    T, tensor, F32, ffp = api.T, api.tensor, api.F32, api.force_full_precision
    HD = D // H

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
            ln1 = ffp(lambda t, g=p[q + "ln1.g"], b=p[q + "ln1.b"]: T.layernorm(t, g, b), z.dtype)
            a1 = ln1(z)
            qkv = T.add(T.matmul(a1, p[q + "qkv.w"]), p[q + "qkv.b"])  # (B*NP, 3D)
            qkv = T.reshape(qkv, (B, NP, 3, H, HD))
            qkv = T.transpose(qkv, (2, 0, 3, 1, 4))  # (3, B, H, NP, HD)
            shp = (B * H, NP, HD)
            qs = T.reshape(select(qkv, 0, 3), shp)
            ks = T.reshape(select(qkv, 1, 3), shp)
            vs = T.reshape(select(qkv, 2, 3), shp)
            scores = T.div(T.matmul(qs, T.transpose(ks, (0, 2, 1))), math.sqrt(HD))
            probs = ffp(T.softmax, scores.dtype)(scores, axis=-1)
            o = T.matmul(probs, vs)  # (B*H, NP, HD)
            o = T.reshape(T.transpose(T.reshape(o, (B, H, NP, HD)), (0, 2, 1, 3)), (B * NP, D))
            z = T.add(T.add(T.matmul(o, p[q + "proj.w"]), p[q + "proj.b"]), z)
            ln2 = ffp(lambda t, g=p[q + "ln2.g"], b=p[q + "ln2.b"]: T.layernorm(t, g, b), z.dtype)
            h = T.gelu(T.add(T.matmul(ln2(z), p[q + "fc1.w"]), p[q + "fc1.b"]))
            z = T.add(T.add(T.matmul(h, p[q + "fc2.w"]), p[q + "fc2.b"]), z)
        lnf = ffp(lambda t: T.layernorm(t, p["ln_f.g"], p["ln_f.b"]), z.dtype)
        zf = T.reshape(lnf(z), (B, NP, D))
        pooled = ffp(lambda t: T.reduce("mean", t, axis=1), zf.dtype)(zf)
        logits = T.add(T.matmul(pooled, p["head.w"]), p["head.b"])
        return ffp(T.cross_entropy, F32)(logits, a["y"])

    return loss_fn
