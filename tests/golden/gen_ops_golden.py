"""Generate tests/golden/ops_golden.npz by running the REFERENCE itself: the
mpsim tensor operators (tensors.py:220-555) with their backward rules
(autodiff.py:94-290) on seeded inputs, and the reference's own training
harness (bench.fit, bench.py:255-295) on its single-block attention model in
f32, f16 and bf16.

Run in the build container (where /root/reference exists):
    python tests/golden/gen_ops_golden.py
tests/test_tensor_ops_gpu.py compares the device operators
(paper_2507_03312_b200.tensors) against these fixtures.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from mpsim import BF16, F16, F32, I32, tensor, value_and_grad  # noqa: E402
from mpsim import bench as RB  # noqa: E402
from mpsim import tensors as T  # noqa: E402

OUT = Path(__file__).resolve().parent / "ops_golden.npz"
FMT = {"f32": F32, "f16": F16, "bf16": BF16}


def f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def main():
    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(11)

    def rnd(*shape, scale=1.0, pos=False):
        x = rng.standard_normal(shape).astype(np.float32) * scale
        return np.abs(x) + 0.1 if pos else x

    # -- 1. forward ops and their input gradients under loss = sum(op(...) * w)
    cases = []
    for fmt in ("f32", "f16", "bf16"):
        cases += [
            (f"add_bcast_{fmt}", "add", [rnd(4, 5), rnd(5)], [fmt, fmt]),
            (f"sub_{fmt}", "sub", [rnd(3, 7), rnd(3, 7)], [fmt, fmt]),
            (f"mul_bcast_{fmt}", "mul", [rnd(2, 3, 4), rnd(3, 1)], [fmt, fmt]),
            (f"div_{fmt}", "div", [rnd(6, 5), rnd(6, 5, pos=True)], [fmt, fmt]),
            (f"neg_{fmt}", "neg", [rnd(9)], [fmt]),
            (f"exp_{fmt}", "exp", [rnd(5, 6)], [fmt]),
            (f"log_{fmt}", "log", [rnd(5, 6, pos=True)], [fmt]),
            (f"sqrt_{fmt}", "sqrt", [rnd(5, 6, pos=True)], [fmt]),
            (f"relu_{fmt}", "relu", [rnd(5, 6)], [fmt]),
            (f"gelu_{fmt}", "gelu", [rnd(5, 6, scale=2.0)], [fmt]),
            (f"sum_ax0_{fmt}", "sum0", [rnd(7, 5)], [fmt]),
            (f"sum_all_{fmt}", "sumall", [rnd(3, 4, 5)], [fmt]),
            (f"mean_ax1_{fmt}", "mean1", [rnd(4, 9)], [fmt]),
            (f"max_ax1_{fmt}", "max1", [np.round(rnd(4, 9) * 2) / 2], [fmt]),
            (f"softmax_last_{fmt}", "softmax-1", [rnd(4, 11, scale=3.0)], [fmt]),
            (f"softmax_ax0_{fmt}", "softmax0", [rnd(6, 3, scale=3.0)], [fmt]),
            (f"layernorm_{fmt}", "layernorm", [rnd(5, 16, scale=2.0), 1 + 0.1 * rnd(16), 0.1 * rnd(16)],
             [fmt, fmt, fmt]),
            (f"matmul_{fmt}", "matmul", [rnd(7, 13), rnd(13, 5)], [fmt, fmt]),
            (f"matmul_batched_{fmt}", "matmul", [rnd(3, 7, 13), rnd(13, 5)], [fmt, fmt]),
            (f"matmul_vec_{fmt}", "matmul", [rnd(13), rnd(13, 5)], [fmt, fmt]),
            (f"matmul_tc_{fmt}", "matmul", [rnd(2, 24, 32), rnd(2, 32, 16)], [fmt, fmt]),
            (f"xent_{fmt}", "xent", [rnd(6, 10, scale=2.0), rng.integers(0, 10, 6).astype(np.int32)], [fmt, "i32"]),
            (f"scalar_ops_{fmt}", "scalars", [rnd(4, 4, pos=True)], [fmt]),
            (f"transpose_reshape_{fmt}", "perm", [rnd(2, 3, 4), rnd(12, 2)], [fmt, fmt]),
        ]
    cases += [("add_mixed_f16_bf16", "add", [rnd(4, 5), rnd(4, 5)], ["f16", "bf16"]),
              ("mul_mixed_f16_f32", "mul", [rnd(4, 5), rnd(5)], ["f16", "f32"])]

    def fwd(kind, ts):
        if kind in ("add", "sub", "mul", "div"):
            return getattr(T, kind)(ts[0], ts[1])
        if kind in ("neg", "exp", "log", "sqrt", "relu", "gelu"):
            return getattr(T, kind)(ts[0])
        if kind == "sum0":
            return T.reduce("sum", ts[0], axis=0)
        if kind == "sumall":
            return T.reduce("sum", ts[0])
        if kind == "mean1":
            return T.reduce("mean", ts[0], axis=1)
        if kind == "max1":
            return T.reduce("max", ts[0], axis=1)
        if kind.startswith("softmax"):
            return T.softmax(ts[0], axis=int(kind[len("softmax"):]))
        if kind == "layernorm":
            return T.layernorm(ts[0], ts[1], ts[2])
        if kind == "matmul":
            return T.matmul(ts[0], ts[1])
        if kind == "xent":
            return T.cross_entropy(ts[0], ts[1])
        if kind == "scalars":
            x = ts[0]
            return T.add(T.sub(2.0, T.mul(x, 3.0)), T.div(1.5, x))
        if kind == "perm":
            a = T.transpose(ts[0], (2, 0, 1))  # (4, 2, 3)
            return T.matmul(T.reshape(a, (4, 6)), T.reshape(ts[1], (6, 4)))
        raise KeyError(kind)

    names = []
    for name, kind, arrays, fmts in cases:
        names.append(name)
        g[f"{name}__kind"] = np.array(kind)
        g[f"{name}__fmts"] = np.array(",".join(fmts))
        for i, a in enumerate(arrays):
            g[f"{name}__in{i}"] = a
        ts = [tensor(a, FMT[f]) if f != "i32" else tensor(a, I32) for a, f in zip(arrays, fmts)]
        out = fwd(kind, ts)
        g[f"{name}__out"] = f32(out.payload)
        g[f"{name}__out_dtype"] = np.array(out.dtype.value)
        w = tensor(np.random.default_rng(5).standard_normal(out.shape).astype(np.float32), out.dtype)
        g[f"{name}__w"] = f32(w.payload)
        fl = [i for i, f in enumerate(fmts) if f != "i32"]

        def loss(params, args, kind=kind, fl=fl, ts=ts):
            full = list(ts)
            for j, i in enumerate(fl):
                full[i] = params[j]
            o = fwd(kind, full)
            return T.reduce("sum", T.mul(o, args["w"]))

        val, grads = value_and_grad(loss, [ts[i] for i in fl], {"w": w})
        g[f"{name}__loss"] = f32(val.payload)
        for j, i in enumerate(fl):
            g[f"{name}__grad{i}"] = f32(grads[j].payload)
            g[f"{name}__grad{i}_dtype"] = np.array(grads[j].dtype.value)
    g["cases"] = np.array(names)

    # -- 2. the reference's attention classifier trained by its own harness
    for prec in ("f32", "f16", "bf16"):
        cfg = RB.RunConfig(precision=prec, steps=12, batch_size=32, seed=0, model="attention", feature_dim=16,
                           num_heads=4, num_classes=2, lr=1e-2)
        model0 = RB.build_model(cfg)
        for path, leaf in RB._all_tensor_leaves(model0):
            g[f"attn_{prec}__p0__{path}"] = f32(leaf.payload)
        recs, model = RB.fit(cfg)
        g[f"attn_{prec}__loss"] = np.array([r.loss for r in recs], dtype=np.float64)
        g[f"attn_{prec}__scale"] = np.array([r.scale for r in recs], dtype=np.float64)
        g[f"attn_{prec}__finite"] = np.array([int(r.grads_finite) for r in recs], dtype=np.int32)
        for path, leaf in RB._all_tensor_leaves(model):
            g[f"attn_{prec}__p_final__{path}"] = f32(leaf.payload)
        if prec == "f32":
            for step in range(cfg.steps):
                x, y = RB.synth_data(RB._step_seed(cfg.seed, step), cfg.batch_size, cfg.num_classes,
                                     cfg.feature_dim)
                g[f"attn_data_x_{step}"] = f32(x.payload)
                g[f"attn_data_y_{step}"] = np.asarray(y.payload, dtype=np.int32)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(names)} op cases)")


if __name__ == "__main__":
    main()
