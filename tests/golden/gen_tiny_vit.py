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

import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

import mpsim  # noqa: E402
from mpsim import F16, F32, I32, LossScaling, adam_init, filter_value_and_grad, force_full_precision, tensor  # noqa: E402
from mpsim import tensors as T  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent))
import tiny_vit_model as TM  # noqa: E402  (the model source shared with the GPU test)

HD64 = "--hd64" in sys.argv
D, H = (128, 2) if HD64 else (64, 4)
B = TM.B
batch = TM.batch


def param_shapes():
    return TM.param_shapes(D)


def init_params(seed=0):
    return TM.init_params(seed, D)


loss_fn = TM.make_loss_fn(SimpleNamespace(T=T, tensor=tensor, F32=F32, force_full_precision=force_full_precision),
                          D=D, H=H)


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
    --margins [--probe=F]: at every step also evaluate the SAME model/batch at
    scale/F and scale*F (F = 1.25 by default; not applied); a step is marginal
    when those two flags differ, i.e. the overflow boundary lies within a
    factor F of the scale used, where f32 vs stepwise-f16 accumulation may
    legitimately flip it."""
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    log2 = int(args[0]) if len(args) > 0 else 15
    steps = int(args[1]) if len(args) > 1 else 20
    gi = _opt("gi", 2000)
    margins = "--margins" in sys.argv
    probe = 1.25
    for a in sys.argv[1:]:
        if a.startswith("--probe="):
            probe = float(a.split("=", 1)[1])
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
            for mult, col in ((1.0 / probe, lo_flags), (probe, hi_flags)):
                probed = scaling._replace(loss_scale=scaling.loss_scale * mult)
                col.append(bool(filter_value_and_grad(loss_fn, probed)(model, args_).grads_finite))
        model, opt = mpsim.optimizer_update(model, opt, res.grads, res.grads_finite)
        losses.append(float(res.value.item()))
        scales.append(scaling.loss_scale)
        flags.append(bool(res.grads_finite))
        sums.append(checksum(model))
        scaling = res.scaling
        print(f"step {step} loss {losses[-1]:.6f} scale {scales[-1]} finite {flags[-1]}"
              + (f" (s/{probe} {lo_flags[-1]}, {probe}s {hi_flags[-1]})" if margins else "") + f" ({time.time() - t0:.1f}s)",
              flush=True)
    tag = f"s{log2}" + (f"_gi{gi}" if gi != 2000 else "") + (f"_m{probe:g}" if margins else "")
    out = Path(__file__).resolve().parent / (f"tiny_vit_hd64_{tag}.npz" if HD64 else f"tiny_vit_{tag}.npz")
    extra = {"flags_scale_down": np.asarray(lo_flags), "flags_scale_up": np.asarray(hi_flags),
             "probe_factor": np.asarray(probe)} if margins else {}
    np.savez_compressed(out, losses=np.asarray(losses), scales=np.asarray(scales), flags=np.asarray(flags),
                        checksums=np.asarray(sums, dtype=np.uint64), growth_interval=np.asarray(gi),
                        **extra, **{"init." + k: v for k, v in p0.items()})
    print("wrote", out)


if __name__ == "__main__":
    main()
