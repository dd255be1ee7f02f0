"""Generate tests/golden/acceptance_golden.npz by running the REFERENCE's own
acceptance criteria 7 and 8 (pkg/tests/test_acceptance.py:276-339): its MLP
trained by its harness (bench.fit) for 500 steps in f32 and f16 on seeds
0-2 (criterion 7: loss / 10 and an accuracy gap <= 2 pp), and the f16 run
from an absurd 2^30 loss scale (criterion 8: overflow recovery).  Also the
first batches and the held-out set of the reference's synthetic task, which
pin tests/test_acceptance_gpu.py's restatement of its data generator.

    python tests/golden/gen_acceptance_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from mpsim import bench as RB  # noqa: E402

OUT = Path(__file__).resolve().parent / "acceptance_golden.npz"


def main():
    g = {}
    for seed in (0, 1, 2):
        cfg = RB.RunConfig(precision="f32", steps=500, batch_size=32, model="mlp", feature_dim=16, seed=seed,
                           lr=1e-2)
        model0 = RB.build_model(cfg)
        for i, layer in enumerate(model0["layers"]):
            g[f"s{seed}_init_w{i}"] = np.asarray(layer["w"].payload, np.float32)
            g[f"s{seed}_init_b{i}"] = np.asarray(layer["b"].payload, np.float32)
        for step in range(2):
            x, y = RB.synth_data(RB._step_seed(seed, step), 32, 2, 16)
            g[f"s{seed}_x{step}"] = np.asarray(x.payload, np.float32)
            g[f"s{seed}_y{step}"] = np.asarray(y.payload, np.int32)
        ex, ey = RB.synth_data(np.random.SeedSequence((seed, 0x0E7A1)), 512, 2, 16)
        g[f"s{seed}_eval_x"] = np.asarray(ex.payload, np.float32)
        g[f"s{seed}_eval_y"] = np.asarray(ey.payload, np.int32)
        for prec in ("f32", "f16"):
            cfg = RB.RunConfig(precision=prec, steps=500, batch_size=32, model="mlp", feature_dim=16, seed=seed,
                               lr=1e-2)
            recs, model = RB.fit(cfg)
            g[f"s{seed}_{prec}_loss"] = np.array([r.loss for r in recs])
            g[f"s{seed}_{prec}_acc"] = np.asarray(RB.evaluate_accuracy(cfg, model))
            print(seed, prec, recs[0].loss, recs[-1].loss, float(g[f"s{seed}_{prec}_acc"]), flush=True)
    cfg = RB.RunConfig(precision="f16", steps=500, batch_size=32, model="mlp", feature_dim=16, seed=0, lr=1e-2,
                       loss_scale_init=2.0 ** 30)
    recs, model = RB.fit(cfg)
    g["c8_flags"] = np.array([int(r.grads_finite) for r in recs], np.int32)
    g["c8_scales"] = np.array([r.scale for r in recs])
    g["c8_loss"] = np.array([r.loss for r in recs])
    g["c8_acc"] = np.asarray(RB.evaluate_accuracy(cfg, model))
    print("c8 skipped", int((g["c8_flags"] == 0).sum()), "acc", float(g["c8_acc"]))
    np.savez_compressed(OUT, **g)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
