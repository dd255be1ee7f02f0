"""The reference's acceptance criteria 7 and 8 (pkg/tests/test_acceptance.py:
276-339) on the B200 through the drop-in API: its MLP (bench.py:161-168)
written against paper_2507_03312_b200.tensors, trained with
filter_value_and_grad + optimizer_update (the harness loop, bench.py:255-295)
on its synthetic task, against the reference's own runs
(tests/golden/gen_acceptance_golden.py).

  C7  f32 / f16 training parity: 500 steps on seeds 0-2, the final loss below
      a tenth of the first, held-out accuracy within 2 pp of the f32 run (and of
      the reference's accuracies);
  C8  overflow recovery from a 2^30 loss scale: the scale halves every step
      until the first finite one (the same number of skips as the reference),
      skipped steps leave the parameters bit-identical, the scale column
      replays on the reference's state machine, then training recovers
      (loss / 10, accuracy > 0.95)."""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import mpx_oracle as O

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).resolve().parent / "golden" / "acceptance_golden.npz")
STEPS = 500


def _centers(num_classes=2, dim=16):
    """the task's fixed cluster geometry (bench.py:109-113)"""
    rng = np.random.default_rng(1234)
    c = rng.standard_normal((num_classes, dim))
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    return (c * 6.0).astype(np.float32)


def _synth(seed_seq, batch, num_classes=2, dim=16):
    """one batch of the reference's synthetic task (bench.py:116-122)"""
    rng = np.random.default_rng(seed_seq)
    labels = rng.integers(0, num_classes, size=batch)
    x = _centers(num_classes, dim)[labels] + rng.standard_normal((batch, dim))
    return x.astype(np.float32), labels.astype(np.int32)


def _step_seed(seed, step):
    return np.random.SeedSequence((seed, 1 + step))


def _mlp(T, params, x):
    z = x
    layers = params["layers"]
    for i, layer in enumerate(layers):
        z = z @ layer["w"] + layer["b"]
        if i < len(layers) - 1:
            z = T.relu(z)
    return z


def _train(seed, prec, init_scale=2.0 ** 15, record_params=False):
    import paper_2507_03312_b200 as mpx
    from paper_2507_03312_b200 import tensors as T

    model = {"layers": [{"w": T.tensor(G[f"s{seed}_init_w{i}"]), "b": T.tensor(G[f"s{seed}_init_b{i}"])}
                        for i in range(3)]}
    state = mpx.adam_init(model, 1e-2)
    scaling = mpx.LossScaling(init_scale)

    def loss_fn(p, b):
        return T.cross_entropy(_mlp(T, p, b["x"]), b["y"])

    losses, scales, flags, snaps = [], [], [], []
    with mpx.half_precision("f16"):
        for step in range(STEPS):
            x, y = _synth(_step_seed(seed, step), 32)
            res = mpx.filter_value_and_grad(loss_fn, scaling, use_mixed_precision=prec != "f32")(
                model, {"x": T.tensor(x), "y": T.tensor(y, "i32")})
            model, state = mpx.optimizer_update(model, state, res.grads, res.grads_finite)
            losses.append(float(res.value.item()))
            scales.append(scaling.loss_scale)
            flags.append(int(bool(res.grads_finite)))
            if record_params and step < 40:
                snaps.append(np.concatenate([t.detach().float().cpu().numpy().reshape(-1)
                                             for layer in model["layers"] for t in (layer["w"], layer["b"])]))
            scaling = res.scaling
    ex, ey = G[f"s{seed}_eval_x"], G[f"s{seed}_eval_y"]
    logits = _mlp(T, model, T.tensor(ex))  # evaluated in f32 (bench.py:300-306)
    acc = float((np.argmax(logits.detach().float().cpu().numpy(), axis=1) == ey).mean())
    return np.array(losses), scales, flags, acc, snaps


def test_synthetic_task_restatement_matches_reference():
    for seed in (0, 1, 2):
        for step in range(2):
            x, y = _synth(_step_seed(seed, step), 32)
            assert np.array_equal(x, G[f"s{seed}_x{step}"]) and np.array_equal(y, G[f"s{seed}_y{step}"])
        ex, ey = _synth(np.random.SeedSequence((seed, 0x0E7A1)), 512)
        assert np.array_equal(ex, G[f"s{seed}_eval_x"]) and np.array_equal(ey, G[f"s{seed}_eval_y"])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_criterion_7_training_parity(cuda, seed):
    acc = {}
    for prec in ("f32", "f16"):
        losses, _, flags, acc[prec], _ = _train(seed, prec)
        assert losses[-1] < 0.1 * losses[0], (seed, prec, losses[0], losses[-1])
        assert abs(losses[0] - G[f"s{seed}_{prec}_loss"][0]) <= 1e-2 * G[f"s{seed}_{prec}_loss"][0]
        assert abs(acc[prec] - float(G[f"s{seed}_{prec}_acc"])) <= 0.02, (seed, prec, acc[prec])
    assert abs(acc["f32"] - acc["f16"]) <= 0.02, (seed, acc)


def test_criterion_8_overflow_recovery(cuda):
    losses, scales, flags, acc, snaps = _train(0, "f16", init_scale=2.0 ** 30, record_params=True)
    ref_flags = G["c8_flags"].tolist()
    assert flags[0] == 0
    first = flags.index(1)
    assert abs(first - ref_flags.index(1)) <= 1, (first, ref_flags.index(1))  # the marginal step may flip
    for i in range(first):
        assert scales[i] == 2.0 ** 30 * 0.5 ** i  # halves every step
    sim = O.simulate_scaling(2.0 ** 30, 2.0, 0.5, 2000, 1.0, flags)
    assert scales[1:] == [s for s, _ in sim[:-1]]
    init = np.concatenate([np.concatenate([G[f"s0_init_w{i}"].reshape(-1), G[f"s0_init_b{i}"]]) for i in range(3)])
    for i in range(first):  # skipped steps leave the parameters bit-identical
        assert np.array_equal(snaps[i].view(np.uint32), init.view(np.uint32)), i
    assert np.isfinite(losses[first]) and losses[-1] < 0.1 * losses[first]
    assert acc > 0.95
