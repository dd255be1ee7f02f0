"""The benchmarked arena path at config-2 scale (BASELINE configs[1]), f16
and bf16: FusedMPStep on the full ViT-B pytree (152 leaves, 86,567,656
params) driven exactly as bench.py drives it — the SURVEY.md §8(d) recipe
(numpy default_rng(0) params and scaled grads, the grads rounded to the half
grid by K1), +inf at blocks.5.fc1.w[17, 123] on steps = 3 (mod 10), 20
steps — against the pinned oracle step (oracle.mp_step's arithmetic,
ThreadedStep over leaf shards).  Bar: bit-exact p32, m, v, p_half, the
per-step finite flags and used loss scales, the final scaling state and the
applied-step counter.  This covers what the per-leaf golden tests do not:
the finite_scan fast path of K2, a one-range leaf table of ~42K tiles and
K4's multi-wave grid."""
import os

import numpy as np
import pytest
import torch

import bench
import paper_2507_03312_b200 as mpx
from oracle import mpx_oracle as O
from paper_2507_03312_b200 import kernels as K
from paper_2507_03312_b200.step import FusedMPStep
from paper_2507_03312_b200.vit_config import VIT_B16

pytestmark = pytest.mark.gpu

STEPS = 20


@pytest.mark.parametrize("half", ["f16", "bf16"])
def test_arena_step_bit_exact_vs_oracle_full_vit_b(cuda, half):
    shapes = VIT_B16.param_shapes()
    params, grads32 = bench.recipe_host(shapes)
    n = sum(p.size for p in params)
    assert len(shapes) == 152 and n == 86_567_656
    step = FusedMPStep({k: torch.from_numpy(p).to(cuda) for (k, _), p in zip(shapes, params)}, lr=1e-3,
                       half_dtype=mpx.as_dtype(half), scaling=mpx.DynamicLossScaling(2.0 ** 15, device=cuda))
    K.cast_into([torch.from_numpy(g).to(cuda) for g in grads32], step.grad.views)
    clean = step.grad.buf
    li, flat = bench.poison_flat_index(shapes)
    assert shapes[li][0] == "blocks.5.fc1.w"
    pois = clean.clone()
    pois[step.offsets[li] + flat] = float("inf")

    # oracle: the same inputs, the reference's arithmetic, the half copy of every step
    g_clean = [O.quantize(g, half) for g in grads32]
    g_pois = list(g_clean)
    g_pois[li] = g_clean[li].copy()
    g_pois[li].reshape(-1)[flat] = np.inf
    # the device grads ARE the oracle's rounding of the recipe (K1 vs numpy)
    dev_g = clean.float().cpu().numpy()
    for (k, _), o, g in zip(shapes, step.offsets, g_clean):
        assert np.array_equal(dev_g[o:o + g.size].view(np.uint32), g.reshape(-1).view(np.uint32)), k
    del dev_g
    ref = O.ThreadedStep([p.copy() for p in params], [np.zeros_like(p) for p in params],
                         [np.zeros_like(p) for p in params], os.cpu_count() or 1, lr=1e-3, half_fmt=half)
    state, t = (2.0 ** 15, 2.0, 0.5, 2000, 0, 1.0), 0
    for i in range(STEPS):
        bad = i % 10 == 3
        step.step((pois if bad else clean).data_ptr())
        used = state[0]
        state, t, fin = ref.step(g_pois if bad else g_clean, state, t)
        torch.cuda.synchronize()
        assert fin == (not bad)
        assert int(step.flag.item()) == int(fin), i
        assert float(step.used_scale.item()) == used, i
    ref.close()
    host = step.scaling.to_host()
    assert (host.loss_scale, host.steps_since_growth) == (state[0], state[4])
    assert step.step_count == t == STEPS - 2
    arenas = {"p32": step.p32.buf.cpu().numpy(), "m": step.m.buf.cpu().numpy(), "v": step.v.buf.cpu().numpy(),
              "half": step.p_half.buf.float().cpu().numpy()}
    want = {"p32": ref.params, "m": ref.m, "v": ref.v, "half": ref.half}
    for kind, arr in arenas.items():
        for (k, _), o, w in zip(shapes, step.offsets, want[kind]):
            got = arr[o:o + w.size]
            assert np.array_equal(got.view(np.uint32), np.asarray(w, np.float32).reshape(-1).view(np.uint32)), \
                (kind, k)
