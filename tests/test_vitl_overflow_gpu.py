"""BASELINE.json configs[4]: ViT-L/16 fp16 with initial loss scale 2^32 —
the overflow stress.  Parity: the device scale trajectory
must equal the reference state machine (oracle.simulate_scaling) fed the
run's own flags, bit for bit; skipped steps must leave the f32 master
weights, the moments and the step counter bit-identical (optim.py:102-103);
the scale must back off until steps go through."""
import numpy as np
import pytest
import torch

from oracle import mpx_oracle as O
from paper_2507_03312_b200 import F16
from paper_2507_03312_b200.trainer import ViTTrainer
from paper_2507_03312_b200.vit_config import VIT_L16

pytestmark = pytest.mark.gpu


def test_vitl16_overflow_stress_trajectory(cuda):
    tr = ViTTrainer(VIT_L16, 8, half=F16, lr=1e-4, device=cuda, loss_scale=2.0 ** 32)
    g = torch.Generator(device=cuda).manual_seed(5)
    used, flags = [], []
    for step in range(24):
        x = torch.randn(8, 224, 224, 3, device=cuda, generator=g)
        y = torch.randint(0, 1000, (8,), device=cuda, generator=g).to(torch.int32)
        before = (tr.mp.p32.buf.clone(), tr.mp.m.buf.clone(), tr.mp.step_count) if step < 3 else None
        tr.step(x, y)
        fin = bool(tr.grads_finite)
        used.append(float(tr.mp.used_scale.item()))
        flags.append(fin)
        if before is not None and not fin:
            assert torch.equal(tr.mp.p32.buf, before[0]) and torch.equal(tr.mp.m.buf, before[1])
            assert tr.mp.step_count == before[2]
    sim = O.simulate_scaling(2.0 ** 32, 2.0, 0.5, 2000, 1.0, flags)
    assert used[0] == 2.0 ** 32
    assert used[1:] == [s for s, _ in sim[:-1]], (used, flags)
    assert tr.scaling.loss_scale == sim[-1][0]
    assert not flags[0], "2^32 must overflow the f16 backward"
    assert any(flags), f"scale never backed off far enough: {used}"
    assert np.isfinite(tr.engine.loss.item())
