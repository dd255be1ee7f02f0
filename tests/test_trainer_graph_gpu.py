"""ViTTrainer: the captured CUDA-graph step (two captures over two input
buffers, PDL edges for the MP-step chain inside) replays bit-identically to
eager steps — master weights, moments, half copy, loss-scale state and step
counter — including a step that overflows (skip + backoff)."""
import pytest
import torch

from paper_2507_03312_b200 import F16
from paper_2507_03312_b200.trainer import ViTTrainer
from paper_2507_03312_b200.vit_config import ViTConfig

pytestmark = pytest.mark.gpu
CFG = ViTConfig(img=32, patch=4, dim=128, depth=2, heads=2, mlp=256, classes=10, pool="cls")


def _batches(dev, n, B):
    g = torch.Generator(device=dev).manual_seed(11)
    out = []
    for i in range(n):
        x = torch.randn(B, 32, 32, 3, device=dev, generator=g)
        if i == 2:
            x[0, 0, 0, 0] = 1e30  # overflows the f16 forward: a skipped step
        out.append((x, torch.randint(0, 10, (B,), device=dev, generator=g).to(torch.int32)))
    return out


def _state(tr):
    torch.cuda.synchronize()
    return (tr.mp.p32.buf.clone(), tr.mp.m.buf.clone(), tr.mp.v.buf.clone(), tr.mp.p_half.buf.clone(),
            tr.scaling.to_host(), tr.mp.step_count)


def test_graph_replay_matches_eager(cuda):
    B, steps = 8, 6
    data = _batches(cuda, steps, B)
    eager = ViTTrainer(CFG, B, half=F16, lr=1e-3, device=cuda, loss_scale=2.0 ** 15)
    for x, y in data:
        eager.step(x, y)
    graph = ViTTrainer(CFG, B, half=F16, lr=1e-3, device=cuda, loss_scale=2.0 ** 15)
    bufs = [(torch.empty_like(data[0][0]), torch.empty_like(data[0][1])) for _ in range(2)]
    # capture() runs `warmup` eager steps first: feed it the first batches
    bufs[0][0].copy_(data[0][0])
    bufs[0][1].copy_(data[0][1])
    g0 = graph.capture(*bufs[0], warmup=1)  # step 0 (eager warm-up) ...
    # the warm-up consumed batch 0; replay the rest alternating the two captures
    bufs[1][0].copy_(data[1][0])
    bufs[1][1].copy_(data[1][1])
    g1 = graph.capture(*bufs[1], warmup=1)  # ... step 1 (eager warm-up)
    for i in range(2, steps):
        b = i % 2
        bufs[b][0].copy_(data[i][0])
        bufs[b][1].copy_(data[i][1])
        graph.replay(g0 if b == 0 else g1)
    se, sg = _state(eager), _state(graph)
    for a, b in zip(se[:4], sg[:4]):
        assert torch.equal(a, b)
    assert se[4] == sg[4] and se[5] == sg[5]
    assert se[5] == steps - 1, "the overflow step must be skipped"
