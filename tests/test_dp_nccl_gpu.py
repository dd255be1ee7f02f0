"""The data-parallel path of the ViT trainer — per-bucket async NCCL
all-reduce launched from the backward, the finite-flag MIN all-reduce, and
under ZeRO-1 the per-bucket reduce-scatter and the all-gather of the half
working copy — run through real NCCL on one GPU with world size 1.  Every
collective is an identity there, so the production N > 1 code path must
reproduce the single-process trainer bit for bit (master weights, moments,
loss scale, step count).  The multi-rank sums themselves are covered by the
gloo tests (tests/test_dp_cpu.py)."""
import pytest
import torch
import torch.distributed as dist

from paper_2507_03312_b200.trainer import ViTTrainer
from paper_2507_03312_b200.tree import float_leaves
from paper_2507_03312_b200.vit_config import ViTConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1(cuda):
    if dist.is_initialized():
        pytest.skip("a process group already exists in this process")
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("zero", [False, True])
def test_dp_trainer_world1_equals_single_process(cuda, nccl_world1, zero):
    cfg = ViTConfig(img=32, patch=4, dim=128, depth=2, heads=2, mlp=256, classes=16, pool="cls")
    B = 8
    ref = ViTTrainer(cfg, B, half="f16", device=cuda, seed=0, loss_scale=2.0 ** 15)
    dp = ViTTrainer(cfg, B, half="f16", device=cuda, seed=0, loss_scale=2.0 ** 15, group=nccl_world1,
                    world_size=1, zero=zero)
    g = torch.Generator(device=cuda).manual_seed(0)
    for i in range(4):
        x = torch.randn(B, 32, 32, 3, device=cuda, generator=g)
        y = torch.randint(0, 16, (B,), device=cuda, generator=g).to(torch.int32)
        if i == 2:
            x[0, 0, 0, 0] = float("inf")  # a non-finite step: both must skip it
        l1 = ref.step(x, y)
        l2 = dp.step(x, y)
        torch.cuda.synchronize()
        assert bool(ref.grads_finite) == bool(dp.grads_finite) == (i != 2)
        if i != 2:
            assert torch.equal(l1, l2), i
    for kind in ("p32", "m", "v", "half"):
        # under ZeRO-1 the f32 state is all-gathered from the shards
        a = [x for _, x in float_leaves(ref.mp.gather(kind))]
        b = [x for _, x in float_leaves(dp.mp.gather(kind))]
        for path, va, vb in zip(ref.mp.paths, a, b):
            assert torch.equal(va, vb), (kind, path)
    assert ref.mp.step_count == dp.mp.step_count == 3
    assert ref.scaling.to_host().loss_scale == dp.scaling.to_host().loss_scale


@pytest.mark.parametrize("zero", [False, True])
def test_dp_trainer_graph_world1_equals_eager(cuda, nccl_world1, zero):
    """The data-parallel step captured as one CUDA graph (NCCL collectives
    inside) replays bit-identically to eager data-parallel steps."""
    cfg = ViTConfig(img=32, patch=4, dim=128, depth=2, heads=2, mlp=256, classes=16, pool="cls")
    B = 8
    eager = ViTTrainer(cfg, B, half="f16", device=cuda, seed=0, group=nccl_world1, world_size=1, zero=zero)
    graph = ViTTrainer(cfg, B, half="f16", device=cuda, seed=0, group=nccl_world1, world_size=1, zero=zero)
    g = torch.Generator(device=cuda).manual_seed(1)
    x = torch.randn(B, 32, 32, 3, device=cuda, generator=g)
    y = torch.randint(0, 16, (B,), device=cuda, generator=g).to(torch.int32)
    xs, ys = x.clone(), y.clone()
    graph.capture(xs, ys, warmup=2)  # two warm-up steps run eagerly inside capture()
    for _ in range(2):
        eager.step(x, y)
    for i in range(3):
        x2 = torch.randn(B, 32, 32, 3, device=cuda, generator=g)
        y2 = torch.randint(0, 16, (B,), device=cuda, generator=g).to(torch.int32)
        xs.copy_(x2)
        ys.copy_(y2)
        l1 = eager.step(x2, y2)
        l2 = graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(l1, l2), i
    for kind in ("p32", "m", "v", "half"):
        a = [x for _, x in float_leaves(eager.mp.gather(kind))]
        b = [x for _, x in float_leaves(graph.mp.gather(kind))]
        for path, va, vb in zip(eager.mp.paths, a, b):
            assert torch.equal(va, vb), (kind, path)
