"""ZeRO-1 sharded optimizer step on one GPU: two
FusedMPStep shards (world 2, ranks 0 and 1) with the reduce-scatter and
all-gather done by hand must equal the replicated step on the summed grads
bit for bit — master weights, moments, half working copy, scale state, step
counter — including a step whose only non-finite value lives in the other
rank's shard (the flag AND makes both skip)."""
import pytest
import torch

import paper_2507_03312_b200 as mpx
from paper_2507_03312_b200 import F16
from paper_2507_03312_b200.dp import zero_bucket_views
from paper_2507_03312_b200.step import FusedMPStep
from paper_2507_03312_b200.vit import init_params
from paper_2507_03312_b200.vit_config import VIT_TINY

pytestmark = pytest.mark.gpu


def _leafwise(step, kind):
    return dict(zip(step.paths, {"p32": step.p32, "half": step.p_half}[kind].views))


def test_zero_shards_equal_replicated(cuda):
    params = init_params(VIT_TINY, cuda, seed=1)
    full = FusedMPStep(params, 1e-3, half_dtype=F16, scaling=mpx.DynamicLossScaling(2.0 ** 10, device=cuda))
    shards = [FusedMPStep(params, 1e-3, half_dtype=F16, scaling=mpx.DynamicLossScaling(2.0 ** 10, device=cuda),
                          zero=True, zero_world=2, zero_rank=r) for r in range(2)]
    g = torch.Generator(device=cuda).manual_seed(3)
    for it in range(5):
        # two ranks' local (scaled) grads, per leaf
        local = [{p: (torch.randn(v.shape, device=cuda, generator=g) * 4.0).half()
                  for p, v in zip(full.paths, full.grad.views)} for _ in range(2)]
        if it == 3:  # one +inf on rank 1, in a leaf rank 0's shard does not own
            local[1][full.paths[-3]].view(-1)[1] = float("inf")
        summed = {p: (local[0][p].float() + local[1][p].float()).half() for p in full.paths}
        for v, p in zip(full.grad.views, full.paths):
            v.copy_(summed[p])
        full.step()
        # ZeRO: each shard holds its own local grads, reduce-scatter by hand
        for r in range(2):
            for v, p in zip(shards[r].grad.views, shards[r].paths):
                v.copy_(local[r][p])
        views = [zero_bucket_views(s.grad.buf, s.ranges, 2, r) for r, s in enumerate(shards)]
        for b in range(len(views[0])):
            tot = views[0][b][0].float() + views[1][b][0].float()  # whole bucket, summed over ranks
            for r in range(2):
                whole, mine = views[r][b]
                o = (mine.data_ptr() - whole.data_ptr()) // 2
                mine.copy_(tot[o:o + mine.numel()].half())
        for s in shards:
            s.k2()
        f = torch.minimum(shards[0].flag, shards[1].flag)  # the flag all-reduce (MIN)
        for s in shards:
            s.flag.copy_(f)
            s.k4()
            s.k3()
        hv = [zero_bucket_views(s.p_half.buf, s.ranges, 2, r) for r, s in enumerate(shards)]
        for b in range(len(hv[0])):  # all-gather of the half working copy
            for r in range(2):
                src = hv[r][b][1]
                o = (src.data_ptr() - hv[r][b][0].data_ptr()) // 2
                hv[1 - r][b][0][o:o + src.numel()].copy_(src)
        torch.cuda.synchronize()
        assert bool(full.grads_finite) == bool(shards[0].grads_finite) == (it != 3)
    for kind in ("p32", "m", "v"):  # each rank holds exactly its chunks, equal to the replicated state
        want = {"p32": full.p32, "m": full.m, "v": full.v}[kind].buf
        covered = [torch.zeros(v.numel(), dtype=torch.bool, device=cuda) for v in full.grad.views]
        for r, s in enumerate(shards):
            chunks = s.shard_chunks(kind)
            assert 2 * sum(c.numel() for _, c in chunks) == s.numel  # 1/W of the f32 state per rank
            canvas = torch.full((s.numel,), float("nan"), device=cuda)
            for off, c in chunks:
                canvas[off:off + c.numel()] = c
            for i, v in enumerate(full.grad.views):
                got = canvas[s.offsets[i]:s.offsets[i] + v.numel()]
                ref = want[full.offsets[i]:full.offsets[i] + v.numel()]
                mine = ~torch.isnan(got)
                assert torch.equal(got[mine], ref[mine]), (kind, r, s.paths[i])
                covered[i] |= mine
        assert all(bool(c.all()) for c in covered)  # the two shards cover every element
        with pytest.raises(ValueError):
            shards[0].tree(kind)
    for s in shards:  # the gathered half copy is whole on both ranks
        for p, h in _leafwise(s, "half").items():
            assert torch.equal(h, _leafwise(full, "half")[p]), p
        assert s.step_count == full.step_count == 4
        assert s.scaling.to_host() == full.scaling.to_host()
