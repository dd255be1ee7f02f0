"""The torch-free data-parallel exchange of the C ABI (mpx_comm_*,
mpx_allreduce_flag, mpx_allreduce_grads; include/mpx_b200.h) on a real
NCCL communicator of world size 1 on one B200.  At W = 1 the collectives are
identities, so the step driven through them must equal the plain step bit
for bit; the flag reduction must keep the full 32-bit word (a MIN over a
flag with stray upper bytes would misread 'finite').  Multi-rank sums are
NCCL's own; the decision logic they feed is covered by the gloo tests."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(cuda):
    from paper_2507_03312_b200.dp import NativeComm

    c = NativeComm(1, NativeComm.unique_id(), 0, cuda.index or 0)
    yield c
    c.close()


def test_comm_size_and_flag_min(comm, cuda):
    assert comm.size == 1
    for v in (0, 1):
        f = torch.full((1,), v, dtype=torch.int32, device=cuda)
        comm.allreduce_flag(f)
        torch.cuda.synchronize()
        assert int(f.item()) == v


def test_allreduce_grads_identity(comm, cuda):
    g = torch.randn(10007, device=cuda).to(torch.float16)
    g[5] = float("inf")
    want = g.clone()
    comm.allreduce_grads(g)
    torch.cuda.synchronize()
    assert torch.equal(g.view(torch.int16), want.view(torch.int16))
    with pytest.raises(TypeError):
        comm.allreduce_grads(torch.zeros(4, dtype=torch.int32, device=cuda))


def test_bad_unique_id_length():
    from paper_2507_03312_b200.dp import NativeComm

    with pytest.raises(ValueError):
        NativeComm(1, b"short", 0, 0)


@pytest.mark.parametrize("half", ["f16", "bf16"])
def test_fused_step_through_native_comm_matches_plain(comm, cuda, half):
    import paper_2507_03312_b200 as mpx
    from paper_2507_03312_b200.step import FusedMPStep

    rng = np.random.default_rng(3)
    shapes = {"a": (33, 65), "b": (4099,), "c": (5,)}
    p0 = {k: torch.from_numpy(rng.standard_normal(s).astype(np.float32) * 0.05).to(cuda) for k, s in shapes.items()}
    steps = [FusedMPStep(p0, lr=1e-3, half_dtype=half, scaling=mpx.DynamicLossScaling(2.0 ** 15, device=cuda),
                         comm=c) for c in (None, comm)]
    for i in range(6):
        g = {k: torch.from_numpy(rng.standard_normal(s).astype(np.float32) * 30.0) for k, s in shapes.items()}
        if i == 2:
            g["b"][11] = float("inf")
        for st in steps:
            tr = st.tree("grad")
            for k in shapes:
                tr[k].copy_(g[k].to(cuda).to(tr[k].dtype))
            st.step()
        torch.cuda.synchronize()
        assert bool(steps[0].grads_finite) == bool(steps[1].grads_finite) == (i != 2)
    for kind in ("p32", "m", "v", "half"):
        a, b = steps[0].tree(kind), steps[1].tree(kind)
        for k in shapes:
            assert torch.equal(a[k], b[k]), (kind, k)
    assert steps[0].step_count == steps[1].step_count == 5
    assert steps[0].scaling.to_host().loss_scale == steps[1].scaling.to_host().loss_scale


def test_comm_excludes_torch_group(comm, cuda):
    from paper_2507_03312_b200.step import FusedMPStep

    with pytest.raises(ValueError):
        FusedMPStep({"w": torch.zeros(8, device=cuda)}, lr=1e-3, zero=True, zero_world=1, zero_rank=0, comm=comm)
