"""Randomised shape / stride / broadcast coverage of the drop-in tensor layer
(paper_2507_03312_b200.tensors) against float64 torch on the same values:
non-contiguous (transposed, sliced, expanded) operands, broadcasting in
every position, batched matmuls with broadcast batch dims on both the
tcgen05 path (aligned half operands) and the SIMT path, reductions and
softmax over every axis, and gradients through torch.autograd.  The golden
fixtures (test_tensor_ops_gpu.py) pin the numerics against mpsim; this file
pins the indexing."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 2e-5, torch.float16: 2e-3, torch.bfloat16: 1.6e-2}


def close(got, want, dt, scale=1.0):
    got = got.detach().double().cpu()
    want = want.detach().double().cpu()
    assert got.shape == want.shape, (got.shape, want.shape)
    err = (got - want).abs().max().item() if got.numel() else 0.0
    ref = max(want.abs().max().item() if want.numel() else 0.0, 1.0)
    assert err <= TOL[dt] * ref * scale, (err, ref)


def _views(t, rng):
    """the tensor itself, or a non-contiguous view holding the same values"""
    k = rng.integers(0, 3)
    if k == 0 or t.ndim < 2:
        return t
    if k == 1:  # a transposed copy viewed back
        return t.transpose(-1, -2).contiguous().transpose(-1, -2)
    big = torch.zeros(*t.shape[:-1], t.shape[-1] * 2, dtype=t.dtype, device=t.device)
    big[..., ::2] = t
    return big[..., ::2]  # strided slice


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_binary_broadcast_and_grads(cuda, seed, dt):
    from paper_2507_03312_b200 import tensors as T

    rng = np.random.default_rng(seed)
    nd = int(rng.integers(1, 5))
    shape = [int(rng.integers(1, 7)) for _ in range(nd)]
    bshape = [1 if rng.random() < 0.4 else s for s in shape][int(rng.integers(0, nd)):]
    a64 = torch.randn(*shape, dtype=torch.float64)
    b64 = torch.randn(*bshape, dtype=torch.float64).abs() + 0.5
    a = _views(a64.to(dt).to(cuda), rng).as_subclass(T.Tensor).requires_grad_()
    b = _views(b64.to(dt).to(cuda), rng).as_subclass(T.Tensor).requires_grad_()
    ar, br = a.detach().double().requires_grad_(), b.detach().double().requires_grad_()
    op = ["add", "sub", "mul", "div"][seed % 4]
    out = getattr(T, op)(a, b)
    ref = {"add": ar + br, "sub": ar - br, "mul": ar * br, "div": ar / br}[op]
    close(out, ref, dt)
    w = torch.randn(out.shape, dtype=torch.float64)
    ga, gb = torch.autograd.grad(T.reduce("sum", T.mul(out, T.tensor(w.numpy(), dt))), (a, b))
    gra, grb = torch.autograd.grad((ref * w.to(ref.device)).sum(), (ar, br))
    close(ga, gra, dt, 4)
    close(gb, grb, dt, 4 * max(1, out.numel() // max(1, b.numel())))


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_matmul_shapes(cuda, seed, dt):
    from paper_2507_03312_b200 import tensors as T

    rng = np.random.default_rng(100 + seed)
    aligned = seed % 2 == 0  # multiples of 8 on K and N: the tcgen05 path for half operands
    M = int(rng.integers(1, 40))
    K = 8 * int(rng.integers(1, 6)) if aligned else int(rng.integers(1, 30))
    N = 8 * int(rng.integers(1, 6)) if aligned else int(rng.integers(1, 30))
    lead_a = [int(rng.integers(1, 4)) for _ in range(int(rng.integers(0, 3)))]
    lead_b = [1 if rng.random() < 0.5 else s for s in lead_a][int(rng.integers(0, len(lead_a) + 1)):]
    a64 = torch.randn(*lead_a, M, K, dtype=torch.float64)
    b64 = torch.randn(*lead_b, K, N, dtype=torch.float64)
    if seed % 5 == 4:
        a64 = torch.randn(K, dtype=torch.float64)  # 1-d operand (numpy rules: a row, dropped again)
    a = _views(a64.to(dt).to(cuda), rng).as_subclass(T.Tensor).requires_grad_()
    b = _views(b64.to(dt).to(cuda), rng).as_subclass(T.Tensor).requires_grad_()
    ar, br = a.detach().double().requires_grad_(), b.detach().double().requires_grad_()
    out = a @ b
    ref = torch.matmul(ar, br)
    close(out, ref, dt, K ** 0.5)
    w = torch.randn(out.shape, dtype=torch.float64, device=cuda)
    ga, gb = torch.autograd.grad(T.reduce("sum", T.mul(out, T.tensor(w.cpu().numpy(), dt))), (a, b))
    gra, grb = torch.autograd.grad((ref * w).sum(), (ar, br))
    close(ga, gra, dt, 8 * (N ** 0.5))
    close(gb, grb, dt, 8 * (max(M, 1) ** 0.5) * max(1, out.numel() // max(1, M * N)))


@pytest.mark.parametrize("seed", range(10))
def test_reduce_softmax_axes(cuda, seed):
    from paper_2507_03312_b200 import tensors as T

    rng = np.random.default_rng(200 + seed)
    nd = int(rng.integers(1, 4))
    shape = [int(rng.integers(1, 9)) for _ in range(nd)]
    x64 = torch.randn(*shape, dtype=torch.float64) * 3
    x = _views(x64.float().to(cuda), rng).as_subclass(T.Tensor).requires_grad_()
    xr = x.detach().double().requires_grad_()
    ax = int(rng.integers(-nd, nd))
    for op, ref in (("sum", xr.sum(ax)), ("mean", xr.mean(ax)), ("max", xr.amax(ax))):
        close(T.reduce(op, x, axis=ax), ref, torch.float32, shape[ax])
    close(T.reduce("sum", x), xr.sum(), torch.float32, x.numel())
    y = T.softmax(x, axis=ax)
    yr = torch.softmax(xr, ax)
    close(y, yr, torch.float32)
    w = torch.randn(y.shape, dtype=torch.float64, device=cuda)
    (g,) = torch.autograd.grad(T.reduce("sum", T.mul(y, T.tensor(w.cpu().numpy()))), (x,))
    (gr,) = torch.autograd.grad((yr * w).sum(), (xr,))
    close(g, gr, torch.float32, 4)


@pytest.mark.parametrize("seed", range(6))
def test_layernorm_and_cross_entropy_rows(cuda, seed):
    from paper_2507_03312_b200 import tensors as T

    rng = np.random.default_rng(300 + seed)
    rows, n = int(rng.integers(1, 50)), int(rng.integers(2, 40))
    x64 = torch.randn(rows, n, dtype=torch.float64) * 2 + 0.5
    g64 = 1 + 0.1 * torch.randn(n, dtype=torch.float64)
    b64 = 0.1 * torch.randn(n, dtype=torch.float64)
    x, g, b = (T.tensor(t.numpy().astype(np.float32)).requires_grad_() for t in (x64, g64, b64))
    xr, gr, br = (t.detach().double().requires_grad_() for t in (x, g, b))
    y = T.layernorm(x, g, b)
    yr = torch.nn.functional.layer_norm(xr, (n,), gr, br, eps=1e-5)
    close(y, yr, torch.float32, 4)
    w = torch.randn(rows, n, dtype=torch.float64, device=cuda)
    grads = torch.autograd.grad(T.reduce("sum", T.mul(y, T.tensor(w.cpu().numpy()))), (x, g, b))
    grefs = torch.autograd.grad((yr * w).sum(), (xr, gr, br))
    for a_, b_ in zip(grads, grefs):
        close(a_, b_, torch.float32, 8 * rows)
    lab = rng.integers(0, n, rows).astype(np.int32)
    loss = T.cross_entropy(x, T.tensor(lab, "i32"))
    lr_ = torch.nn.functional.cross_entropy(xr, torch.from_numpy(lab).long().to(cuda))
    close(loss, lr_, torch.float32, 4)
