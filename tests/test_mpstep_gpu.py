"""Parity of the CUDA mixed-precision step (K1-K4) with the reference.

Golden vectors come from running mpsim itself (tests/golden/gen_golden.py);
random cases are checked against the pinned CPU oracle.  Bar: bit-exact
(NaN compared by class)."""
import math

import numpy as np
import pytest
import torch

import paper_2507_03312_b200 as mpx
from paper_2507_03312_b200 import kernels as K
from oracle import mpx_oracle as O

pytestmark = pytest.mark.gpu

TORCH = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}


def f32(bits):
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def same_bits(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    if a.shape != b.shape:
        return False
    nan = np.isnan(a) & np.isnan(b)
    return bool(np.all(nan | (a.view(np.uint32) == b.view(np.uint32))))


def dev(x, fmt, cuda):
    """device tensor of format fmt holding values already on fmt's grid"""
    return torch.from_numpy(np.asarray(x, np.float32)).to(cuda).to(TORCH[fmt])


# ---------------------------------------------------------------- K1 cast
@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_cast_matches_reference_tables(cuda, golden, fmt):
    x = torch.from_numpy(f32(golden[f"quant_{fmt}_in"])).to(cuda)
    out = mpx.cast_tree({"w": x}, mpx.as_dtype(fmt))["w"]
    assert out.dtype == TORCH[fmt]
    assert same_bits(host(out), f32(golden[f"quant_{fmt}_out"]))


@pytest.mark.parametrize("src,dst", [("f32", "f16"), ("f32", "bf16"), ("f16", "bf16"), ("bf16", "f16"),
                                     ("f16", "f32"), ("bf16", "f32")])
def test_cast_ragged_multi_leaf(cuda, src, dst):
    rng = np.random.default_rng(3)
    sizes = [0, 1, 7, 2047, 2048, 2049, 4096 + 13, 70000]
    raw = [(rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))).astype(np.float32) for n in sizes]
    leaves = [dev(O.quantize(r, src), src, cuda) for r in raw]
    # a misaligned view (offset by one element) exercises the scalar path
    base = dev(O.quantize(raw[-1], src), src, cuda)
    leaves.append(base[1:])
    outs = mpx.cast_tree(leaves, mpx.as_dtype(dst))
    for x, y in zip(leaves, outs):
        assert same_bits(host(y), O.quantize(host(x), dst))


def test_cast_tree_semantics(cuda):
    t = {"w": mpx.tensor([1.0, 2.0 ** -25]), "k": mpx.tensor([7], mpx.I32), "s": "opaque",
         "weak": mpx.Scalar(0.1), "strong": mpx.Scalar(0.1, weak=False, dtype=mpx.F32)}
    out = mpx.cast_tree(t, mpx.F16)
    assert out["w"].dtype == torch.float16 and host(out["w"]).tolist() == [1.0, 0.0]
    assert out["k"] is t["k"] and out["s"] is t["s"] and out["weak"] is t["weak"]
    assert out["strong"].dtype is mpx.F16 and out["strong"].value == pytest.approx(0.0999755859375)
    assert mpx.cast_tree({}, mpx.F16) == {} and mpx.cast_tree([], mpx.F32) == []
    with pytest.raises(ValueError):
        mpx.cast_tree(t, mpx.I32)
    h = {"w": mpx.tensor([0.1, 65504.0], mpx.F16)}
    assert torch.equal(mpx.cast_tree(h, mpx.F16)["w"], h["w"])


def test_cast_aliases_and_process_switch(cuda):
    t = {"w": mpx.tensor([1.0])}
    assert mpx.cast_to_float16(t)["w"].dtype == torch.float16
    assert mpx.cast_to_bfloat16(t)["w"].dtype == torch.bfloat16
    assert mpx.cast_to_float32(mpx.cast_to_float16(t))["w"].dtype == torch.float32
    assert mpx.get_half_precision() is mpx.F16
    assert mpx.cast_to_half_precision(t)["w"].dtype == torch.float16
    with mpx.half_precision(mpx.BF16):
        assert mpx.cast_to_half_precision(t)["w"].dtype == torch.bfloat16
    assert mpx.get_half_precision() is mpx.F16
    with pytest.raises(ValueError):
        mpx.set_half_precision(mpx.F32)


def test_cast_function_and_islands(cuda):
    g = mpx.cast_function(lambda x: x, mpx.F16)
    out = g(mpx.tensor([0.1]))
    assert out.dtype == torch.float16 and host(out)[0] == np.float32(np.float16(0.1))
    s = mpx.cast_function(lambda x: x.sum(), mpx.F16, return_dtype=mpx.F32)(mpx.tensor([60000.0, 60000.0]))
    assert s.dtype == torch.float32 and math.isinf(s.item())
    with pytest.raises(ValueError):
        mpx.force_full_precision(lambda x: x, None)
    sm = mpx.force_full_precision(lambda x, dim: torch.softmax(x, dim), mpx.F16)
    p = sm(mpx.tensor([3.0, 3.0], mpx.F16), dim=0)
    assert p.dtype == torch.float16 and host(p).tolist() == [0.5, 0.5]
    ident = mpx.force_full_precision(lambda x: x, mpx.BF16)(mpx.tensor([0.1], mpx.F16))
    want = O.quantize(O.quantize(np.float32(0.1), "f16"), "bf16")
    assert ident.dtype == torch.bfloat16 and same_bits(host(ident), want.reshape(1))


def test_cast_is_differentiable(cuda):
    w = mpx.tensor([0.1, 3.0]).requires_grad_(True)
    h = mpx.cast_tree({"w": w}, mpx.F16)["w"]
    (h * h).sum().backward()
    assert w.grad.dtype == torch.float32
    np.testing.assert_allclose(host(w.grad), 2 * O.quantize(np.float32([0.1, 3.0]), "f16"), rtol=1e-3)


# --------------------------------------------------- LossScaling scale/unscale
@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_scale_unscale_match_reference(cuda, golden, fmt):
    x = dev(f32(golden[f"su_{fmt}_x"]), fmt, cuda)
    for k, s in enumerate(golden["su_scales"]):
        for ls in (mpx.LossScaling(float(s)), mpx.DynamicLossScaling(float(s))):
            sc = ls.scale({"g": x})["g"]
            assert sc.dtype == x.dtype
            assert same_bits(host(sc), f32(golden[f"su_{fmt}_scaled_{k}"])), (fmt, s, type(ls))
            us = ls.unscale({"g": x})["g"]
            assert us.dtype == torch.float32
            assert same_bits(host(us), f32(golden[f"su_{fmt}_unscaled_{k}"])), (fmt, s, type(ls))


def test_scale_kats(cuda):
    # test_precision.py:142-177
    out = mpx.LossScaling(1024.0).scale({"g": mpx.tensor([0.5], mpx.F16)})["g"]
    assert out.dtype == torch.float16 and host(out).tolist() == [512.0]
    assert math.isinf(mpx.LossScaling(65536.0).scale({"g": mpx.tensor([2.0], mpx.F16)})["g"].item())
    u = mpx.LossScaling(1024.0).unscale({"g": mpx.tensor([512.0], mpx.F16)})["g"]
    assert u.dtype == torch.float32 and u.item() == 0.5
    assert math.isinf(mpx.LossScaling(1024.0).unscale({"g": mpx.tensor([np.inf], mpx.F16)})["g"].item())
    assert mpx.LossScaling(8.0).unscale({}) == {}


def test_unscale_overflow_is_flagged(cuda):
    # finite bf16 / 0.5 -> inf must count as non-finite
    g = [mpx.tensor([3.3e38], mpx.BF16)]
    outs, flag = K.unscale_finite(g, 0.5)
    assert math.isinf(outs[0].item()) and flag.item() == 0
    _, flag = K.unscale_finite(g, 0.5, write_f32=False)
    assert flag.item() == 0


# ---------------------------------------------------------------- K2 finite
@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_all_finite_positions(cuda, fmt):
    sizes = [5, 2048, 6000, 70001]
    for bad in ("inf", "-inf", "nan"):
        for li, n in enumerate(sizes):
            for pos in (0, n // 2, n - 1):
                leaves = {f"l{i}": torch.zeros(m, dtype=TORCH[fmt], device=cuda) for i, m in enumerate(sizes)}
                leaves[f"l{li}"][pos] = float(bad)
                assert mpx.all_finite(leaves) is False, (bad, li, pos)
    assert mpx.all_finite({"a": torch.ones(9000, dtype=TORCH[fmt], device=cuda), "k": mpx.tensor([1], mpx.I32)})
    assert mpx.all_finite({}) is True and mpx.all_finite({"s": "x"}) is True


# --------------------------------------------------------------- K3 adjust
def test_device_adjust_replays_reference(cuda, golden):
    flags = golden["adj_flags"]
    n_seq, T = flags.shape
    for i in range(n_seq):
        st = K.pack_scaling_state(golden["adj_inits"][i], golden["adj_gfs"][i], golden["adj_bfs"][i],
                                  int(golden["adj_intervals"][i]), 0, golden["adj_mins"][i], cuda)
        fl = torch.from_numpy(flags[i].astype(np.int32)).to(cuda)
        used = torch.empty(T, dtype=torch.float64, device=cuda)
        for t in range(T):
            K.N.check(K.N.load().mpx_scaling_adjust(st.data_ptr(), fl.data_ptr() + 4 * t, None,
                                                    used.data_ptr() + 8 * t, K.stream_handle(cuda)), "adjust")
        s = K.unpack_scaling_state(st)
        traj = np.append(used.cpu().numpy()[1:], s.loss_scale)
        assert np.array_equal(traj, golden["adj_scales"][i]), i
        assert s.steps_since_growth == golden["adj_counters"][i][-1]


def test_dynamic_loss_scaling_object(cuda):
    d = mpx.DynamicLossScaling(1024.0)
    d2 = d.adjust(False)
    assert d.loss_scale == 1024.0 and d2.loss_scale == 512.0 and d2.steps_since_growth == 0
    d3 = mpx.DynamicLossScaling(1024.0, growth_interval=2000, steps_since_growth=1999).adjust(True)
    assert d3.loss_scale == 2048.0 and d3.steps_since_growth == 0
    assert mpx.DynamicLossScaling(2.0 ** 127, growth_interval=1).adjust(True).loss_scale == 2.0 ** 127
    assert mpx.DynamicLossScaling(1.0).adjust(False).loss_scale == 1.0
    assert mpx.LossScaling(3.0, 1.5).to_device().to_host() == mpx.LossScaling(3.0, 1.5)


# ---------------------------------------------------------- K4 optimizer
@pytest.mark.parametrize("kind,variant", [("adam", "a"), ("adam", "b"), ("sgd", "a"), ("sgd", "b")])
@pytest.mark.parametrize("gate", ["host", "device"])
@pytest.mark.parametrize("donate", [False, True])
def test_optimizer_matches_reference(cuda, golden, kind, variant, gate, donate):
    lr = float(golden[f"opt_{kind}{variant}_lr"])
    fmts = ["f32", "f16", "f32", "f32"]
    keys = ["w", "h", "x", "y"]
    model = {k: dev(O.quantize(f32(golden[f"opt_p0_{j}"]), fmts[j]), fmts[j], cuda) for j, k in enumerate(keys)}
    state = mpx.adam_init(model, lr) if kind == "adam" else mpx.sgd_init(model, lr)
    finite = golden["opt_finite"]
    for k in range(len(finite)):
        grads = {key: dev(f32(golden[f"opt_g_{j}_s{k}"]), "f32", cuda) for j, key in enumerate(keys)}
        if gate == "host":
            fl = bool(finite[k])
        else:
            fl = mpx.DeviceBool(torch.tensor(int(finite[k]), dtype=torch.int32, device=cuda))
        m2, s2 = mpx.optimizer_update(model, state, grads, fl, donate=donate)
        if gate == "host" and not finite[k]:
            assert m2 is model and s2 is state
        model, state = m2, s2
        if f"opt_{kind}{variant}_p0_s{k}" not in golden:
            continue
        for j, key in enumerate(keys):
            assert model[key].dtype == TORCH[fmts[j]]
            assert same_bits(host(model[key]), f32(golden[f"opt_{kind}{variant}_p{j}_s{k}"])), (k, j)
            if kind == "adam":
                assert same_bits(host(state.mu[key]), f32(golden[f"opt_{kind}{variant}_m{j}_s{k}"])), (k, j)
                assert same_bits(host(state.nu[key]), f32(golden[f"opt_{kind}{variant}_v{j}_s{k}"])), (k, j)
        assert state.step_count == int(golden[f"opt_{kind}{variant}_count_s{k}"])


def test_fused_scaled_grads_equal_materialized(cuda):
    """K4 unscaling scaled half grads in-kernel == K2 materialise + K4 on f32."""
    rng = np.random.default_rng(5)
    shapes = [(300, 77), (4096,), (5,)]
    p = {f"p{i}": dev(rng.standard_normal(s).astype(np.float32) * 0.1, "f32", cuda) for i, s in enumerate(shapes)}
    for scale in (2.0 ** 15, 3.0, 0.375):
        for fmt in ("f16", "bf16"):
            gh = {k: dev(O.quantize(rng.standard_normal(v.shape).astype(np.float32) * 100, fmt), fmt, cuda)
                  for k, v in p.items()}
            s1 = mpx.adam_init(p, 1e-3)
            a, sa = mpx.optimizer_update(p, s1, mpx.LossScaling(scale).unscale(gh), True)
            b, sb = mpx.optimizer_update(p, s1, mpx.ScaledGrads(gh, scale), True)
            for k in p:
                assert same_bits(host(a[k]), host(b[k])) and same_bits(host(sa.mu[k]), host(sb.mu[k]))


def test_half_copy_written_in_same_pass(cuda):
    rng = np.random.default_rng(9)
    p = {"a": dev(rng.standard_normal(5000).astype(np.float32), "f32", cuda),
         "b": dev(rng.standard_normal(33).astype(np.float32), "f32", cuda)}
    for fmt in ("f16", "bf16"):
        half = {k: torch.empty_like(v, dtype=TORCH[fmt]) for k, v in p.items()}
        g = {k: torch.randn_like(v) for k, v in p.items()}
        new, _ = mpx.optimizer_update(p, mpx.adam_init(p, 1e-2), g, True, half_copy=half)
        for k in p:
            assert same_bits(host(half[k]), O.quantize(host(new[k]), fmt))


def test_gating_and_functional_semantics(cuda):
    model = {"w": mpx.tensor([1.0]), "k": mpx.tensor([3], mpx.I32), "name": "net"}
    state = mpx.adam_init(model, 0.1)
    m2, s2 = mpx.optimizer_update(model, state, {"w": mpx.tensor([np.inf]), "k": None, "name": None}, False)
    assert m2 is model and s2 is state and s2.step_count == 0
    # device-flag skip: nothing changes, bit for bit
    before = host(model["w"]).copy()
    flag = mpx.DeviceBool(torch.zeros((), dtype=torch.int32, device=cuda))
    m3, s3 = mpx.optimizer_update(model, state, {"w": mpx.tensor([np.nan]), "k": None, "name": None}, flag)
    assert same_bits(host(m3["w"]), before) and s3.step_count == 0
    assert host(s3.mu["w"]).tolist() == [0.0]
    # none-marker leaves untouched; compute_updates leaves its input alone
    sg = mpx.sgd_init(model, 0.1)
    m4, _ = mpx.optimizer_update(model, sg, {"w": mpx.tensor([1.0]), "k": None, "name": None}, True)
    assert m4["k"] is model["k"] and m4["name"] is model["name"]
    np.testing.assert_allclose(host(m4["w"]), [0.9], rtol=1e-7)
    upd, s5 = mpx.compute_updates(state, {"w": mpx.tensor([1.0]), "k": None, "name": None})
    assert state.step_count == 0 and s5.step_count == 1 and upd["k"] is None
    np.testing.assert_allclose(host(upd["w"]), [-0.1 / (1 + 1e-8)], rtol=1e-6)
    via_gate, _ = mpx.optimizer_update(model, state, {"w": mpx.tensor([1.0]), "k": None, "name": None}, True)
    assert same_bits(host(via_gate["w"]), host(model["w"]) + host(upd["w"]))
    with pytest.raises(mpx.TreeError):
        mpx.compute_updates(state, {"v": mpx.tensor([1.0])})
    with pytest.raises(ValueError):
        mpx.sgd_init({"k": mpx.tensor([1], mpx.I32)}, 0.1)


# ------------------------------------------------ filter_value_and_grad KATs
def _square(p, a):
    return p["w"] * p["w"]


@pytest.mark.parametrize("scaling_cls", [mpx.LossScaling, mpx.DynamicLossScaling])
def test_transform_simple_square(cuda, scaling_cls):
    res = mpx.filter_value_and_grad(_square, scaling_cls(1024.0))({"w": mpx.tensor(3.0)}, {})
    assert isinstance(res, mpx.GradResult)
    assert res.value.item() == 9.0 and res.value.dtype == torch.float32
    assert bool(res.grads_finite)
    assert res.grads["w"].dtype == torch.float32 and res.grads["w"].item() == 6.0
    assert res.scaling.steps_since_growth == 1 and res.scaling.loss_scale == 1024.0


@pytest.mark.parametrize("scaling_cls", [mpx.LossScaling, mpx.DynamicLossScaling])
def test_transform_overflow_backs_off(cuda, scaling_cls):
    f = lambda p, a: (p["w"] * 60000.0).sum()  # noqa: E731
    res = mpx.filter_value_and_grad(f, scaling_cls(65536.0))({"w": mpx.tensor([2.0])}, {})
    assert not bool(res.grads_finite) and not mpx.all_finite(res.grads)
    assert res.scaling.loss_scale == 32768.0 and res.scaling.steps_since_growth == 0
    for _, leaf in mpx.float_leaves(res.grads):
        assert leaf.dtype == torch.float32


def test_transform_host_contract_returns_python_bool(cuda):
    f = lambda p, a: (p["w"] * 60000.0).sum()  # noqa: E731
    res = mpx.filter_value_and_grad(f, mpx.LossScaling(65536.0))({"w": mpx.tensor([2.0])}, {})
    assert res.grads_finite is False


def test_transform_full_precision_passthrough(cuda):
    params = {"w": mpx.tensor([1.5, -2.0])}
    f = lambda p, a: (p["w"] * p["w"]).sum()  # noqa: E731
    scaling = mpx.LossScaling(4096.0, steps_since_growth=7)
    res = mpx.filter_value_and_grad(f, scaling, use_mixed_precision=False)(params, {})
    _, plain = mpx.value_and_grad(f, params, {})
    assert torch.equal(res.grads["w"], plain["w"]) and res.scaling is scaling and res.grads_finite


def test_transform_unused_leaf_and_half_selection(cuda):
    res = mpx.filter_value_and_grad(_square, mpx.LossScaling(8.0))(
        {"w": mpx.tensor(2.0), "idle": mpx.tensor([1.0], mpx.BF16)}, {})
    assert res.grads["idle"].dtype == torch.float32 and host(res.grads["idle"]).tolist() == [0.0]
    seen = []

    def f(p, a):
        seen.append(p["w"].dtype)
        return p["w"] * p["w"]

    with mpx.half_precision(mpx.BF16):
        tr = mpx.filter_value_and_grad(f, mpx.LossScaling(2.0))
    tr({"w": mpx.tensor(3.0)}, {})
    assert seen == [torch.bfloat16]


def test_transform_aux_value_and_filter_grad(cuda):
    def f(p, a):
        h = p["w"] * p["w"]
        return h.sum(), {"h": h}

    res = mpx.filter_value_and_grad(f, mpx.LossScaling(64.0), has_aux=True)({"w": mpx.tensor([2.0])}, {})
    assert res.aux["h"].dtype == torch.float16 and res.grads_finite
    r2 = mpx.filter_grad(_square, mpx.LossScaling(1024.0))({"w": mpx.tensor(3.0)}, {})
    assert r2.value is None and r2.grads["w"].item() == 6.0
    r3 = mpx.filter_value_and_grad(lambda p, a: (p["w"] * p["w"]).sum(), mpx.LossScaling(2.0))(
        {"w": mpx.tensor([np.nan])}, {})
    assert not r3.grads_finite
    with pytest.raises(ValueError):
        mpx.filter_value_and_grad(lambda p, a: p["w"] * 2, mpx.LossScaling(2.0))({"w": mpx.tensor([1.0, 2.0])}, {})


def test_transform_tape_hook_reports_activation_bytes(cuda):
    box = []
    mpx.filter_value_and_grad(lambda p, a: (torch.tanh(p["w"] @ a["x"])).sum(), mpx.LossScaling(8.0),
                              tape_hook=box.append)({"w": torch.randn(8, 16, device=cuda)},
                                                   {"x": torch.randn(16, 4, device=cuda)})
    assert box and box[0].activation_bytes() > 0


def test_mixed_vs_full_gradient_agreement(cuda):
    # test_precision.py:345-376 with torch ops on the half leaves
    rng = np.random.default_rng(42)
    widths = [6, 8, 4]
    params = {"layers": [{"w": mpx.tensor(rng.standard_normal((widths[i], widths[i + 1])) / math.sqrt(widths[i])),
                          "b": mpx.tensor(np.zeros(widths[i + 1]))} for i in range(2)]}
    x = mpx.tensor(rng.standard_normal((8, 6)))
    y = torch.from_numpy(rng.integers(0, 4, 8)).to(cuda)

    def loss(p, a):
        z = a["x"]
        for i, layer in enumerate(p["layers"]):
            z = z @ layer["w"] + layer["b"]
            if i == 0:
                z = torch.relu(z)
        return torch.nn.functional.cross_entropy(z.float(), a["y"])

    full = mpx.filter_value_and_grad(loss, mpx.LossScaling(2.0 ** 15), use_mixed_precision=False)(
        params, {"x": x, "y": y})
    mixed = mpx.filter_value_and_grad(loss, mpx.LossScaling(2.0 ** 15))(params, {"x": x, "y": y})
    assert mixed.grads_finite and full.grads_finite
    for (path, a), (_, b) in zip(mpx.float_leaves(full.grads), mpx.float_leaves(mixed.grads)):
        mag = host(a).__abs__().max()
        if mag <= 1e-4:
            continue
        assert np.abs(host(b) - host(a)).max() / mag <= 5e-2, path


def test_non_cuda_tensors_raise(cuda):
    with pytest.raises(Exception):
        mpx.cast_tree({"w": torch.ones(3)}, mpx.F16)


@pytest.mark.parametrize("gate", ["host", "device"])
def test_optimizer_accepts_mixed_gradient_formats(cuda, gate):
    """The reference's optimizer takes any float gradient leaves (optim.py:58-97):
    f32, f16 and bf16 gradients in one tree step with one t, and the step
    counter advances once per applied step (optim.py:77)."""
    rng = np.random.default_rng(9)
    fmts = {"a": "f16", "b": "bf16", "c": "f32", "d": "f16"}
    shapes = {"a": (33, 17), "b": (1000,), "c": (7, 3), "d": (64,)}
    p0 = {k: (rng.standard_normal(s) * 0.1).astype(np.float32) for k, s in shapes.items()}
    model = {k: dev(v, "f32", cuda) for k, v in p0.items()}
    state = mpx.adam_init(model, 1e-3)
    ref_p = dict(p0)
    ref_m = {k: np.zeros_like(v) for k, v in p0.items()}
    ref_v = {k: np.zeros_like(v) for k, v in p0.items()}
    t = 0
    for step, finite in enumerate([True, True, False, True]):
        g = {k: O.quantize((rng.standard_normal(s) * 0.01).astype(np.float32), fmts[k]) for k, s in shapes.items()}
        grads = {k: dev(g[k], fmts[k], cuda) for k in shapes}
        fl = finite if gate == "host" else mpx.DeviceBool(torch.tensor(int(finite), dtype=torch.int32, device=cuda))
        model, state = mpx.optimizer_update(model, state, grads, fl)
        if finite:
            t += 1
            for k in shapes:
                ref_p[k], ref_m[k], ref_v[k], _ = O.adam_leaf(ref_p[k], "f32", ref_m[k], ref_v[k], g[k], t, 1e-3)
        for k in shapes:
            assert same_bits(host(model[k]), ref_p[k]), (step, k)
            assert same_bits(host(state.mu[k]), ref_m[k]), (step, k)
        assert state.step_count == t
