"""Pin the CPU oracle to the reference: every oracle function against the
golden vectors produced by running mpsim itself (tests/golden/gen_golden.py)
and against the reference's own known-answer tests."""
import math

import numpy as np
import pytest

from oracle import mpx_oracle as O


def f32(bits):
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def same_bits(a, b):
    """bitwise equality, NaN compared by class (test_dtypes.py:27-30)."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    nan = np.isnan(a) & np.isnan(b)
    return bool(np.all(nan | (a.view(np.uint32) == b.view(np.uint32))))


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
def test_quantize_matches_reference_tables(golden, fmt):
    x = f32(golden[f"quant_{fmt}_in"])
    got = O.quantize(x, fmt)
    assert same_bits(got, f32(golden[f"quant_{fmt}_out"]))
    # and the reference's exact-rational quantizer (oracles.py:34-67)
    assert same_bits(got, f32(golden[f"quant_{fmt}_exact"]))


@pytest.mark.parametrize("value,fmt,expected", [
    (1.0, "f16", 1.0), (100000.0, "f16", math.inf), (2.0 ** -25, "f16", 0.0),
    (0.2, "bf16", 0.2001953125), (65504.0, "f16", 65504.0), (65520.0, "f16", math.inf),
    (-0.0, "f16", -0.0), (math.inf, "bf16", math.inf),
])
def test_quantize_reference_kats(value, fmt, expected):
    # test_dtypes.py:40-52
    assert same_bits(O.quantize(np.float32(value), fmt), np.float32(expected))


def test_half_bits_round_trip():
    x = np.float32([1.0, -2.5, 65504.0, 2.0 ** -24, np.inf])
    for fmt in ("f16", "bf16"):
        q = O.quantize(x, fmt)
        assert same_bits(O.from_half_bits(O.to_half_bits(q, fmt), fmt), q)


@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_scale_unscale_match_reference(golden, fmt):
    x = f32(golden[f"su_{fmt}_x"])
    for k, s in enumerate(golden["su_scales"]):
        assert same_bits(O.scale(x, s, fmt), f32(golden[f"su_{fmt}_scaled_{k}"])), (fmt, s)
        assert same_bits(O.unscale(x, s), f32(golden[f"su_{fmt}_unscaled_{k}"])), (fmt, s)


def test_adjust_replays_reference_trajectories(golden):
    flags = golden["adj_flags"]
    for i in range(flags.shape[0]):
        traj = O.simulate_scaling(golden["adj_inits"][i], golden["adj_gfs"][i], golden["adj_bfs"][i],
                                  int(golden["adj_intervals"][i]), golden["adj_mins"][i], flags[i])
        assert np.array_equal([s for s, _ in traj], golden["adj_scales"][i])
        assert np.array_equal([c for _, c in traj], golden["adj_counters"][i])


def test_adjust_kats():
    # test_precision.py:180-221
    st = (1024.0, 2.0, 0.5, 2000, 0, 1.0)
    assert O.adjust(st, False)[0] == 512.0
    assert O.adjust((1024.0, 2.0, 0.5, 2000, 1999, 1.0), True)[:5:4] == (2048.0, 0)
    assert O.adjust((1.0, 2.0, 0.5, 2000, 0, 1.0), False)[0] == 1.0
    assert O.adjust((2.0 ** 127, 2.0, 0.5, 1, 0, 1.0), True)[0] == 2.0 ** 127
    assert O.adjust((2.0 ** 126, 2.0, 0.5, 1, 0, 1.0), True)[0] == 2.0 ** 127


@pytest.mark.parametrize("kind,variant", [("adam", "a"), ("adam", "b"), ("sgd", "a"), ("sgd", "b")])
def test_optimizer_matches_reference(golden, kind, variant):
    lr = float(golden[f"opt_{kind}{variant}_lr"])
    fmts = ["f32", "f16", "f32", "f32"]
    p = [O.quantize(f32(golden[f"opt_p0_{j}"]), fmts[j]) for j in range(4)]
    m = [np.zeros_like(x) for x in p]
    v = [np.zeros_like(x) for x in p]
    finite = golden["opt_finite"]
    t = 0
    for k in range(len(finite)):
        g = [f32(golden[f"opt_g_{j}_s{k}"]) for j in range(4)]
        if finite[k]:
            t += 1
            for j in range(4):
                if kind == "adam":
                    p[j], m[j], v[j], _ = O.adam_leaf(p[j], fmts[j], m[j], v[j], g[j], t, lr)
                else:
                    p[j], _ = O.sgd_leaf(p[j], fmts[j], g[j], lr)
        key = f"opt_{kind}{variant}_p0_s{k}"
        if key not in golden:
            continue
        for j in range(4):
            assert same_bits(p[j], f32(golden[f"opt_{kind}{variant}_p{j}_s{k}"])), (k, j)
            if kind == "adam":
                assert same_bits(m[j], f32(golden[f"opt_{kind}{variant}_m{j}_s{k}"])), (k, j)
                assert same_bits(v[j], f32(golden[f"opt_{kind}{variant}_v{j}_s{k}"])), (k, j)
        assert int(golden[f"opt_{kind}{variant}_count_s{k}"]) == t


def test_adam_first_step_closed_form():
    # test_optim.py:58-67
    p, m, v, u = O.adam_leaf(np.float32([1.0]), "f32", np.zeros(1, np.float32), np.zeros(1, np.float32),
                             np.float32([1.0]), 1, 0.1)
    np.testing.assert_allclose(u, [-0.1 / (1 + 1e-8)], rtol=1e-6)
    np.testing.assert_allclose(m, [0.1], rtol=1e-6)
    np.testing.assert_allclose(v, [0.001], rtol=1e-5)


def test_mp_step_skips_and_backs_off():
    p = [np.ones(4, np.float32)]
    g = [np.float32([1.0, np.inf, 0.0, 2.0])]
    out = O.mp_step(p, ["f32"], [np.zeros(4, np.float32)], [np.zeros(4, np.float32)], g,
                    (1024.0, 2.0, 0.5, 2000, 5, 1.0), 3, 1e-3)
    assert out[5] is False and out[4] == 3 and out[3][0] == 512.0 and out[3][4] == 0
    assert same_bits(out[0][0], p[0])


def test_vit_b16_pytree_size():
    shapes = O.vit_b16_leaf_shapes()
    assert len(shapes) == 152 and O.n_params(shapes) == 86_567_656
