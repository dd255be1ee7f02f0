"""Generate tests/golden/mpstep_golden.npz by running the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/gen_golden.py
The reference cannot travel to the GPU box, so its outputs are committed as
fixtures; tests compare both the CPU oracle (oracle/mpx_oracle.py) and the
CUDA path against them.  Every block names the reference test it extends.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import mpsim  # noqa: E402
from mpsim import BF16, F16, F32, LossScaling, adam_init, optimizer_update, sgd_init, tensor  # noqa: E402
from mpsim.dtypes import quantize_array  # noqa: E402
from oracles import boundary_values, ref_quantize, simulate_scaling_batch  # noqa: E402

OUT = Path(__file__).resolve().parent / "mpstep_golden.npz"
SAVED_STEPS = (0, 2, 3, 5, 8)  # first, both skips, the step after a skip, last


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint32)


def main():
    g: dict[str, np.ndarray] = {}

    # -- 1. quantization tables (test_acceptance.py:70-85 C1; test_dtypes.py:72-87)
    rng = np.random.default_rng(20240801)
    rand = rng.integers(0, 2 ** 32, size=10_000, dtype=np.uint32).view(np.float32)
    for fmt, dt in (("f16", F16), ("bf16", BF16)):
        vals = np.concatenate([rand, np.asarray(boundary_values(fmt), dtype=np.float32)])
        g[f"quant_{fmt}_in"] = bits(vals)
        g[f"quant_{fmt}_out"] = bits(quantize_array(vals, dt))
        g[f"quant_{fmt}_exact"] = bits([ref_quantize(float(v), fmt) for v in vals])

    # -- 2. scale / unscale (test_precision.py:142-177, 246-254)
    rng = np.random.default_rng(7)
    scales = [1.0, 2.0 ** 15, 2.0 ** -3, 1024.0, 3.0, 0.75, 1e-3, 2.0 ** 127, 2.0 ** -140, 65536.0 * 1.5]
    base = (rng.standard_normal(1024) * np.exp(rng.uniform(-12, 12, 1024))).astype(np.float32)
    base[:8] = [np.inf, -np.inf, np.nan, 0.0, -0.0, 65504.0, 3.3e38, 1e-45]
    g["su_scales"] = np.asarray(scales, dtype=np.float64)
    for fmt, dt in (("f16", F16), ("bf16", BF16), ("f32", F32)):
        x = tensor(base, dt)
        g[f"su_{fmt}_x"] = bits(x.payload)
        for k, s in enumerate(scales):
            ls = LossScaling(s)
            g[f"su_{fmt}_scaled_{k}"] = bits(ls.scale({"g": x})["g"].payload)
            g[f"su_{fmt}_unscaled_{k}"] = bits(ls.unscale({"g": x})["g"].payload)

    # -- 3. loss-scale state machine (test_acceptance.py:165-206 C4 recipe, subset)
    n_seq, length = 32, 1500
    rng = np.random.default_rng(1717)
    inits = rng.choice([1.0, 2.0 ** 15, 2.0 ** 20, 2.0 ** 120, 2.0 ** 126], size=n_seq)
    intervals = rng.choice([1, 2, 3, 5, 100, 2000], size=n_seq)
    gfs = rng.choice([2.0, 4.0, 1.5], size=n_seq, p=[0.6, 0.2, 0.2])
    bfs = rng.choice([0.5, 0.25, 0.75], size=n_seq, p=[0.6, 0.2, 0.2])
    mins = rng.choice([1.0, 0.25, 2.0 ** -10], size=n_seq)
    inits[0], intervals[0], gfs[0], bfs[0], mins[0] = 2.0 ** 126, 1, 2.0, 0.5, 1.0
    inits[1], intervals[1], gfs[1], bfs[1], mins[1] = 1.0, 2, 2.0, 0.5, 1.0
    inits[2], intervals[2] = 2.0 ** 15, 2000
    prob = rng.choice([0.0, 0.5, 0.9, 0.99, 1.0], size=n_seq)
    flags = rng.random((n_seq, length)) < prob[:, None]
    flags[0, :] = True
    flags[1, :] = False
    ref_s, ref_c = simulate_scaling_batch(inits, gfs, bfs, intervals, mins, flags)
    # and the reference implementation itself
    got_s = np.empty_like(ref_s)
    got_c = np.empty_like(ref_c)
    for i in range(n_seq):
        st = LossScaling(float(inits[i]), float(gfs[i]), float(bfs[i]), int(intervals[i]), 0, float(mins[i]))
        for t, f in enumerate(flags[i].tolist()):
            st = st.adjust(f)
            got_s[i, t], got_c[i, t] = st.loss_scale, st.steps_since_growth
    assert np.array_equal(got_s, ref_s) and np.array_equal(got_c, ref_c)
    g.update(adj_inits=inits, adj_intervals=intervals, adj_gfs=gfs, adj_bfs=bfs, adj_mins=mins,
             adj_flags=flags, adj_scales=got_s, adj_counters=got_c)

    # -- 4. Adam / SGD over multi-leaf trees incl. skipped steps and an f16
    #       master leaf (test_optim.py:50-173, test_acceptance.py:230-254)
    rng = np.random.default_rng(31)
    shapes = [(3, 5), (1061,), (2, 2048), (7,)]
    p0 = [rng.standard_normal(s).astype(np.float32) * 0.05 for s in shapes]
    n_steps = 9
    grads = [[(rng.standard_normal(s) * 10 ** rng.uniform(-4, 1)).astype(np.float32) for s in shapes]
             for _ in range(n_steps)]
    finite = [True, True, False, True, True, False, True, True, True]
    for k, fl in enumerate(finite):
        if not fl:
            grads[k][1][17] = np.inf if k == 2 else np.nan
    for kind in ("adam", "sgd"):
        for variant, lr in (("a", 1e-3), ("b", 0.05)):
            model = {"w": tensor(p0[0]), "h": tensor(p0[1], F16), "x": tensor(p0[2]), "y": tensor(p0[3])}
            order = ["w", "h", "x", "y"]
            state = adam_init(model, lr) if kind == "adam" else sgd_init(model, lr)
            for k in range(n_steps):
                gt = {key: tensor(grads[k][j]) for j, key in enumerate(order)}
                model, state = optimizer_update(model, state, gt, finite[k])
                if k not in SAVED_STEPS:
                    continue
                for j, key in enumerate(order):
                    g[f"opt_{kind}{variant}_p{j}_s{k}"] = bits(model[key].payload)
                    if kind == "adam":
                        g[f"opt_{kind}{variant}_m{j}_s{k}"] = bits(state.mu[key].payload)
                        g[f"opt_{kind}{variant}_v{j}_s{k}"] = bits(state.nu[key].payload)
                g[f"opt_{kind}{variant}_count_s{k}"] = np.asarray(state.step_count)
            g[f"opt_{kind}{variant}_lr"] = np.asarray(lr)
    for j, p in enumerate(p0):
        g[f"opt_p0_{j}"] = bits(p)
        for k in range(n_steps):
            g[f"opt_g_{j}_s{k}"] = bits(grads[k][j])
    g["opt_finite"] = np.asarray(finite)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays, mpsim {mpsim.__version__})")


if __name__ == "__main__":
    main()
