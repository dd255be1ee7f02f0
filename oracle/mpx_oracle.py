"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's mixed-precision step (mpsim,
/root/reference/pkg/src/mpsim).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker or the timed CPU baseline — never as the product path.

Representation follows the reference: every value is a float32 numpy array;
a value "is" f16/bf16 when it sits on that grid (dtypes.py:1-21).

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by running the reference itself
(tests/golden/gen_golden.py imports mpsim from /root/reference), including
the reference's own known-answer tests and its exact-rational quantizer
tables.  Parity pinned for cast / scale / unscale / all_finite / adjust /
Adam / SGD; AdamW weight decay has no reference code (SPEC.md lists it as a
non-goal), so the wd != 0 branch is parity UNPINNED (restatement rule: the
decay term is added after the Adam term; wd == 0 takes the exact reference
path).
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

F16, BF16, F32 = "f16", "bf16", "f32"
F32_MAX = float(np.finfo(np.float32).max)


# ---------------------------------------------------------------------------
# dtypes.py:100-123 — quantize_array
# ---------------------------------------------------------------------------
def quantize(a, fmt: str) -> np.ndarray:
    """RNE onto the f16/bf16 grid, values kept as f32 (dtypes.py:100-123).
    f16: IEEE binary16 conversion (numpy's astype, dtypes.py:112-113);
    bf16: round the binary32 encoding on its top 16 bits, ties to even, a
    mantissa carry walking into the exponent = overflow to inf; NaN kept."""
    x = np.asarray(a, dtype=np.float32)
    if not x.flags.c_contiguous:
        x = np.ascontiguousarray(x)
    if fmt == F32:
        return x
    with np.errstate(over="ignore", invalid="ignore"):
        if fmt == F16:
            return x.astype(np.float16).astype(np.float32)
        if fmt != BF16:
            raise ValueError(f"unknown format {fmt!r}")
        u = x.view(np.uint32)
        r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
        return np.where(np.isnan(x), x, r.view(np.float32))


def to_half_bits(a, fmt: str) -> np.ndarray:
    """The 16-bit encoding of values already on a half grid (device layout)."""
    q = quantize(a, fmt)
    if fmt == F16:
        return q.astype(np.float16).view(np.uint16)
    return (q.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_half_bits(bits, fmt: str) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16)
    if fmt == F16:
        return b.view(np.float16).astype(np.float32)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


# ---------------------------------------------------------------------------
# precision.py:134-154 — LossScaling.scale / unscale;  tree.py:125-131
# ---------------------------------------------------------------------------
def scale(a, s: float, fmt: str) -> np.ndarray:
    """T.mul(leaf, s): f32 product of the payload and the weak scalar
    np.float32(s), rounded to the leaf's format (tensors.py:220-241)."""
    with np.errstate(all="ignore"):
        return quantize(np.asarray(a, np.float32) * np.float32(s), fmt)


def unscale(a, s: float) -> np.ndarray:
    """T.div(T.cast(leaf, F32), s): IEEE f32 division by np.float32(s)."""
    with np.errstate(all="ignore"):
        return np.asarray(a, np.float32) / np.float32(s)


def all_finite(arrays) -> bool:
    return all(bool(np.isfinite(a).all()) for a in arrays)


# ---------------------------------------------------------------------------
# precision.py:156-173 — LossScaling.adjust (Python double)
# state = (loss_scale, growth_factor, backoff_factor, growth_interval,
#          steps_since_growth, min_scale)
# ---------------------------------------------------------------------------
def adjust(state: tuple, finite: bool) -> tuple:
    s, gf, bf, interval, n, lo = state
    if not finite:
        s = s * bf
        if s < lo:
            s = lo
        n = 0
    elif n + 1 >= interval:
        g = s * gf
        if g <= F32_MAX:
            s = g
        n = 0
    else:
        n += 1
    return (s, gf, bf, interval, n, lo)


def simulate_scaling(init, gf, bf, interval, lo, flags) -> list[tuple[float, int]]:
    """(scale, counter) after each flag — the state machine above, iterated."""
    st = (float(init), gf, bf, interval, 0, lo)
    out = []
    for f in flags:
        st = adjust(st, bool(f))
        out.append((st[0], st[4]))
    return out


# ---------------------------------------------------------------------------
# optim.py:58-113 — compute_updates + optimizer_update
# ---------------------------------------------------------------------------
def bias_corrections(beta1: float, beta2: float, t: int) -> tuple[np.float32, np.float32]:
    """bc = 1.0 - b**t in Python double, used as a weak scalar -> np.float32
    (optim.py:73-76)."""
    return np.float32(1.0 - beta1 ** t), np.float32(1.0 - beta2 ** t)


def adam_leaf(p, p_fmt, m, v, g, t, lr, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0):
    """One Adam step of one leaf, f32 ops in the reference's order
    (optim.py:78-97 then apply_leaf optim.py:106-111).  Returns (p', m', v', u)."""
    f32 = np.float32
    with np.errstate(all="ignore"):
        g = np.asarray(g, f32)
        m1 = (np.asarray(m, f32) * f32(beta1)) + (g * f32(1.0 - beta1))
        v1 = (np.asarray(v, f32) * f32(beta2)) + ((g * g) * f32(1.0 - beta2))
        bc1, bc2 = bias_corrections(beta1, beta2, t)
        mh = m1 / bc1
        vh = v1 / bc2
        u = -((mh * f32(lr)) / (np.sqrt(vh) + f32(eps)))
        pn = np.asarray(p, f32) + u
        if wd:
            pn = pn + np.asarray(p, f32) * f32(-lr * wd)
        return quantize(pn, p_fmt), m1.astype(f32), v1.astype(f32), u.astype(f32)


def sgd_leaf(p, p_fmt, g, lr):
    """u = g * (-lr) (optim.py:60-66); p' = q(p + u)."""
    f32 = np.float32
    with np.errstate(all="ignore"):
        u = np.asarray(g, f32) * f32(-lr)
        return quantize(np.asarray(p, f32) + u, p_fmt), u.astype(f32)


def mp_step(params, p_fmts, m, v, g_half, state: tuple, step_count: int, lr: float, beta1=0.9,
            beta2=0.999, eps=1e-8, wd=0.0, half_fmt=None):
    """The reference's whole post-backward mixed-precision step over a list of
    leaves: unscale (precision.py:225) -> all_finite (:226) -> adjust (:227)
    -> gated Adam (optim.py:100-113).  Pure function; returns
    (params', m', v', state', step_count', finite, half_copy or None)."""
    s = state[0]
    g32 = [unscale(g, s) for g in g_half]
    finite = all_finite(g32)
    new_state = adjust(state, finite)
    if not finite:
        half = [quantize(p, half_fmt) for p in params] if half_fmt else None
        return list(params), list(m), list(v), new_state, step_count, False, half
    t = step_count + 1
    out_p, out_m, out_v = [], [], []
    for p, f, mm, vv, g in zip(params, p_fmts, m, v, g32):
        pn, m1, v1, _ = adam_leaf(p, f, mm, vv, g, t, lr, beta1, beta2, eps, wd)
        out_p.append(pn)
        out_m.append(m1)
        out_v.append(v1)
    half = [quantize(p, half_fmt) for p in out_p] if half_fmt else None
    return out_p, out_m, out_v, new_state, t, True, half


# ---------------------------------------------------------------------------
# CPU baseline driver: the same step over balanced leaf shards on a thread
# pool (numpy ufuncs release the GIL), flags AND-ed across shards.
# ---------------------------------------------------------------------------
def _balanced_shards(sizes, n_shards):
    order = sorted(range(len(sizes)), key=lambda i: -sizes[i])
    loads = [0] * n_shards
    shards = [[] for _ in range(n_shards)]
    for i in order:
        k = loads.index(min(loads))
        shards[k].append(i)
        loads[k] += sizes[i]
    return [sorted(s) for s in shards if s]


class ThreadedStep:
    """In-place (buffer-reusing) variant of mp_step for timing on many cores."""

    def __init__(self, params, m, v, n_threads: int, lr: float, beta1=0.9, beta2=0.999, eps=1e-8,
                 half_fmt=None):
        self.params, self.m, self.v = params, m, v
        self.half_fmt = half_fmt  # also produce the next step's half working copy (cast_tree, precision.py:209)
        self.half = [None] * len(params)
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.shards = _balanced_shards([p.size for p in params], max(1, n_threads))
        self.pool = ThreadPoolExecutor(max_workers=max(1, n_threads))
        self.n_threads = n_threads

    def step(self, g_half, state, step_count):
        s = state[0]

        def check(idx):
            return all(bool(np.isfinite(unscale(g_half[i], s)).all()) for i in idx)

        finite = all(self.pool.map(check, self.shards))
        new_state = adjust(state, finite)
        if not finite:
            return new_state, step_count, False
        t = step_count + 1

        def upd(idx):
            for i in idx:
                g = unscale(g_half[i], s)
                pn, m1, v1, _ = adam_leaf(self.params[i], F32, self.m[i], self.v[i], g, t, self.lr,
                                          self.beta1, self.beta2, self.eps)
                self.params[i], self.m[i], self.v[i] = pn, m1, v1
                if self.half_fmt:
                    self.half[i] = quantize(pn, self.half_fmt)
            return True

        list(self.pool.map(upd, self.shards))
        return new_state, t, True

    def close(self):
        self.pool.shutdown()


def vit_b16_leaf_shapes(num_classes: int = 1000, depth: int = 12, dim: int = 768, mlp: int = 3072,
                        patch: int = 16, img: int = 224, chans: int = 3):
    """(path, shape) of the ViT-B/16 pytree used by config 2:
    weights stored [fan_in, fan_out] and used as x @ W (bench.py:129-131)."""
    n_tok = (img // patch) ** 2 + 1
    shapes = [("patch.w", (patch * patch * chans, dim)), ("patch.b", (dim,)), ("cls", (1, dim)),
              ("pos", (n_tok, dim))]
    for i in range(depth):
        b = f"blocks.{i}."
        shapes += [(b + "ln1.g", (dim,)), (b + "ln1.b", (dim,)), (b + "qkv.w", (dim, 3 * dim)),
                   (b + "qkv.b", (3 * dim,)), (b + "proj.w", (dim, dim)), (b + "proj.b", (dim,)),
                   (b + "ln2.g", (dim,)), (b + "ln2.b", (dim,)), (b + "fc1.w", (dim, mlp)), (b + "fc1.b", (mlp,)),
                   (b + "fc2.w", (mlp, dim)), (b + "fc2.b", (dim,))]
    shapes += [("ln_f.g", (dim,)), ("ln_f.b", (dim,)), ("head.w", (dim, num_classes)),
               ("head.b", (num_classes,))]
    return shapes


def n_params(shapes) -> int:
    return int(sum(math.prod(s) for _, s in shapes))
