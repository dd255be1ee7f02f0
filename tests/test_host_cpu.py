"""Host-side logic that runs without a GPU: the C ABI library loads and
exports every declared symbol, the dtype lattice, pytree algebra, the host
loss-scale state machine, the host-side rounding of hyper-parameters, and
that nothing silently falls back to the CPU."""
import math
import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2507_03312_b200 as mpx
from paper_2507_03312_b200 import _native
from paper_2507_03312_b200 import kernels as K
from oracle import mpx_oracle as O

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "mpx_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 7
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} declared in mpx_b200.h but not bound in _native.py"
    assert lib.mpx_version() >= 1


def test_struct_layouts_match_header():
    import ctypes

    assert ctypes.sizeof(_native.ScalingStateC) == 48
    assert ctypes.sizeof(_native.AdamHParamsC) == 32
    assert K.SCALING_STATE_BYTES == 48


def test_native_errors_are_raised_not_swallowed():
    lib = _native.load()
    rc = lib.mpx_cast(None, None, None, 1, 7, 0, 1.0, None, None)
    assert rc != 0
    with pytest.raises(_native.NativeError, match="bad dtype"):
        _native.check(rc, "mpx_cast")


# ------------------------------------------------------------------ dtypes
JOIN = {("f16", "f16"): "f16", ("f16", "bf16"): "f32", ("f16", "f32"): "f32", ("f16", "i32"): "f16",
        ("bf16", "bf16"): "bf16", ("bf16", "f32"): "f32", ("bf16", "i32"): "bf16", ("f32", "f32"): "f32",
        ("f32", "i32"): "f32", ("i32", "i32"): "i32"}


def test_promotion_lattice():
    # oracles.py:127-144 join table, both orders
    for (a, b), w in JOIN.items():
        assert mpx.promote(mpx.DType(a), mpx.DType(b)) is mpx.DType(w)
        assert mpx.promote(mpx.DType(b), mpx.DType(a)) is mpx.DType(w)
    ds = list(mpx.DType)
    for a in ds:
        for b in ds:
            for c in ds:
                assert mpx.promote(mpx.promote(a, b), c) is mpx.promote(a, mpx.promote(b, c))


def test_scalars_and_metadata():
    assert mpx.promote_with_scalar(mpx.F16, mpx.Scalar(2.0)) is mpx.F16
    assert mpx.promote_with_scalar(mpx.F16, mpx.Scalar(0.5, weak=False, dtype=mpx.F32)) is mpx.F32
    assert mpx.promote_with_scalar(mpx.F16, mpx.Scalar(1, weak=False)) is mpx.F16
    assert mpx.Scalar(1.5, weak=False).dtype is mpx.F32 and mpx.Scalar(2, weak=False).dtype is mpx.I32
    assert mpx.F16.byte_width == 2 and mpx.F32.byte_width == 4 and not mpx.I32.is_float
    assert mpx.as_dtype(torch.bfloat16) is mpx.BF16 and mpx.as_dtype("f16") is mpx.F16


def test_host_scalar_quantize_matches_oracle():
    rng = np.random.default_rng(0)
    vals = rng.integers(0, 2 ** 32, 2000, dtype=np.uint32).view(np.float32)
    from paper_2507_03312_b200.dtypes import quantize_host_scalar

    for fmt in ("f16", "bf16"):
        for v in vals[:500]:
            got = quantize_host_scalar(float(v), mpx.DType(fmt))
            want = float(O.quantize(np.float32(v), fmt))
            assert (math.isnan(got) and math.isnan(want)) or np.float32(got).view(np.uint32) == np.float32(
                want).view(np.uint32)


# -------------------------------------------------------------------- trees
def test_tree_map_and_errors():
    t = {"a": [1, 2], "b": (3, {"c": 4})}
    assert mpx.tree_map(lambda x: x * 10, t) == {"a": [10, 20], "b": (30, {"c": 40})}
    assert mpx.tree_leaves(t) == [1, 2, 3, 4]
    with pytest.raises(mpx.TreeError, match="b.1.c"):
        mpx.tree_map(lambda x: 1 / (x - 4), t)
    with pytest.raises(mpx.TreeError, match="diverge"):
        mpx.tree_zip_map(lambda a, b: a, {"a": 1}, {"b": 1})
    with pytest.raises(mpx.TreeError, match="lengths"):
        mpx.tree_zip_map(lambda a, b: a, [1, 2], [1])
    with pytest.raises(mpx.TreeError, match="node kinds"):
        mpx.tree_zip_map(lambda a, b: a, [1], (1,))
    assert mpx.tree_structure({"x": [1, (2,)]}) == ("dict", ("x",), (("list", ("leaf", ("tuple", ("leaf",)))),))


def test_float_leaves_and_format():
    t = {"w": torch.zeros(2), "k": torch.zeros(2, dtype=torch.int32), "h": [torch.ones(1, dtype=torch.float16)],
         "s": "x"}
    assert [p for p, _ in mpx.float_leaves(t)] == ["w", "h.0"]
    txt = mpx.format_tree({"w": torch.tensor([1.0, 2.0]), "n": [1, "a"], "e": {}})
    assert txt == "w: tensor f32[2] [1.0, 2.0]\nn:\n  - 1\n  - 'a'\ne:\n  {}\n"


# ----------------------------------------------------- host loss scaling
def test_host_adjust_replays_reference(golden):
    flags = golden["adj_flags"]
    for i in range(flags.shape[0]):
        st = mpx.LossScaling(float(golden["adj_inits"][i]), float(golden["adj_gfs"][i]),
                             float(golden["adj_bfs"][i]), int(golden["adj_intervals"][i]), 0,
                             float(golden["adj_mins"][i]))
        s, c = [], []
        for f in flags[i].tolist():
            st = st.adjust(f)
            s.append(st.loss_scale)
            c.append(st.steps_since_growth)
        assert np.array_equal(s, golden["adj_scales"][i]) and np.array_equal(c, golden["adj_counters"][i])


def test_host_adjust_kats():
    assert mpx.LossScaling(1024.0).adjust(False) == (512.0, 2.0, 0.5, 2000, 0, 1.0)
    assert mpx.LossScaling(1024.0, steps_since_growth=1999).adjust(True).loss_scale == 2048.0
    assert mpx.LossScaling(1024.0).adjust(True).steps_since_growth == 1
    assert mpx.LossScaling(2.0 ** 127, growth_interval=1).adjust(True).loss_scale == 2.0 ** 127
    s = mpx.LossScaling(1.0, growth_interval=1)
    rng = np.random.default_rng(0)
    for f in rng.random(200) < 0.7:
        s = s.adjust(bool(f))
        assert math.frexp(s.loss_scale)[0] == 0.5


# ------------------------------------------- hyper-parameter rounding
def test_adam_hparams_round_like_weak_scalars():
    hp = K.adam_hparams(1e-3, 0.9, 0.999, 1e-8, 0.0)
    assert np.float32(hp.omb1) == np.float32(1.0 - 0.9) == np.float32(0.1)
    assert np.float32(hp.omb2) == np.float32(1.0 - 0.999)
    assert np.float32(hp.lr) == np.float32(1e-3) and hp.neg_lr_wd == 0.0


def test_bias_correction_table_matches_oracle():
    tab = K.bias_correction_table(0.9, 0.999, "cpu").numpy().reshape(-1, 2)
    for t in (1, 2, 3, 10, 100, 1000, 5000, len(tab)):
        a, b = O.bias_corrections(0.9, 0.999, t)
        assert tab[t - 1, 0] == a and tab[t - 1, 1] == b
    assert tab[-1, 0] == 1.0 and tab[-1, 1] == 1.0  # clamping beyond the end is exact


# --------------------------------------------------------- no CPU fallback
def test_cpu_tensors_are_rejected():
    with pytest.raises(TypeError, match="CUDA"):
        K.cast_leaves([torch.ones(4)], mpx.F16)
    with pytest.raises(TypeError, match="CUDA"):
        K.unscale_finite([torch.ones(4, dtype=torch.float16)], 2.0)


def test_package_has_no_oracle_imports():
    pkg = ROOT / "paper_2507_03312_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", f.read_text(), flags=re.M), f


# the reference's public surface, pkg/src/mpsim/__init__.py:10-30 (Tape /
# TapeEntry are the reference's own autodiff engine: torch.autograd replaces
# it)
REFERENCE_NAMES = [
    "grad", "value_and_grad", "BF16", "DType", "F16", "F32", "I32", "Scalar", "promote", "promote_with_scalar",
    "quantize", "quantize_array", "OptimizerState", "adam_init", "compute_updates", "optimizer_update", "sgd_init",
    "GradResult", "LossScaling", "cast_function", "cast_to_bfloat16", "cast_to_float16", "cast_to_float32",
    "cast_to_half_precision", "cast_tree", "filter_grad", "filter_value_and_grad", "force_full_precision",
    "get_half_precision", "half_precision", "set_half_precision", "Tensor", "bytes_of", "cross_entropy",
    "elementwise", "layernorm", "matmul", "reduce", "softmax", "tensor", "TreeError", "all_finite", "float_leaves",
    "format_tree", "tree_leaves", "tree_map", "tree_structure", "tree_zip_map",
]
# mpsim.tensors (the `T` namespace the reference's models use, tensors.py:104-555)
REFERENCE_T_NAMES = ["Tensor", "tensor", "zeros", "zeros_like", "ones", "bytes_of", "add", "sub", "mul", "div", "neg",
                     "exp", "log", "sqrt", "relu", "gelu", "elementwise", "reduce", "matmul", "softmax", "layernorm",
                     "cross_entropy", "cast", "reshape", "transpose"]


def test_drop_in_names_exported():
    import paper_2507_03312_b200 as mpx
    from paper_2507_03312_b200 import tensors as T

    missing = [n for n in REFERENCE_NAMES if not hasattr(mpx, n)]
    assert not missing, missing
    missing = [n for n in REFERENCE_T_NAMES if not hasattr(T, n)]
    assert not missing, missing
    assert issubclass(mpx.Tensor, __import__("torch").Tensor)
    assert mpx.DynamicLossScaling is not None  # the paper's name for LossScaling


def test_drop_in_ops_refuse_cpu_tensors():
    import torch

    from paper_2507_03312_b200 import tensors as T

    x = torch.ones(2, 2).as_subclass(T.Tensor)
    with pytest.raises(Exception):
        T.add(x, x)
    with pytest.raises(Exception):
        x @ x
