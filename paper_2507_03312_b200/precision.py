"""MPX API: tree casting, precision islands, dynamic loss scaling and the
mixed-precision gradient transform (mirror of mpsim.precision).

    set/get_half_precision, half_precision   precision.py:27-50
    cast_tree + cast_to_* aliases            precision.py:53-85   -> K1
    cast_function, force_full_precision      precision.py:88-114  -> K1 (+ autograd)
    LossScaling (host, Python-double)        precision.py:120-173 -> K1 / K2 for scale / unscale
    DynamicLossScaling (device-resident)     PAPER.md:111-121     -> K1 / K2 / K3, no host sync
    GradResult, filter_value_and_grad,
    filter_grad                              precision.py:176-245 -> torch.autograd + K1/K2/K3

Semantics follow the reference exactly: the loss is scaled in its own dtype
(T.mul(loss, s), precision.py:213-219), gradients come back unscaled in f32
(precision.py:225), finiteness is judged on the unscaled f32 values
(precision.py:226), and the reported value is f32(scaled_loss)/f32(s)
(precision.py:228).
"""
from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import kernels as K
from .dtypes import BF16, F16, F32, DType, Scalar, as_dtype, dtype_of, is_float_leaf, quantize_host_scalar
from .tensors import _note
from .tree import tree_leaves, tree_map

_HALF: DType = F16


def set_half_precision(dtype):
    """Select the process-wide half format, F16 (default) or BF16."""
    global _HALF
    d = as_dtype(dtype)
    if d not in (F16, BF16):
        raise ValueError("half precision must be f16 or bf16")
    _HALF = d


def get_half_precision() -> DType:
    return _HALF


@contextmanager
def half_precision(dtype):
    prev = get_half_precision()
    set_half_precision(dtype)
    try:
        yield
    finally:
        set_half_precision(prev)


# ---------------------------------------------------------------------------
# casting
# ---------------------------------------------------------------------------
class _CastLeaves(torch.autograd.Function):
    """Differentiable multi-leaf cast; backward casts each cotangent back to
    its input's dtype (autodiff.py:279-280), also with K1."""

    @staticmethod
    def forward(ctx, dst_code, *leaves):
        ctx.in_dtypes = [t.dtype for t in leaves]
        dst = {0: torch.float32, 1: torch.float16, 2: torch.bfloat16}[dst_code]
        outs = [torch.empty(t.shape, dtype=dst, device=t.device) for t in leaves]
        K.cast_into(leaves, outs)
        return tuple(_keep_type(o, t) for o, t in zip(outs, leaves))

    @staticmethod
    def backward(ctx, *grads):
        res = [None]
        srcs, dsts, slots = [], [], []
        for g, dt in zip(grads, ctx.in_dtypes):
            if g is None:
                res.append(None)
                continue
            out = torch.empty(g.shape, dtype=dt, device=g.device)
            srcs.append(g.contiguous())
            dsts.append(out)
            res.append(out)
        K.cast_into(srcs, dsts)
        return tuple(res)


def _cast_tensor_leaves(leaves: list[torch.Tensor], d: DType) -> list[torch.Tensor]:
    if not leaves:
        return []
    if torch.is_grad_enabled() and any(t.requires_grad for t in leaves):
        return list(_CastLeaves.apply(d.code, *leaves))
    return [_keep_type(o, t) for o, t in zip(K.cast_leaves(leaves, d), leaves)]


def _keep_type(out: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """A result stays a tensors.Tensor (the reference's operator sugar) when its source was one."""
    from .tensors import Tensor

    return out.as_subclass(Tensor) if isinstance(src, Tensor) and not isinstance(out, Tensor) else out


def cast_tree(t, dtype):
    """Re-round every float tensor leaf to `dtype` (precision.py:53-69).

    Integer tensors, weak scalars and opaque leaves come back as the same
    objects; strong float Scalars are re-rounded.  Leaves already of `dtype`
    are returned as-is (values are unchanged, as torch's `.to` does)."""
    d = as_dtype(dtype)
    if not d.is_float:
        raise ValueError("cast target must be a float dtype")
    todo = []
    seen = set()
    for x in tree_leaves(t):
        if is_float_leaf(x) and dtype_of(x) is not d and id(x) not in seen:
            seen.add(id(x))
            todo.append(x)
    outs = dict(zip(map(id, todo), _cast_tensor_leaves(todo, d)))

    from .tensors import _note  # a tape entry per float leaf (T.cast records even same-format casts)

    def leaf(x):
        if is_float_leaf(x):
            return _note(outs.get(id(x), x))
        if isinstance(x, Scalar) and not x.weak and x.dtype.is_float:
            return Scalar(quantize_host_scalar(x.value, d), weak=False, dtype=d)
        return x

    return tree_map(leaf, t)


def cast_to_float16(x):
    return cast_tree(x, F16)


def cast_to_bfloat16(x):
    return cast_tree(x, BF16)


def cast_to_float32(x):
    return cast_tree(x, F32)


def cast_to_half_precision(x):
    return cast_tree(x, get_half_precision())


def cast_function(f, dtype, return_dtype=None):
    """Wrap f: cast call arguments to `dtype`, outputs to `return_dtype`
    (precision.py:88-103).  Closure-captured tensors are not cast."""
    d = as_dtype(dtype)
    if not d.is_float:
        raise ValueError("cast target must be a float dtype")
    rd = as_dtype(return_dtype) if return_dtype is not None else None
    if rd is not None and not rd.is_float:
        raise ValueError("return dtype must be a float dtype")

    def wrapped(*args, **kwargs):
        cargs, ckwargs = cast_tree((args, kwargs), d)
        out = f(*cargs, **ckwargs)
        return out if rd is None else cast_tree(out, rd)

    return wrapped


def force_full_precision(f, return_dtype):
    """Run f in f32 whatever the input precision, cast outputs to return_dtype
    (precision.py:106-114)."""
    if return_dtype is None:
        raise ValueError("force_full_precision needs a return dtype")
    return cast_function(f, F32, return_dtype)


# ---------------------------------------------------------------------------
# loss scaling
# ---------------------------------------------------------------------------
_F32_MAX = float(np.finfo(np.float32).max)


def _float_leaf_positions(t):
    return [x for x in tree_leaves(t) if is_float_leaf(x)]


def _substitute(t, mapping: dict):
    return tree_map(lambda x: mapping.get(id(x), x) if is_float_leaf(x) else x, t)


def _scale_tree(t, scale: float = 1.0, d_scale: torch.Tensor | None = None):
    leaves = list({id(x): x for x in _float_leaf_positions(t)}.values())
    outs = [torch.empty_like(x, memory_format=torch.contiguous_format) for x in leaves]
    K.cast_into(leaves, outs, scale, d_scale)
    return _substitute(t, {id(x): _keep_type(o, x) for x, o in zip(leaves, outs)})


def _unscale_tree(t, scale: float = 1.0, d_scale: torch.Tensor | None = None):
    leaves = list({id(x): x for x in _float_leaf_positions(t)}.values())
    outs, flag = K.unscale_finite(leaves, scale, d_scale, write_f32=True)
    return _substitute(t, {id(x): _keep_type(o, x) for x, o in zip(leaves, outs)}), flag


class LossScaling(NamedTuple):
    """Dynamic loss-scaling state as an immutable host value (precision.py:120-173).

    `adjust` is the reference's Python-double state machine; `scale` and
    `unscale` run on the device (K1 / K2)."""

    loss_scale: float
    growth_factor: float = 2.0
    backoff_factor: float = 0.5
    growth_interval: int = 2000
    steps_since_growth: int = 0
    min_scale: float = 1.0

    def scale(self, t):
        """Every float leaf times the scale, rounded to the leaf's own dtype."""
        return _scale_tree(t, self.loss_scale)

    def unscale(self, t):
        """Float leaves to f32, then divided by the scale (IEEE division)."""
        return _unscale_tree(t, self.loss_scale)[0]

    def adjust(self, grads_finite) -> "LossScaling":
        """Back off on overflow, grow after `growth_interval` finite steps."""
        scale, gf, bf, interval, n, lo = self
        if not bool(grads_finite):
            scale = scale * bf
            if scale < lo:
                scale = lo
            n = 0
        elif n + 1 >= interval:
            grown = scale * gf
            scale = grown if grown <= _F32_MAX else scale
            n = 0
        else:
            n += 1
        return tuple.__new__(LossScaling, (scale, gf, bf, interval, n, lo))

    def to_device(self, device=None) -> "DynamicLossScaling":
        return DynamicLossScaling(*self, device=device)


class DeviceBool:
    """A finite flag that lives on the device.  `bool(x)` synchronises; the
    optimizer consumes the device word directly, so a training loop that
    never calls bool() never syncs."""

    __slots__ = ("tensor",)

    def __init__(self, tensor: torch.Tensor):
        self.tensor = tensor

    def __bool__(self):
        return bool(self.tensor.item())

    def __eq__(self, other):
        if isinstance(other, (bool, np.bool_, DeviceBool)):
            return bool(self) == bool(other)
        return NotImplemented

    def __hash__(self):
        return hash(bool(self))

    def __repr__(self):
        return f"DeviceBool({bool(self)})"


class DynamicLossScaling:
    """Device-resident loss-scaling state (the MPX `DynamicLossScaling`,
    PAPER.md:111-121): the six reference fields packed as mpx_scaling_state
    in 48 bytes of device memory.  scale/unscale read the scale on the
    device; adjust runs K3 on a copy of the state, so values stay immutable
    like the reference's NamedTuple and no step ever waits for the host."""

    def __init__(self, loss_scale: float = 2.0 ** 15, growth_factor: float = 2.0, backoff_factor: float = 0.5,
                 growth_interval: int = 2000, steps_since_growth: int = 0, min_scale: float = 1.0, *,
                 device=None, _state: torch.Tensor | None = None):
        self.growth_factor = float(growth_factor)
        self.backoff_factor = float(backoff_factor)
        self.growth_interval = int(growth_interval)
        self.min_scale = float(min_scale)
        if _state is None:
            dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
            _state = K.pack_scaling_state(loss_scale, growth_factor, backoff_factor, growth_interval,
                                          steps_since_growth, min_scale, dev)
        self.state = _state

    # device views ------------------------------------------------------
    @property
    def d_scale(self) -> torch.Tensor:
        """float64 view of state.loss_scale (the first field)."""
        return self.state[:8].view(torch.float64)

    @property
    def device(self):
        return self.state.device

    # host views (synchronising) -----------------------------------------
    def to_host(self) -> LossScaling:
        s = K.unpack_scaling_state(self.state)
        return LossScaling(s.loss_scale, s.growth_factor, s.backoff_factor, s.growth_interval,
                           s.steps_since_growth, s.min_scale)

    @property
    def loss_scale(self) -> float:
        return self.to_host().loss_scale

    @property
    def steps_since_growth(self) -> int:
        return self.to_host().steps_since_growth

    # MPX methods ---------------------------------------------------------
    def scale(self, t):
        return _scale_tree(t, d_scale=self.d_scale)

    def unscale(self, t):
        return _unscale_tree(t, d_scale=self.d_scale)[0]

    def adjust(self, grads_finite) -> "DynamicLossScaling":
        if isinstance(grads_finite, DeviceBool):
            flag = grads_finite.tensor
        elif isinstance(grads_finite, torch.Tensor):
            flag = grads_finite
        else:
            flag = torch.full((), int(bool(grads_finite)), dtype=torch.int32, device=self.device)
        new = DynamicLossScaling(0.0, self.growth_factor, self.backoff_factor, self.growth_interval, 0,
                                 self.min_scale, _state=self.state.clone())
        K.scaling_adjust(new.state, flag)
        return new

    def __repr__(self):
        return f"DynamicLossScaling({self.to_host()})"


# ---------------------------------------------------------------------------
# the gradient transform
# ---------------------------------------------------------------------------
@dataclass
class GradResult:
    """scaling after adjust, finiteness, f32 grads shaped like params, aux, and
    the unscaled f32 loss (precision.py:176-186)."""

    scaling: object
    grads_finite: object
    grads: object
    aux: object = None
    value: torch.Tensor | None = None


class ScaledGrads:
    """Scaled half-precision gradients with the scale that produced them —
    the input of the fused optimizer path (unscale folded into K4).
    `unscale()` gives the reference's f32 tree."""

    def __init__(self, tree, scale: float = 1.0, d_scale: torch.Tensor | None = None):
        self.tree = tree
        self.scale = scale
        self.d_scale = d_scale

    def unscale(self):
        return _unscale_tree(self.tree, self.scale, self.d_scale)[0]


class _ScaleLoss(torch.autograd.Function):
    """y = round_{dtype(x)}(x * f32(s)); dy/dx cotangent c -> round(c * f32(s))
    (T.mul with a weak scalar and its backward rule, autodiff.py:131-138)."""

    @staticmethod
    def forward(ctx, x, scale, d_scale):
        ctx.scale, ctx.d_scale = scale, d_scale
        out = torch.empty_like(x)
        K.cast_into([x], [out], scale, d_scale)
        return out

    @staticmethod
    def backward(ctx, c):
        out = torch.empty_like(c)
        K.cast_into([c.contiguous()], [out], ctx.scale, ctx.d_scale)
        return out, None, None


class ActivationTape:
    """Stand-in for the reference Tape handed to tape_hook (autodiff.py:34-45):
    records the tensors autograd saves for backward during the forward, so
    `activation_bytes()` is the analytic activation footprint."""

    def __init__(self):
        self._seen: dict[tuple, int] = {}
        self._outputs = 0  # bytes of the drop-in tensor ops' outputs (the reference's tape entries)
        self._n_outputs = 0

    def note_output(self, t):
        """A drop-in tensor op produced `t` (tensors._note): the reference's
        tape entry (tensors.py:173-180), counted at its nominal width."""
        if isinstance(t, torch.Tensor):
            self._outputs += t.numel() * t.element_size()
            self._n_outputs += 1

    def pack(self, t: torch.Tensor):
        if isinstance(t, torch.Tensor) and t.device.type != "meta":
            key = (t.untyped_storage().data_ptr(), t.storage_offset(), tuple(t.shape), t.dtype)
            self._seen[key] = t.numel() * t.element_size()
        return t

    @staticmethod
    def unpack(t):
        return t

    def activation_bytes(self) -> int:
        """The reference's definition (autodiff.py:43-45: every forward
        intermediate on the tape) when the forward ran on the drop-in tensor
        ops; otherwise (the fused ViT engine) the tensors autograd saved."""
        if self._n_outputs:
            return int(self._outputs)
        return int(sum(self._seen.values()))


def value_and_grad(f, params, args, has_aux: bool = False, *, tape_hook=None):
    """(value, grads[, aux]) of f(params, args) w.r.t. the float leaves of
    params (autodiff.py:332-366): unused float leaves get zeros of their
    dtype, non-float leaves get None; args are never differentiated."""
    leaves = [x for x in tree_leaves(params) if is_float_leaf(x)]
    uniq = list({id(x): x for x in leaves}.values())
    live = {id(x): x.detach().requires_grad_(True) for x in uniq}
    p = tree_map(lambda x: live.get(id(x), x) if is_float_leaf(x) else x, params)
    tape = ActivationTape()
    from .tensors import recording

    with torch.enable_grad(), torch.autograd.graph.saved_tensors_hooks(tape.pack, tape.unpack), recording(tape):
        out = f(p, args)
    if has_aux:
        try:
            loss, aux = out
        except (TypeError, ValueError) as exc:
            raise ValueError("has_aux function must return (loss, aux)") from exc
    else:
        loss, aux = out, None
    if not is_float_leaf(loss):
        raise ValueError("differentiated function must return a float tensor")
    if loss.dim() != 0:
        raise ValueError(f"differentiated function must return a scalar, got shape {tuple(loss.shape)}")
    if tape_hook is not None:
        tape_hook(tape)
    inputs = list(live.values())
    if loss.requires_grad and inputs:
        gs = torch.autograd.grad(loss, inputs, allow_unused=True)
    else:
        gs = [None] * len(inputs)
    gmap = {}
    for x, g in zip(uniq, gs):
        gmap[id(x)] = g.detach() if g is not None else torch.zeros_like(x)
    grads = tree_map(lambda x: gmap[id(x)] if is_float_leaf(x) else None, params)
    value = loss.detach()
    return (value, grads, aux) if has_aux else (value, grads)


def grad(f, params, args, has_aux: bool = False):
    res = value_and_grad(f, params, args, has_aux=has_aux)
    return (res[1], res[2]) if has_aux else res[1]


def filter_value_and_grad(f, scaling, has_aux: bool = False, use_mixed_precision: bool = True, *,
                          tape_hook=None, materialize_grads: bool = True):
    """Mixed-precision value-and-grad transform (precision.py:189-231).

    `scaling` is a LossScaling (host state: grads_finite comes back as a
    Python bool, one 4-byte sync per call — the reference's contract) or a
    DynamicLossScaling (device state: grads_finite is a DeviceBool, nothing
    syncs).  With materialize_grads=False the result's `grads` is a
    ScaledGrads (half grads + scale) that optimizer_update unscales inside
    its fused pass instead of materialising f32 gradients."""
    half = get_half_precision()
    on_device = isinstance(scaling, DynamicLossScaling)

    def transformed(params, args) -> GradResult:
        if not use_mixed_precision:
            p32 = cast_tree(params, F32)
            a32 = cast_tree(args, F32)
            res = value_and_grad(f, p32, a32, has_aux=has_aux, tape_hook=tape_hook)
            value, grads = res[0], res[1]
            aux = res[2] if has_aux else None
            flag = K.all_finite_flag(_float_leaf_positions(grads))
            finite = DeviceBool(flag) if on_device else bool(flag.item())
            v32 = cast_tree(value, F32)
            return GradResult(scaling, finite, grads, aux, v32)

        params_h = cast_tree(params, half)
        args_h = cast_tree(args, half)
        s = 1.0 if on_device else float(scaling.loss_scale)
        d_s = scaling.d_scale if on_device else None

        if has_aux:
            def scaled_f(p, a):
                loss, aux = f(p, a)
                return _note(_ScaleLoss.apply(loss, s, d_s)), aux
        else:
            def scaled_f(p, a):
                return _note(_ScaleLoss.apply(f(p, a), s, d_s))

        res = value_and_grad(scaled_f, params_h, args_h, has_aux=has_aux, tape_hook=tape_hook)
        scaled_value, grads_h = res[0], res[1]
        aux = res[2] if has_aux else None
        if materialize_grads:
            grads, flag = _unscale_tree(grads_h, s, d_s)
        else:
            leaves = list({id(x): x for x in _float_leaf_positions(grads_h)}.values())
            _, flag = K.unscale_finite(leaves, s, d_s, write_f32=False)
            grads = ScaledGrads(grads_h, s, d_s)
        (value,), _ = K.unscale_finite([scaled_value], s, d_s, write_f32=True)
        if on_device:
            finite = DeviceBool(flag)
            new_scaling = scaling.adjust(flag)
        else:
            finite = bool(flag.item())
            new_scaling = scaling.adjust(finite)
        return GradResult(new_scaling, finite, grads, aux, value)

    return transformed


def filter_grad(f, scaling, has_aux: bool = False, use_mixed_precision: bool = True, *, tape_hook=None,
                materialize_grads: bool = True):
    """filter_value_and_grad without the value (precision.py:234-245)."""
    inner = filter_value_and_grad(f, scaling, has_aux=has_aux, use_mixed_precision=use_mixed_precision,
                                  tape_hook=tape_hook, materialize_grads=materialize_grads)

    def transformed(params, args) -> GradResult:
        r = inner(params, args)
        return GradResult(r.scaling, r.grads_finite, r.grads, r.aux, None)

    return transformed
