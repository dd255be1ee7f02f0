"""The reference's tensor layer (mpsim.tensors, the `T` namespace its models
are written against) on the device.

    from paper_2507_03312_b200 import tensors as T     # was: from mpsim import tensors as T

`Tensor` is a torch.Tensor subclass whose operators (+ - * / unary -, @, .T)
call this module's functions, so a model written for mpsim — e.g.
`attention_forward` (pkg/src/mpsim/bench.py:172-208) — runs unchanged on a
B200, differentiably (torch.autograd drives the backward rules below, which
restate autodiff.py:94-290).  Every arithmetic op runs in libmpx_b200.so:

    elementwise add/sub/mul/div/neg/exp/log/sqrt/relu/gelu   mpx_ew           tensors.py:220-324
    reduce sum/mean/max                                      mpx_reduce       tensors.py:353-384
    matmul (f16/bf16 with TMA-addressable operands)          mpx_gemm (tcgen05, f32 accumulate)
    matmul (f32, mixed formats, other strides)               mpx_matmul_simt  tensors.py:387-422
    softmax / layernorm / cross_entropy                      mpx_softmax_axis / mpx_layernorm_ref / mpx_xent_*
    cast / quantize_array                                    mpx_cast (K1)    tensors.py:529-538, dtypes.py:100-128

Values are physically stored in their format (2 bytes for f16/bf16).  Each
op evaluates in f32 and rounds once onto the result format; accumulations
are the reference's stepwise ones (see csrc/mpx_ops.cu).  There is no CPU
fallback: non-CUDA operands raise.

Differences from mpsim's Tensor, all forced by torch.Tensor: `dtype` is the
torch dtype (`dtype_of(t)` gives the DType), `size()` is torch's method
(`t.numel()` is the reference's `t.size`), and the payload is on the device
(`t.payload` copies it to a host f32 / i32 numpy array).
"""
from __future__ import annotations

import ctypes
import math
import threading

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from .dtypes import F32, I32, DType, Scalar, as_dtype, dtype_of, promote, promote_with_scalar

_MAX_I32 = 2 ** 31 - 1
_MIN_I32 = -(2 ** 31)
_FLOATS = (torch.float16, torch.bfloat16, torch.float32)


class Tensor(torch.Tensor):
    """A device tensor with the reference's operator sugar (tensors.py:38-101)."""

    __torch_function__ = torch._C._disabled_torch_function_impl

    def __add__(self, other):
        return add(self, other)

    __radd__ = __add__

    def __sub__(self, other):
        return sub(self, other)

    def __rsub__(self, other):
        return sub(other, self)

    def __mul__(self, other):
        return mul(self, other)

    __rmul__ = __mul__

    def __truediv__(self, other):
        return div(self, other)

    def __rtruediv__(self, other):
        return div(other, self)

    def __neg__(self):
        return neg(self)

    def __matmul__(self, other):
        return matmul(self, other)

    def __rmatmul__(self, other):
        return matmul(other, self)

    @property
    def T(self):  # noqa: N802 - the reference's name
        return transpose(self)

    @property
    def payload(self) -> np.ndarray:
        """Host copy in the reference's payload convention (f32 on the grid / i32)."""
        t = self.detach()
        return (t.float() if t.is_floating_point() else t).cpu().numpy()

    def __repr__(self) -> str:
        d = dtype_of(self)
        return f"Tensor({d.value if d else self.dtype}{list(self.shape)} on {self.device})"


def _wrap(t: torch.Tensor) -> Tensor:
    return t if isinstance(t, Tensor) else t.as_subclass(Tensor)


# the reference's tape records every primitive's output (tensors.py:173-180,
# _record); Tape.activation_bytes sums bytes_of over them (autodiff.py:43-45).
# precision.value_and_grad installs an ActivationTape here while the forward
# runs, and every public op below reports its output to it.
_REC = threading.local()


def _note(out):
    rec = getattr(_REC, "tape", None)
    if rec is not None:
        rec.note_output(out)
    return out


class recording:
    """Context manager: route op outputs to `tape.note_output` (thread-local)."""

    def __init__(self, tape):
        self.tape = tape

    def __enter__(self):
        self.prev = getattr(_REC, "tape", None)
        _REC.tape = self.tape
        return self.tape

    def __exit__(self, *exc):
        _REC.tape = self.prev


def _device(device):
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


# ---------------------------------------------------------------- constructors
def quantize_array(values, dtype) -> np.ndarray:
    """Round an array onto a float dtype's grid (dtypes.py:100-123), on the
    device (K1); returns a host f32 array like the reference.  bf16 keeps the
    input's NaN payloads as the reference does (dtypes.py:122-123)."""
    d = as_dtype(dtype)
    if not d.is_float:
        raise ValueError("integers are never quantized")
    a = np.asarray(values, dtype=np.float32)
    if d is F32 or a.size == 0:
        return a
    dev = _device(None)
    src = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev)
    out = K.cast_leaves([src], d)[0].float().cpu().numpy().reshape(a.shape)
    return np.where(np.isnan(a), a, out) if d.value == "bf16" else out


def quantize(value: float, dtype) -> float:
    """Scalar wrapper around quantize_array (dtypes.py:126-128)."""
    return float(quantize_array(np.float32(value), dtype))


def tensor(data, dtype=F32, device=None) -> Tensor:
    """Build a device tensor quantized onto the dtype's grid (tensors.py:104-111)."""
    d = as_dtype(dtype)
    dev = _device(device)
    if not d.is_float:
        arr = np.asarray(data, dtype=np.int64)
        if arr.size and (arr.max() > _MAX_I32 or arr.min() < _MIN_I32):
            raise ValueError("value out of 32-bit signed integer range")
        return _wrap(torch.from_numpy(arr.astype(np.int32)).to(dev))
    f32 = torch.from_numpy(np.array(data, dtype=np.float32, order="C")).to(dev)
    if d is F32:
        return _wrap(f32)
    return _wrap(K.cast_leaves([f32], d)[0])


def zeros(shape, dtype=F32, device=None) -> Tensor:
    return _wrap(torch.zeros(shape, dtype=as_dtype(dtype).torch, device=_device(device)))


def zeros_like(t) -> Tensor:
    return _wrap(torch.zeros(t.shape, dtype=t.dtype, device=t.device))


def ones(shape, dtype=F32, device=None) -> Tensor:
    return _wrap(torch.ones(shape, dtype=as_dtype(dtype).torch, device=_device(device)))


def bytes_of(t: torch.Tensor) -> int:
    """Footprint at the nominal precision (tensors.py:130-132)."""
    d = dtype_of(t)
    return t.numel() * (d.byte_width if d is not None else t.element_size())


# ---------------------------------------------------------------- raw device ops (no autograd)
def _code(t_or_dtype) -> int:
    dt = t_or_dtype.dtype if isinstance(t_or_dtype, torch.Tensor) else t_or_dtype
    return as_dtype(dt).code


def _i64(values):
    arr = (ctypes.c_int64 * max(len(values), 1))(*[int(v) for v in values])
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64)), arr


def _ew(op: int, a: torch.Tensor, b=None, *, scalar: float = 0.0, side: int = 0, out_dtype=None,
        grad_dtype=None) -> Tensor:
    """out = op(a, b | scalar) over the broadcast shape, strided operands."""
    shape = tuple(torch.broadcast_shapes(a.shape, b.shape)) if isinstance(b, torch.Tensor) else tuple(a.shape)
    if len(shape) > 8:
        raise ValueError("elementwise ops support up to 8 dimensions")
    od = out_dtype if out_dtype is not None else a.dtype
    out = torch.empty(shape, dtype=od, device=a.device)
    if out.numel() == 0:
        return _wrap(out)
    ae = a.expand(shape)
    sp, _k0 = _i64(shape)
    sa, _k1 = _i64(ae.stride())
    if isinstance(b, torch.Tensor):
        be = b.expand(shape)
        sb, _k2 = _i64(be.stride())
        bptr, bcode = be.data_ptr(), _code(be)
    else:
        sb, bptr, bcode = None, None, N.MPX_F32
    N.check(N.load().mpx_ew(op, len(shape), sp, out.data_ptr(), _code(od), ae.data_ptr(), _code(ae), sa, bptr, bcode,
                            sb, float(scalar), int(side), _code(grad_dtype if grad_dtype is not None else od),
                            K.stream_handle(a.device)), "mpx_ew")
    return _wrap(out)


def _cast_to(t: torch.Tensor, dtype) -> Tensor:
    """Round onto another format (a contiguous copy when the format matches)."""
    if t.dtype == dtype and t.is_contiguous():
        return _wrap(t)
    return _ew(N.MPX_EW_COPY, t, out_dtype=dtype)


def _contig(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_contiguous() else _ew(N.MPX_EW_COPY, t)


def _split(shape, ax):
    outer = math.prod(shape[:ax])
    return outer, shape[ax], math.prod(shape[ax + 1:])


def _reduce_raw(op: int, a: torch.Tensor, ax: int) -> Tensor:
    a = _contig(a)
    outer, n, inner = _split(tuple(a.shape), ax)
    out = torch.empty(tuple(a.shape[:ax]) + tuple(a.shape[ax + 1:]), dtype=a.dtype, device=a.device)
    N.check(N.load().mpx_reduce(op, a.data_ptr(), _code(a), outer, n, inner, out.data_ptr(), _code(a),
                                K.stream_handle(a.device)), "mpx_reduce")
    return _wrap(out)


def _unbroadcast(c: torch.Tensor, shape) -> torch.Tensor:
    """Sum a cotangent down to a broadcast operand's shape (autodiff.py:92-99)."""
    shape = tuple(shape)
    while c.ndim > len(shape):
        c = _reduce_raw(N.MPX_RED_SUM, c, 0)
    for ax, n in enumerate(shape):
        if n == 1 and c.shape[ax] != 1:
            c = _reduce_raw(N.MPX_RED_SUM, c, ax).view(c.shape[:ax] + (1,) + c.shape[ax + 1:])
    return c


def _grad_for(g: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    """torch autograd wants a cotangent in the input's own format."""
    return _cast_to(g, like.dtype) if g.dtype != like.dtype else g


# ---- matmul
def _tma_ok(t: torch.Tensor) -> bool:
    return t.data_ptr() % 16 == 0 and all(s % 8 == 0 for s in t.stride()[:-2])


def _mm_layout(t: torch.Tensor, k_axis: int):
    """(ld, mn_major) when TMA can read the 2-D slices, else None.  k_axis is
    -1 for A ([.., M, K]) and -2 for B ([.., K, N])."""
    s_last, s_prev = t.stride(-1), t.stride(-2)
    if t.shape[-1] > 1 and t.shape[-2] > 1 and s_last == 1 and s_prev % 8 == 0:
        return s_prev, k_axis == -2  # rows contiguous: K-major for A, MN-major for B
    if t.shape[-1] > 1 and t.shape[-2] > 1 and s_prev == 1 and s_last % 8 == 0:
        return s_last, k_axis == -1
    return None


def _mm_raw(A: torch.Tensor, B: torch.Tensor, out_dtype: torch.dtype) -> Tensor:
    """[.., M, K] @ [.., K, N] with broadcast leading dims, any strides."""
    lead = tuple(torch.broadcast_shapes(A.shape[:-2], B.shape[:-2]))
    M, Kd, Nn = A.shape[-2], A.shape[-1], B.shape[-1]
    Ae, Be = A.expand(lead + (M, Kd)), B.expand(lead + (Kd, Nn))
    out = torch.empty(lead + (M, Nn), dtype=out_dtype, device=A.device)
    if out.numel() == 0:
        return _wrap(out)
    if Kd == 0:
        return _wrap(out.zero_())
    la, lb = _mm_layout(Ae, -1), _mm_layout(Be, -2)
    use_tc = (A.dtype == B.dtype == out_dtype and A.dtype in (torch.float16, torch.bfloat16) and len(lead) <= 2
              and la is not None and lb is not None and _tma_ok(Ae) and _tma_ok(Be) and Kd % 8 == 0
              and Nn % 8 == 0)
    if use_tc:
        from . import vit_kernels as VK

        nb = tuple(reversed(lead)) + (1,) * (2 - len(lead))  # nb1 = innermost batch dim
        def sbs(t):
            s = tuple(reversed(t.stride()[:len(lead)]))
            return s + (0,) * (2 - len(s))
        VK.gemm(Ae, Be, M=M, N=Nn, K=Kd, lda=la[0], ldb=lb[0], a_mn=la[1], b_mn=lb[1], out=out, ldc=Nn,
                nb=nb, a_sb=sbs(Ae), b_sb=sbs(Be), c_sb=sbs(out))
        return _wrap(out)
    if len(lead) > 4:
        raise ValueError("matmul supports up to 4 broadcast batch dimensions")
    st, _k0 = _i64([Ae.stride(-2), Ae.stride(-1), Be.stride(-2), Be.stride(-1), out.stride(-2), out.stride(-1)])
    bs, _k1 = _i64(lead)
    sa, _k2 = _i64(Ae.stride()[:len(lead)])
    sb, _k3 = _i64(Be.stride()[:len(lead)])
    sc, _k4 = _i64(out.stride()[:len(lead)])
    N.check(N.load().mpx_matmul_simt(Ae.data_ptr(), _code(Ae), Be.data_ptr(), _code(Be), out.data_ptr(),
                                     _code(out_dtype), M, Nn, Kd, st, len(lead), bs, sa, sb, sc,
                                     K.stream_handle(A.device)), "mpx_matmul_simt")
    return _wrap(out)


def _swap_last(t: torch.Tensor) -> torch.Tensor:
    return t.transpose(-1, -2)


# ---------------------------------------------------------------- operand checks
def _as_operand(x):
    if isinstance(x, (torch.Tensor, Scalar)):
        return x
    if isinstance(x, (bool,)):
        raise TypeError("cannot use bool as an operand")
    if isinstance(x, (int, float, np.integer, np.floating)):
        return Scalar(float(x))
    raise TypeError(f"cannot use {type(x).__name__} as an operand")


def _require_float(t: torch.Tensor, op: str):
    if t.dtype not in _FLOATS:
        raise TypeError(f"{op} requires float tensors, got {dtype_of(t).value if dtype_of(t) else t.dtype}")
    K.require_cuda([t], op)


# ---------------------------------------------------------------- elementwise (autograd)
_BIN = {"add": N.MPX_EW_ADD, "sub": N.MPX_EW_SUB, "mul": N.MPX_EW_MUL, "div": N.MPX_EW_DIV}


class _Binary(torch.autograd.Function):
    @staticmethod
    def forward(ctx, name, a, b, scalar, side, out_dtype):
        ctx.name, ctx.scalar, ctx.side = name, scalar, side
        t = a if a is not None else b
        ctx.shapes = (a.shape if a is not None else None, b.shape if b is not None else None)
        ctx.save_for_backward(a if a is not None else t.new_empty(0), b if b is not None else t.new_empty(0))
        ctx.has = (a is not None, b is not None)
        if a is not None and b is not None:
            return _ew(_BIN[name], a, b, out_dtype=out_dtype)
        return _ew(_BIN[name], t, scalar=scalar, side=side, out_dtype=out_dtype)

    @staticmethod
    def backward(ctx, c):
        a, b = ctx.saved_tensors
        has_a, has_b = ctx.has
        name, s = ctx.name, ctx.scalar
        ga = gb = None
        # the reference's rules (autodiff.py:102-150); `x` is a tensor operand or the weak scalar s
        A = a if has_a else None
        B = b if has_b else None

        def mul_(x, y):
            if isinstance(y, torch.Tensor):
                return _ew(N.MPX_EW_MUL, x, y, out_dtype=_ptype(x, y))
            return _ew(N.MPX_EW_MUL, x, scalar=y)

        def div_(x, y, rev=False):
            if isinstance(y, torch.Tensor):
                return _ew(N.MPX_EW_DIV, x, y, out_dtype=_ptype(x, y))
            return _ew(N.MPX_EW_DIV, x, scalar=y, side=int(rev))

        other_a = A if has_a else s
        other_b = B if has_b else s
        if name == "add":
            ga, gb = c, c
        elif name == "sub":
            ga, gb = c, _ew(N.MPX_EW_NEG, c)
        elif name == "mul":
            ga, gb = mul_(c, other_b), mul_(c, other_a)
        else:  # div: d/da = c / b; d/db = -(c * a) / (b * b)
            ga = div_(c, other_b)
            if has_b:
                num = mul_(c, other_a)
                den = _ew(N.MPX_EW_MUL, B, B)
                gb = _ew(N.MPX_EW_NEG, _ew(N.MPX_EW_DIV, num, den, out_dtype=_ptype(num, den)))
        outs = []
        for idx, (has, g, t, shp) in enumerate(((has_a, ga, A, ctx.shapes[0]), (has_b, gb, B, ctx.shapes[1]))):
            if not has or g is None or not ctx.needs_input_grad[1 + idx]:
                outs.append(None)
                continue
            outs.append(_grad_for(_unbroadcast(g, shp), t))
        return None, outs[0], outs[1], None, None, None


def _ptype(x: torch.Tensor, y: torch.Tensor) -> torch.dtype:
    return promote(dtype_of(x), dtype_of(y)).torch


def _binary(name: str, a, b) -> Tensor:
    a, b = _as_operand(a), _as_operand(b)
    ta, tb = isinstance(a, torch.Tensor), isinstance(b, torch.Tensor)
    if ta:
        _require_float(a, name)
    if tb:
        _require_float(b, name)
    if ta and tb:
        out = promote(dtype_of(a), dtype_of(b))
        return _note(_Binary.apply(name, a, b, 0.0, 0, out.torch))
    if ta:
        out = promote_with_scalar(dtype_of(a), b)
        return _note(_Binary.apply(name, a, None, b.value, 0, out.torch))
    if tb:
        out = promote_with_scalar(dtype_of(b), a)
        return _note(_Binary.apply(name, None, b, a.value, 1, out.torch))
    raise TypeError(f"{name} needs at least one tensor operand")


def add(a, b) -> Tensor:
    return _binary("add", a, b)


def sub(a, b) -> Tensor:
    return _binary("sub", a, b)


def mul(a, b) -> Tensor:
    return _binary("mul", a, b)


def div(a, b) -> Tensor:
    return _binary("div", a, b)


_UN = {"neg": N.MPX_EW_NEG, "exp": N.MPX_EW_EXP, "log": N.MPX_EW_LOG, "sqrt": N.MPX_EW_SQRT,
       "relu": N.MPX_EW_RELU, "gelu": N.MPX_EW_GELU}


class _Unary(torch.autograd.Function):
    @staticmethod
    def forward(ctx, name, a):
        out = _ew(_UN[name], a)
        ctx.name = name
        ctx.save_for_backward(a, out)
        return out

    @staticmethod
    def backward(ctx, c):
        a, y = ctx.saved_tensors
        n = ctx.name
        if n == "neg":
            g = _ew(N.MPX_EW_NEG, c)
        elif n == "exp":
            g = _ew(N.MPX_EW_MUL, c, y, out_dtype=_ptype(c, y))
        elif n == "log":
            g = _ew(N.MPX_EW_DIV, c, a, out_dtype=_ptype(c, a))
        elif n == "sqrt":
            h = _ew(N.MPX_EW_MUL, c, scalar=0.5)
            g = _ew(N.MPX_EW_DIV, h, y, out_dtype=_ptype(h, y))
        elif n == "relu":
            g = _ew(N.MPX_EW_RELU_BWD, c, a, out_dtype=c.dtype)
        else:
            g = _ew(N.MPX_EW_GELU_BWD, c, a, out_dtype=c.dtype, grad_dtype=c.dtype)
        return None, _grad_for(g, a)


def _unary(name: str, a) -> Tensor:
    if not isinstance(a, torch.Tensor):
        raise TypeError(f"{name} expects a tensor")
    _require_float(a, name)
    return _note(_Unary.apply(name, a))


def neg(a) -> Tensor:
    return _unary("neg", a)


def exp(a) -> Tensor:
    return _unary("exp", a)


def log(a) -> Tensor:
    return _unary("log", a)


def sqrt(a) -> Tensor:
    return _unary("sqrt", a)


def relu(a) -> Tensor:
    return _unary("relu", a)


def gelu(a) -> Tensor:
    return _unary("gelu", a)


_ELEMENTWISE = {"add": add, "sub": sub, "mul": mul, "div": div, "neg": neg, "exp": exp, "log": log, "sqrt": sqrt,
                "relu": relu, "gelu": gelu}


def elementwise(op_code: str, a, b=None) -> Tensor:
    """Dispatch an elementwise op by name (tensors.py:309-324)."""
    if op_code not in _ELEMENTWISE:
        raise ValueError(f"unknown elementwise op {op_code!r}")
    if op_code in _BIN:
        if b is None:
            raise TypeError(f"{op_code} is binary")
        return _ELEMENTWISE[op_code](a, b)
    if b is not None:
        raise TypeError(f"{op_code} is unary")
    return _ELEMENTWISE[op_code](a)


# ---------------------------------------------------------------- reductions
def _normalize_axis(axis: int, ndim: int, op: str) -> int:
    if not -ndim <= axis < ndim:
        raise ValueError(f"{op}: axis {axis} out of range for {ndim}-d tensor")
    return axis % ndim


class _Reduce(torch.autograd.Function):
    @staticmethod
    def forward(ctx, op, a, axis):
        x = _contig(a).reshape(-1) if axis is None else a
        ax = 0 if axis is None else axis
        code = {"sum": N.MPX_RED_SUM, "mean": N.MPX_RED_MEAN, "max": N.MPX_RED_MAX}[op]
        out = _reduce_raw(code, x, ax)
        ctx.op, ctx.axis, ctx.shape = op, axis, tuple(a.shape)
        ctx.save_for_backward(a, out)
        return out

    @staticmethod
    def backward(ctx, c):
        a, out = ctx.saved_tensors
        shape, axis = ctx.shape, ctx.axis
        cb = c.reshape(()) if axis is None else c.unsqueeze(axis)
        cb = cb.expand(shape)  # _expand (autodiff.py:102-108): exact broadcast
        if ctx.op == "sum":
            g = _cast_to(cb, c.dtype)
        elif ctx.op == "mean":
            n = math.prod(shape) if axis is None else shape[axis]
            g = _ew(N.MPX_EW_DIV, cb, scalar=float(n))
        else:
            x = _contig(a)
            if axis is None:
                outer, n, inner = 1, x.numel(), 1
            else:
                outer, n, inner = _split(shape, axis)
            cc = _contig(c)
            g = torch.empty(shape, dtype=c.dtype, device=c.device)
            N.check(N.load().mpx_reduce_max_bwd(x.data_ptr(), _code(x), out.data_ptr(), cc.data_ptr(), _code(cc),
                                                outer, n, inner, g.data_ptr(), K.stream_handle(c.device)),
                    "mpx_reduce_max_bwd")
            g = _wrap(g)
        return None, _grad_for(g, a), None


def reduce(op_code: str, a, axis: int | None = None) -> Tensor:
    """sum / mean / max with stepwise accumulation in a's dtype (tensors.py:353-384)."""
    if op_code not in ("sum", "mean", "max"):
        raise ValueError(f"unknown reduction {op_code!r}")
    if not isinstance(a, torch.Tensor):
        raise TypeError("reduce expects a tensor")
    _require_float(a, op_code)
    ax = None if axis is None else _normalize_axis(axis, a.ndim, op_code)
    n = a.numel() if ax is None else a.shape[ax]
    if n == 0 and op_code == "mean":
        raise ValueError("mean over an empty axis")
    if n == 0 and op_code == "max":
        raise ValueError("max over an empty axis")
    return _note(_Reduce.apply(op_code, a, ax))


# ---------------------------------------------------------------- matmul
class _Matmul(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b, out_dtype):
        A = a.unsqueeze(0) if a.ndim == 1 else a
        B = b.unsqueeze(1) if b.ndim == 1 else b
        out = _mm_raw(A, B, out_dtype)
        if a.ndim == 1:
            out = out.squeeze(-2)
        if b.ndim == 1:
            out = out.squeeze(-1)
        ctx.save_for_backward(a, b)
        return _wrap(out)

    @staticmethod
    def backward(ctx, c):
        a, b = ctx.saved_tensors
        A = a.unsqueeze(0) if a.ndim == 1 else a
        B = b.unsqueeze(1) if b.ndim == 1 else b
        lead = tuple(torch.broadcast_shapes(A.shape[:-2], B.shape[:-2]))
        C = _contig(c).reshape(lead + (A.shape[-2], B.shape[-1]))
        ga = gb = None
        if ctx.needs_input_grad[0]:
            g = _unbroadcast(_mm_raw(C, _swap_last(B), _ptype(C, B)), A.shape)
            ga = _grad_for(g.reshape(a.shape), a)
        if ctx.needs_input_grad[1]:
            g = _unbroadcast(_mm_raw(_swap_last(A), C, _ptype(A, C)), B.shape)
            gb = _grad_for(g.reshape(b.shape), b)
        return ga, gb, None


def matmul(a, b) -> Tensor:
    """Matrix product with numpy broadcasting (tensors.py:387-422)."""
    if not (isinstance(a, torch.Tensor) and isinstance(b, torch.Tensor)):
        raise TypeError("matmul expects tensors")
    _require_float(a, "matmul")
    _require_float(b, "matmul")
    if a.ndim == 0 or b.ndim == 0:
        raise ValueError("matmul does not accept 0-d tensors")
    ka = a.shape[-1]
    kb = b.shape[0] if b.ndim == 1 else b.shape[-2]
    if ka != kb:
        raise ValueError(f"matmul inner extents disagree: {tuple(a.shape)} @ {tuple(b.shape)}")
    return _note(_Matmul.apply(a, b, promote(dtype_of(a), dtype_of(b)).torch))


# ---------------------------------------------------------------- softmax / layernorm / cross-entropy
class _Softmax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, ax):
        x = _contig(a)
        outer, n, inner = _split(tuple(x.shape), ax)
        out = torch.empty_like(x)
        N.check(N.load().mpx_softmax_axis(x.data_ptr(), _code(x), outer, n, inner, out.data_ptr(),
                                          K.stream_handle(x.device)), "mpx_softmax_axis")
        ctx.ax = ax
        ctx.save_for_backward(out)
        return _wrap(out)

    @staticmethod
    def backward(ctx, c):
        (y,) = ctx.saved_tensors
        cc = _cast_to(c, y.dtype)
        outer, n, inner = _split(tuple(y.shape), ctx.ax)
        g = torch.empty_like(y)
        N.check(N.load().mpx_softmax_axis_bwd(y.data_ptr(), cc.data_ptr(), _code(y), outer, n, inner, g.data_ptr(),
                                              K.stream_handle(y.device)), "mpx_softmax_axis_bwd")
        return _wrap(g), None


def softmax(a, axis: int) -> Tensor:
    """Max-shifted softmax along `axis` in a's dtype (tensors.py:431-446)."""
    if not isinstance(a, torch.Tensor):
        raise TypeError("softmax expects a tensor")
    _require_float(a, "softmax")
    return _note(_Softmax.apply(a, _normalize_axis(axis, a.ndim, "softmax")))


class _LayerNorm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, gain, bias, d):
        x = _contig(a)
        n = x.shape[-1]
        rows = x.numel() // n
        out = torch.empty(x.shape, dtype=d, device=x.device)
        N.check(N.load().mpx_layernorm_ref(x.data_ptr(), _code(x), gain.data_ptr(), _code(gain), bias.data_ptr(),
                                           _code(bias), rows, n, _code(d), out.data_ptr(), K.stream_handle(x.device)),
                "mpx_layernorm_ref")
        ctx.save_for_backward(x, gain, bias)
        return _wrap(out)

    @staticmethod
    def backward(ctx, c):
        x, gain, bias = ctx.saved_tensors
        d = c.dtype
        cc = _contig(c)
        n = x.shape[-1]
        rows = x.numel() // n
        dx = torch.empty(x.shape, dtype=d, device=x.device)
        dgx = torch.empty(x.shape, dtype=d, device=x.device)
        N.check(N.load().mpx_layernorm_ref_bwd(x.data_ptr(), _code(x), gain.data_ptr(), _code(gain), cc.data_ptr(),
                                               rows, n, _code(d), dx.data_ptr(), dgx.data_ptr(),
                                               K.stream_handle(x.device)), "mpx_layernorm_ref_bwd")
        dgain, dbias = _wrap(dgx), _wrap(cc)
        while dgain.ndim > 1:  # T.reduce("sum", ., axis=0) until 1-d (autodiff.py:257-261)
            dgain = _reduce_raw(N.MPX_RED_SUM, dgain, 0)
        while dbias.ndim > 1:
            dbias = _reduce_raw(N.MPX_RED_SUM, dbias, 0)
        return _grad_for(_wrap(dx), x), _grad_for(dgain, gain), _grad_for(dbias, bias), None


def layernorm(a, gain, bias) -> Tensor:
    """(a - mean) / sqrt(var + 1e-5) * gain + bias over the last axis (tensors.py:474-491)."""
    for t in (a, gain, bias):
        if not isinstance(t, torch.Tensor):
            raise TypeError("layernorm expects tensors")
        _require_float(t, "layernorm")
    if a.ndim == 0 or a.shape[-1] == 0:
        raise ValueError("layernorm over an empty axis")
    n = a.shape[-1]
    if tuple(gain.shape) != (n,) or tuple(bias.shape) != (n,):
        raise ValueError(f"gain/bias must have shape ({n},)")
    d = promote(promote(dtype_of(a), dtype_of(gain)), dtype_of(bias))
    return _note(_LayerNorm.apply(a, _contig(gain), _contig(bias), d.torch))


class _CrossEntropy(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, labels):
        x = _contig(logits)
        B, C = x.shape
        st = K.stream_handle(x.device)
        nll = torch.empty(B, dtype=x.dtype, device=x.device)
        lib = N.load()
        N.check(lib.mpx_xent_rows(x.data_ptr(), _code(x), labels.data_ptr(), B, C, nll.data_ptr(), st),
                "mpx_xent_rows")
        out = torch.empty((), dtype=x.dtype, device=x.device)
        N.check(lib.mpx_reduce(N.MPX_RED_MEAN, nll.data_ptr(), _code(x), 1, B, 1, out.data_ptr(), _code(x), st),
                "mpx_reduce")
        ctx.save_for_backward(x, labels)
        return _wrap(out)

    @staticmethod
    def backward(ctx, c):
        x, labels = ctx.saved_tensors
        B, C = x.shape
        cc = _contig(c)
        g = torch.empty_like(x)
        N.check(N.load().mpx_xent_bwd(x.data_ptr(), _code(x), labels.data_ptr(), B, C, cc.data_ptr(), _code(cc),
                                      g.data_ptr(), K.stream_handle(x.device)), "mpx_xent_bwd")
        return _wrap(g), None


def cross_entropy(logits, labels) -> Tensor:
    """Mean negative log-softmax of the true class (tensors.py:494-522)."""
    if not (isinstance(logits, torch.Tensor) and isinstance(labels, torch.Tensor)):
        raise TypeError("cross_entropy expects tensors")
    _require_float(logits, "cross_entropy")
    if labels.dtype != torch.int32:
        raise TypeError("labels must be an I32 tensor")
    if logits.ndim != 2:
        raise ValueError("logits must be 2-d (batch, classes)")
    batch, classes = logits.shape
    if tuple(labels.shape) != (batch,):
        raise ValueError(f"labels must have shape ({batch},)")
    K.require_cuda([labels], "cross_entropy")
    if batch:
        lab = labels.cpu().numpy()  # the reference's range check (tensors.py:509-511) is a host decision
        if lab.min() < 0 or lab.max() >= classes:
            raise ValueError("label out of range")
    return _note(_CrossEntropy.apply(logits, _contig(labels)))


# ---------------------------------------------------------------- structural ops
def cast(a, dtype) -> Tensor:
    """Re-quantize a float tensor onto another grid (tensors.py:529-538), K1."""
    if not isinstance(a, torch.Tensor):
        raise TypeError("cast expects a tensor")
    _require_float(a, "cast")
    d = as_dtype(dtype)
    if not d.is_float:
        raise ValueError("cast target must be a float dtype")
    from .precision import cast_tree

    return _wrap(cast_tree(a, d))


class _Reshape(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, shape):
        ctx.in_shape = tuple(a.shape)
        return _wrap(_contig(a).reshape(shape))

    @staticmethod
    def backward(ctx, c):
        return _wrap(_contig(c).reshape(ctx.in_shape)), None


def reshape(a, shape) -> Tensor:
    if not isinstance(a, torch.Tensor):
        raise TypeError("reshape expects a tensor")
    return _note(_Reshape.apply(a, tuple(shape) if not isinstance(shape, int) else (shape,)))


class _Transpose(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, axes):
        ctx.inv = tuple(int(i) for i in np.argsort(axes))
        return _wrap(a.permute(axes))  # a strided view: the kernels read any strides

    @staticmethod
    def backward(ctx, c):
        return _wrap(c.permute(ctx.inv)), None


def transpose(a, axes=None) -> Tensor:
    if not isinstance(a, torch.Tensor):
        raise TypeError("transpose expects a tensor")
    axes = tuple(range(a.ndim))[::-1] if axes is None else tuple(axes)
    if sorted(axes) != list(range(a.ndim)):
        raise ValueError(f"transpose: {axes} is not a permutation of {a.ndim} axes")
    return _note(_Transpose.apply(a, axes))


__all__ = ["Tensor", "tensor", "zeros", "zeros_like", "ones", "bytes_of", "quantize", "quantize_array", "add", "sub",
           "mul", "div", "neg", "exp", "log", "sqrt", "relu", "gelu", "elementwise", "reduce", "matmul", "softmax",
           "layernorm", "cross_entropy", "cast", "reshape", "transpose", "I32", "DType"]
