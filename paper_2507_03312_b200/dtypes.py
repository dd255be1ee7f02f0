"""Numeric formats and the promotion lattice (mirror of mpsim.dtypes).

In the reference every value is an f32 payload that *sits on* a format's grid
(dtypes.py:1-21).  Here values are physically stored in their format on the
device (torch.float16 / bfloat16 / float32 / int32 CUDA tensors); the DType
enum keeps the reference's names and lattice so user code and tests read the
same.

    DType / F16 / BF16 / F32 / I32      dtypes.py:31-52
    promote (join; F16 v BF16 = F32)    dtypes.py:55-67
    Scalar (weak / strong)              dtypes.py:70-86
    promote_with_scalar                 dtypes.py:89-93
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native


class DType(Enum):
    F16 = "f16"
    BF16 = "bf16"
    F32 = "f32"
    I32 = "i32"

    @property
    def byte_width(self) -> int:
        return 4 if self in (DType.F32, DType.I32) else 2

    @property
    def is_float(self) -> bool:
        return self is not DType.I32

    @property
    def torch(self) -> torch.dtype:
        return _TO_TORCH[self]

    @property
    def code(self) -> int:
        """dtype code of the C ABI (MPX_F32/F16/BF16)."""
        if self is DType.I32:
            raise ValueError("integers are never quantized")
        return _TO_CODE[self]

    def __repr__(self) -> str:
        return self.value


F16 = DType.F16
BF16 = DType.BF16
F32 = DType.F32
I32 = DType.I32

_TO_TORCH = {F16: torch.float16, BF16: torch.bfloat16, F32: torch.float32, I32: torch.int32}
_FROM_TORCH = {v: k for k, v in _TO_TORCH.items()}
_TO_CODE = {F32: _native.MPX_F32, F16: _native.MPX_F16, BF16: _native.MPX_BF16}

# height in the lattice; two distinct dtypes of equal height join to F32
_LEVEL = {I32: 0, F16: 1, BF16: 1, F32: 2}


def promote(a: DType, b: DType) -> DType:
    """Least upper bound of two dtypes (dtypes.py:60-67)."""
    if a is b:
        return a
    la, lb = _LEVEL[a], _LEVEL[b]
    if la == lb:
        return F32
    return b if lb > la else a


def as_dtype(x) -> DType:
    """Accept a DType, a torch.dtype or a dtype name ('f16', 'bf16', ...)."""
    if isinstance(x, DType):
        return x
    if isinstance(x, torch.dtype):
        try:
            return _FROM_TORCH[x]
        except KeyError:
            raise ValueError(f"unsupported torch dtype {x}") from None
    if isinstance(x, str):
        return DType(x)
    raise TypeError(f"not a dtype: {x!r}")


def dtype_of(t: torch.Tensor) -> DType | None:
    """Nominal dtype of a tensor leaf, or None for unsupported storage types."""
    return _FROM_TORCH.get(t.dtype)


def is_float_leaf(x) -> bool:
    """A leaf the numeric transforms act on: a float16/bfloat16/float32 tensor."""
    return isinstance(x, torch.Tensor) and x.dtype in (torch.float16, torch.bfloat16, torch.float32)


@dataclass(frozen=True)
class Scalar:
    """Scalar operand; weak scalars (Python literals) never promote (dtypes.py:70-86)."""

    value: float
    weak: bool = True
    dtype: DType | None = None

    def __post_init__(self):
        if not self.weak and self.dtype is None:
            is_int = isinstance(self.value, int) and not isinstance(self.value, bool)
            object.__setattr__(self, "dtype", I32 if is_int else F32)


def promote_with_scalar(t: DType, s: Scalar) -> DType:
    return t if s.weak else promote(t, s.dtype)


def quantize_host_scalar(value: float, dtype: DType) -> float:
    """Round ONE host-side Python scalar onto a format's grid (strong-Scalar
    metadata only, precision.py:66-67).  Tensor data never takes this path: it
    is cast on the device by K1."""
    if not dtype.is_float:
        raise ValueError("integers are never quantized")
    x = np.float32(value)
    if dtype is F32:
        return float(x)
    with np.errstate(over="ignore", invalid="ignore"):
        if dtype is F16:
            return float(np.float16(x))
        if np.isnan(x):
            return float(x)
        u = int(x.view(np.uint32))
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        return float(np.uint32(u).view(np.float32))
