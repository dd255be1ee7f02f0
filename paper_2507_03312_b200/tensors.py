"""Tensor constructors with the reference's quantize-on-construction rule
(tensors.py:104-132): `tensor(data, F16)` holds round_f16(f32(data)),
rounded on the device by K1.  Tensors are plain torch CUDA tensors."""
from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .dtypes import F32, I32, as_dtype, dtype_of

_MAX_I32 = 2 ** 31 - 1
_MIN_I32 = -(2 ** 31)


def _device(device):
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def tensor(data, dtype=F32, device=None) -> torch.Tensor:
    d = as_dtype(dtype)
    dev = _device(device)
    if not d.is_float:
        arr = np.asarray(data, dtype=np.int64)
        if arr.size and (arr.max() > _MAX_I32 or arr.min() < _MIN_I32):
            raise ValueError("value out of 32-bit signed integer range")
        return torch.from_numpy(arr.astype(np.int32)).to(dev)
    f32 = torch.from_numpy(np.array(data, dtype=np.float32, order="C")).to(dev)
    if d is F32:
        return f32
    return K.cast_leaves([f32], d)[0]


def zeros(shape, dtype=F32, device=None) -> torch.Tensor:
    return torch.zeros(shape, dtype=as_dtype(dtype).torch, device=_device(device))


def ones(shape, dtype=F32, device=None) -> torch.Tensor:
    return torch.ones(shape, dtype=as_dtype(dtype).torch, device=_device(device))


def bytes_of(t: torch.Tensor) -> int:
    """Footprint at the nominal precision (tensors.py:130-132)."""
    d = dtype_of(t)
    return t.numel() * (d.byte_width if d is not None else t.element_size())


__all__ = ["tensor", "zeros", "ones", "bytes_of", "I32"]
