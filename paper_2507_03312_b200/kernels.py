"""Tensor-level wrappers of the C ABI (K1-K4).  Device memory and streams come
from torch; all arithmetic happens in libmpx_b200.so on the caller's current
CUDA stream.  Nothing here has a CPU path: non-CUDA tensors raise."""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .dtypes import BF16, F16, F32, DType, as_dtype, dtype_of

_ALIGN = 8  # elements; 16 B for 2-byte, 32 B for 4-byte types


def stream_handle(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda(tensors: Sequence[torch.Tensor], what: str):
    for t in tensors:
        if not t.is_cuda:
            raise TypeError(f"{what}: mpx_b200 computes on CUDA tensors only (got a {t.device} tensor); "
                            "there is no CPU fallback")
    if tensors and not torch.cuda.is_available():
        raise RuntimeError(f"{what}: no CUDA device")


def _contig(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_contiguous() else t.contiguous()


def new_flag(device) -> torch.Tensor:
    """A 0-d int32 device flag (1 = all finite)."""
    return torch.ones((), dtype=torch.int32, device=device)


def arena_like(leaves: Sequence[torch.Tensor], dtype: torch.dtype) -> list[torch.Tensor]:
    """Fresh output tensors shaped like `leaves`, carved from ONE allocation
    (each leaf 16-byte aligned), so a whole tree is one contiguous arena."""
    if not leaves:
        return []
    offs, total = [], 0
    for t in leaves:
        offs.append(total)
        total += -(-t.numel() // _ALIGN) * _ALIGN
    arena = torch.empty(max(total, 1), dtype=dtype, device=leaves[0].device)
    return [arena[o:o + t.numel()].view(t.shape) for o, t in zip(offs, leaves)]


def _group_by_dtype(leaves):
    groups: dict[DType, list[int]] = {}
    for i, t in enumerate(leaves):
        d = dtype_of(t)
        if d is None or not d.is_float:
            raise TypeError(f"expected a float tensor, got {t.dtype}")
        groups.setdefault(d, []).append(i)
    return groups


# ---------------------------------------------------------------------------
# K1
# ---------------------------------------------------------------------------
def cast_into(srcs: Sequence[torch.Tensor], dsts: Sequence[torch.Tensor], scale: float = 1.0,
              d_scale: torch.Tensor | None = None):
    """dst[i] = round_{dst dtype}(f32(src[i]) * scale) for same-shaped leaves."""
    if not srcs:
        return
    require_cuda(list(srcs) + list(dsts), "cast")
    lib = N.load()
    stream = stream_handle(srcs[0].device)
    dscale_ptr = d_scale.data_ptr() if d_scale is not None else None
    # group by (src dtype, dst dtype): one native call (usually one launch) each
    groups: dict[tuple[DType, DType], list[int]] = {}
    for i, (s, d) in enumerate(zip(srcs, dsts)):
        groups.setdefault((dtype_of(s), dtype_of(d)), []).append(i)
    for (sd, dd), idx in groups.items():
        if sd is None or dd is None or not sd.is_float or not dd.is_float:
            raise TypeError("cast: float tensors only")
        src = [_contig(srcs[i]) for i in idx]
        for i in idx:
            if not dsts[i].is_contiguous():
                raise ValueError("cast: destination must be contiguous")
        sp = N.ptr_array([t.data_ptr() for t in src])
        dp = N.ptr_array([dsts[i].data_ptr() for i in idx])
        _n, n_p = N.i64_array([t.numel() for t in src])
        N.check(lib.mpx_cast(N.as_pp(sp), N.as_pp(dp), n_p, len(idx), sd.code, dd.code, float(scale),
                             dscale_ptr, stream), "mpx_cast")


def cast_leaves(leaves: Sequence[torch.Tensor], dtype, scale: float = 1.0,
                d_scale: torch.Tensor | None = None) -> list[torch.Tensor]:
    """New tensors (one arena) holding round_dtype(leaf * scale)."""
    d = as_dtype(dtype)
    outs = arena_like(leaves, d.torch)
    cast_into(leaves, outs, scale, d_scale)
    return outs


# ---------------------------------------------------------------------------
# K2
# ---------------------------------------------------------------------------
def unscale_finite(leaves: Sequence[torch.Tensor], scale: float = 1.0, d_scale: torch.Tensor | None = None,
                   write_f32: bool = True, flag: torch.Tensor | None = None,
                   reset: bool = True) -> tuple[list[torch.Tensor] | None, torch.Tensor]:
    """(f32 leaves = f32(g)/f32(scale) or None, device finite flag)."""
    if not leaves:
        dev = torch.device("cuda", torch.cuda.current_device())
        return ([] if write_f32 else None), (flag if flag is not None else new_flag(dev))
    require_cuda(leaves, "unscale")
    lib = N.load()
    dev = leaves[0].device
    stream = stream_handle(dev)
    if flag is None:
        flag = torch.empty((), dtype=torch.int32, device=dev)
        reset = True
    outs = arena_like(leaves, torch.float32) if write_f32 else None
    dscale_ptr = d_scale.data_ptr() if d_scale is not None else None
    first = True
    for d, idx in _group_by_dtype(leaves).items():
        src = [_contig(leaves[i]) for i in idx]
        gp = N.ptr_array([t.data_ptr() for t in src])
        op = N.ptr_array([outs[i].data_ptr() for i in idx]) if outs is not None else None
        _n, n_p = N.i64_array([t.numel() for t in src])
        N.check(lib.mpx_unscale_finite(N.as_pp(gp), N.as_pp(op) if op is not None else None, n_p, len(idx),
                                       d.code, float(scale), dscale_ptr, flag.data_ptr(),
                                       1 if (reset and first) else 0, stream), "mpx_unscale_finite")
        first = False
    return outs, flag


def all_finite_flag(leaves: Sequence[torch.Tensor]) -> torch.Tensor:
    return unscale_finite(leaves, 1.0, write_f32=False)[1]


# ---------------------------------------------------------------------------
# K3
# ---------------------------------------------------------------------------
SCALING_STATE_BYTES = ctypes.sizeof(N.ScalingStateC)


def pack_scaling_state(loss_scale, growth_factor, backoff_factor, growth_interval, steps_since_growth,
                       min_scale, device) -> torch.Tensor:
    """48-byte device buffer laid out as mpx_scaling_state (uint8 tensor)."""
    st = N.ScalingStateC(float(loss_scale), float(growth_factor), float(backoff_factor), float(min_scale),
                         int(growth_interval), int(steps_since_growth))
    host = torch.frombuffer(bytearray(bytes(st)), dtype=torch.uint8)
    return host.to(device)


def unpack_scaling_state(buf: torch.Tensor) -> N.ScalingStateC:
    return N.ScalingStateC.from_buffer_copy(bytes(buf.cpu().numpy().tobytes()))


def scaling_adjust(state: torch.Tensor, flag: torch.Tensor, step_counter: torch.Tensor | None = None,
                   used_scale: torch.Tensor | None = None):
    require_cuda([state, flag], "adjust")
    lib = N.load()
    N.check(lib.mpx_scaling_adjust(state.data_ptr(), flag.data_ptr(),
                                   step_counter.data_ptr() if step_counter is not None else None,
                                   used_scale.data_ptr() if used_scale is not None else None,
                                   stream_handle(state.device)), "mpx_scaling_adjust")


# ---------------------------------------------------------------------------
# K4
# ---------------------------------------------------------------------------
def adam_hparams(lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0) -> N.AdamHParamsC:
    """Round the Python-double hyper-parameters exactly as the reference's weak
    scalars are rounded (np.float32 at use; optim.py:78-97)."""
    f = lambda x: float(np.float32(x))  # noqa: E731
    return N.AdamHParamsC(f(beta1), f(1.0 - beta1), f(beta2), f(1.0 - beta2), f(lr), f(eps), f(-lr),
                          f(-lr * weight_decay) if weight_decay else 0.0)


_BC_CACHE: dict[tuple, torch.Tensor] = {}
_BC_MAX = 1 << 22


def bias_correction_table(beta1: float, beta2: float, device) -> torch.Tensor:
    """f32(1 - beta**t) for t = 1..T computed with Python-double `**`
    (optim.py:73-76), up to the step where both entries round to 1.0f for
    good; the kernel clamps t to the table length."""
    key = (float(beta1), float(beta2), str(device))
    tab = _BC_CACHE.get(key)
    if tab is not None:
        return tab
    vals = []
    t = 1
    while t <= _BC_MAX:
        a = np.float32(1.0 - beta1 ** t)
        b = np.float32(1.0 - beta2 ** t)
        vals.append((a, b))
        if a == np.float32(1.0) and b == np.float32(1.0):
            break
        t += 1
    tab = torch.from_numpy(np.asarray(vals, dtype=np.float32).reshape(-1)).to(device)
    _BC_CACHE[key] = tab
    return tab


def optimizer_step(params: Sequence[torch.Tensor], grads: Sequence[torch.Tensor],
                   m: Sequence[torch.Tensor] | None, v: Sequence[torch.Tensor] | None, *,
                   mode: int, hp: N.AdamHParamsC, counter: torch.Tensor, bc_table: torch.Tensor | None,
                   scale: float = 1.0, d_scale: torch.Tensor | None = None, flag: torch.Tensor | None = None,
                   half_out: Sequence[torch.Tensor] | None = None, upd_out: Sequence[torch.Tensor] | None = None):
    """In-place gated Adam (mode 0) / SGD (mode 1) over a leaf table."""
    n = len(params)
    if n == 0:
        return
    require_cuda(list(params) + list(grads), "optimizer_update")
    lib = N.load()
    dev = params[0].device
    gdt = {dtype_of(g) for g in grads}
    if len(gdt) != 1:
        # mixed gradient formats (the reference accepts any float leaves,
        # optim.py:58-97): one K4 call per format group.  Every group must see
        # the same step t = step_count + 1, so all but the last group count on
        # private copies of the counter taken before any group runs; the last
        # group advances the real one (once, when the step is applied).
        order = sorted(gdt, key=lambda d: d.value)
        groups = [[i for i, g in enumerate(grads) if dtype_of(g) is d] for d in order]
        privs = [counter.clone() for _ in groups[:-1]]
        for k, idx in enumerate(groups):
            sel = lambda seq: [seq[i] for i in idx] if seq is not None else None  # noqa: E731
            optimizer_step(sel(params), sel(grads), sel(m), sel(v), mode=mode, hp=hp,
                           counter=privs[k] if k < len(privs) else counter, bc_table=bc_table, scale=scale,
                           d_scale=d_scale, flag=flag, half_out=sel(half_out), upd_out=sel(upd_out))
        return
    gdt = gdt.pop()
    hdt = -1
    if half_out is not None:
        hd = {dtype_of(h) for h in half_out if h is not None}
        if len(hd) > 1:
            raise ValueError("half working copies must share one dtype")
        hdt = hd.pop().code if hd else -1
    for t in list(params) + list(grads) + list(m or []) + list(v or []):
        if not t.is_contiguous():
            raise ValueError("optimizer_update: leaves must be contiguous")
    pp = N.ptr_array([t.data_ptr() for t in params])
    _pd, pd_p = N.i32_array([dtype_of(t).code for t in params])
    mp = N.ptr_array([t.data_ptr() for t in m]) if m is not None else N.ptr_array([0] * n)
    vp = N.ptr_array([t.data_ptr() for t in v]) if v is not None else N.ptr_array([0] * n)
    gp = N.ptr_array([t.data_ptr() for t in grads])
    hp_ = N.ptr_array([(h.data_ptr() if h is not None else 0) for h in half_out]) if half_out is not None else None
    up = N.ptr_array([t.data_ptr() for t in upd_out]) if upd_out is not None else None
    _n, n_p = N.i64_array([t.numel() for t in params])
    rc = lib.mpx_optimizer_step(
        N.as_pp(pp), pd_p, N.as_pp(mp), N.as_pp(vp), N.as_pp(gp),
        N.as_pp(hp_) if hp_ is not None else None, N.as_pp(up) if up is not None else None,
        n_p, n, gdt.code, hdt, mode, hp,
        bc_table.data_ptr() if bc_table is not None else None,
        bc_table.numel() // 2 if bc_table is not None else 0,
        counter.data_ptr(), float(scale), d_scale.data_ptr() if d_scale is not None else None,
        flag.data_ptr() if flag is not None else None, stream_handle(dev))
    N.check(rc, "mpx_optimizer_step")


__all__ = [
    "F16", "BF16", "F32", "cast_into", "cast_leaves", "unscale_finite", "all_finite_flag", "scaling_adjust",
    "pack_scaling_state", "unpack_scaling_state", "adam_hparams", "bias_correction_table", "optimizer_step",
    "arena_like", "new_flag", "stream_handle", "require_cuda",
]
