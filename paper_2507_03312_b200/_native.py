"""ctypes binding of libmpx_b200.so (the C ABI declared in include/mpx_b200.h).

There is no CPU fallback anywhere in this package: if the library is missing
or no CUDA device is present, every compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmpx_b200.so"

MPX_F32, MPX_F16, MPX_BF16 = 0, 1, 2

_P = ctypes.c_void_p
_PP = ctypes.POINTER(ctypes.c_void_p)
_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)


class ScalingStateC(ctypes.Structure):
    """mpx_scaling_state (include/mpx_b200.h) — 48 bytes."""

    _fields_ = [
        ("loss_scale", ctypes.c_double),
        ("growth_factor", ctypes.c_double),
        ("backoff_factor", ctypes.c_double),
        ("min_scale", ctypes.c_double),
        ("growth_interval", ctypes.c_int64),
        ("steps_since_growth", ctypes.c_int64),
    ]


class AdamHParamsC(ctypes.Structure):
    """mpx_adam_hparams (include/mpx_b200.h)."""

    _fields_ = [(n, ctypes.c_float) for n in ("b1", "omb1", "b2", "omb2", "lr", "eps", "neg_lr", "neg_lr_wd")]


class GemmDescC(ctypes.Structure):
    """mpx_gemm_desc (include/mpx_b200.h)."""

    _fields_ = [
        ("ab_dtype", ctypes.c_int), ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int64), ("a_sb1", ctypes.c_int64), ("a_sb2", ctypes.c_int64),
        ("a_mn_major", ctypes.c_int),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("b_sb1", ctypes.c_int64), ("b_sb2", ctypes.c_int64),
        ("b_mn_major", ctypes.c_int),
        ("nb1", ctypes.c_int), ("nb2", ctypes.c_int),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64), ("c_sb1", ctypes.c_int64), ("c_sb2", ctypes.c_int64),
        ("c_dtype", ctypes.c_int),
        ("bias", ctypes.c_void_p), ("residual", ctypes.c_void_p), ("ldr", ctypes.c_int64),
        ("r_sb1", ctypes.c_int64), ("r_sb2", ctypes.c_int64),
        ("aux", ctypes.c_void_p), ("ld_aux", ctypes.c_int64),
        ("alpha", ctypes.c_float), ("act", ctypes.c_int), ("block_n", ctypes.c_int), ("split_k", ctypes.c_int),
        ("workspace", ctypes.c_void_p), ("cta_group", ctypes.c_int), ("tma_store", ctypes.c_int),
        ("colsum_ws", ctypes.c_void_p), ("colsum_out", ctypes.c_void_p),
        ("ln_gain", ctypes.c_void_p), ("ln_bias", ctypes.c_void_p), ("ln_out", ctypes.c_void_p),
        ("ld_ln", ctypes.c_int64), ("ln_mean", ctypes.c_void_p), ("ln_rstd", ctypes.c_void_p),
        ("ln_eps", ctypes.c_float),
    ]


# every symbol include/mpx_b200.h declares: (name, restype, argtypes)
SIGNATURES = {
    "mpx_last_error": (ctypes.c_char_p, []),
    "mpx_version": (ctypes.c_int, []),
    "mpx_num_sms": (ctypes.c_int, [ctypes.c_int]),
    "mpx_launch_count": (ctypes.c_int64, []),
    "mpx_cast": (ctypes.c_int, [_PP, _PP, _I64P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_double, _P, _P]),
    "mpx_unscale_finite": (ctypes.c_int, [_PP, _PP, _I64P, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                          _P, _P, ctypes.c_int, _P]),
    "mpx_scaling_adjust": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "mpx_optimizer_step": (ctypes.c_int, [_PP, _I32P, _PP, _PP, _PP, _PP, _PP, _I64P, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, AdamHParamsC,
                                          _P, ctypes.c_int64, _P, ctypes.c_double, _P, _P, _P]),
    "mpx_gemm": (ctypes.c_int, [ctypes.POINTER(GemmDescC), _P]),
    "mpx_layernorm_fwd": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, _P, _P, _P, ctypes.c_int64, _P, _P,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_float, _P]),
    "mpx_layernorm_bwd_blocks": (ctypes.c_int, [ctypes.c_int]),
    "mpx_layernorm_bwd": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int64, _P,
                                         ctypes.c_int64, _P, ctypes.c_int64, _P, _P, _P, ctypes.c_int, ctypes.c_int,
                                         _P]),
    "mpx_layernorm_bwd2": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int64, _P,
                                          ctypes.c_int64, _P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int64,
                                          ctypes.c_int, ctypes.c_int, _P]),
    "mpx_colsum": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_float,
                                  _P]),
    "mpx_softmax_fwd": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, _P]),
    "mpx_softmax_bwd": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, _P]),
    "mpx_cross_entropy_fwd": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, _P, ctypes.c_int, ctypes.c_int, _P,
                                             _P, _P]),
    "mpx_cross_entropy_bwd": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, _P, ctypes.c_int, ctypes.c_int, _P,
                                             _P, ctypes.c_int64, _P]),
    "mpx_attention_fwd": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_float, _P, ctypes.c_int64, _P, _P, _P]),
    "mpx_attention_psave_bytes": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "mpx_attention_bwd": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_float, _P, _P, _P, _P, _P, _P]),
    "mpx_patchify": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _P]),
    "mpx_transpose": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _P,
                                     ctypes.c_int64, _P]),
    "mpx_transpose_batch": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P]),
    "mpx_copy_rows": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, ctypes.c_int64, _P, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "mpx_rows_add": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _P]),
    "mpx_bcast_rows": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, _P]),
    "mpx_ew": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64P, _P, ctypes.c_int, _P, ctypes.c_int, _I64P, _P,
                              ctypes.c_int, _I64P, ctypes.c_double, ctypes.c_int, ctypes.c_int, _P]),
    "mpx_reduce": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P,
                                  ctypes.c_int, _P]),
    "mpx_reduce_max_bwd": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, _P, _P]),
    "mpx_softmax_axis": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P, _P]),
    "mpx_softmax_axis_bwd": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P,
                                            _P]),
    "mpx_layernorm_ref": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int, _P, _P]),
    "mpx_layernorm_ref_bwd": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int, _P, _P, _P]),
    "mpx_xent_rows": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int64, ctypes.c_int64, _P, _P]),
    "mpx_xent_bwd": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int64, ctypes.c_int64, _P, ctypes.c_int, _P, _P]),
    "mpx_matmul_simt": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int64, _I64P, ctypes.c_int, _I64P, _I64P, _I64P, _I64P,
                                       _P]),
    "mpx_comm_unique_id": (ctypes.c_int, [_P]),
    "mpx_comm_init": (ctypes.c_int, [_PP, ctypes.c_int, _P, ctypes.c_int, ctypes.c_int]),
    "mpx_comm_destroy": (ctypes.c_int, [_P]),
    "mpx_comm_size": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
    "mpx_allreduce_flag": (ctypes.c_int, [_P, _P, _P]),
    "mpx_allreduce_grads": (ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int, _P]),
}

MPX_COMM_ID_BYTES = 128
(MPX_EW_COPY, MPX_EW_ADD, MPX_EW_SUB, MPX_EW_MUL, MPX_EW_DIV, MPX_EW_NEG, MPX_EW_EXP, MPX_EW_LOG, MPX_EW_SQRT,
 MPX_EW_RELU, MPX_EW_GELU, MPX_EW_GELU_BWD, MPX_EW_RELU_BWD) = range(13)
MPX_RED_SUM, MPX_RED_MEAN, MPX_RED_MAX = 0, 1, 2

_lib = None
_lock = threading.Lock()


def load(path: Path | str | None = None):
    """Load (once) and return the native library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path or os.environ.get("MPX_B200_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(
                f"mpx_b200 native library not found at {p}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str):
    if rc != 0:
        msg = load().mpx_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (code {rc}): {msg}")


def ptr_array(values) -> "ctypes.Array":
    arr = (ctypes.c_void_p * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr


def i64_array(values):
    a = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
    return a, a.ctypes.data_as(_I64P)


def i32_array(values):
    a = np.ascontiguousarray(np.asarray(values, dtype=np.int32))
    return a, a.ctypes.data_as(_I32P)


def as_pp(arr) -> "_PP":
    return ctypes.cast(arr, _PP)
