"""ctypes binding of the in-tree C-ABI library ``libattnqat_b200.so``.

The library is the only compute path: if it is missing, or there is no CUDA
device, every operator raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AQ_LIB_PATH") or os.path.join(_HERE, "libattnqat_b200.so")  # override: tuning builds

DT_CODE = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_f = ctypes.c_float
c_vp = ctypes.c_void_p


class AqFwdArgs(ctypes.Structure):
    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp), ("in_dtype", c_int),
        ("heads", c_i64), ("n_q", c_i64), ("n_k", c_i64), ("d", c_i64),
        ("causal", c_int), ("train", c_int),
        ("o", c_vp), ("o_dtype", c_int), ("o_hp", c_vp), ("o_hp_dtype", c_int),
        ("lse", c_vp), ("workspace", c_vp), ("keep_for_bwd", c_int), ("operands_staged", c_int),
        # ABI 3
        ("softmax_scale", c_f), ("q_scale", c_f), ("k_scale", c_f), ("v_scale", c_f), ("p_scale", c_f),
        ("nonfinite", c_vp), ("pf_codes", c_vp), ("pf_scales", c_vp),
    ]


class AqSage3Args(ctypes.Structure):
    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp), ("in_dtype", c_int),
        ("heads", c_i64), ("n_q", c_i64), ("n_k", c_i64), ("d", c_i64),
        ("causal", c_int), ("b_q", c_i64), ("b_k", c_i64),
        ("smooth_q", c_int), ("smooth_k", c_int), ("two_level_p", c_int),
        ("o", c_vp), ("o_dtype", c_int), ("lse", c_vp), ("workspace", c_vp),
    ]


class AqBwdArgs(ctypes.Structure):
    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp), ("in_dtype", c_int),
        ("d_o", c_vp), ("do_dtype", c_int),
        ("o", c_vp), ("o_hp", c_vp), ("o_dtype", c_int),
        ("lse", c_vp),
        ("heads", c_i64), ("n_q", c_i64), ("n_k", c_i64), ("d", c_i64),
        ("causal", c_int), ("variant", c_int),
        ("dq", c_vp), ("dk", c_vp), ("dv", c_vp), ("g_dtype", c_int),
        ("workspace", c_vp), ("fwd_workspace", c_vp),
        # ABI 3
        ("softmax_scale", c_f), ("q_scale", c_f), ("k_scale", c_f), ("v_scale", c_f), ("p_scale", c_f),
        ("nonfinite", c_vp), ("pf_codes", c_vp), ("pf_scales", c_vp),
    ]


# symbol name -> (restype, argtypes); mirrors include/attnqat_b200.h
PROTOTYPES = {
    "aq_abi_version": (c_int, []),
    "aq_status_string": (ctypes.c_char_p, [c_int]),
    "aq_quantize_rows": (c_int, [c_vp, c_int, c_i64, c_i64, c_i64, c_i64, c_i64,
                                 c_vp, c_vp, c_vp, c_int, c_f, c_vp, c_vp]),
    "aq_quantize_cols": (c_int, [c_vp, c_int, c_i64, c_i64, c_i64, c_i64, c_i64,
                                 c_vp, c_vp, c_vp, c_int, c_f, c_vp, c_vp]),
    "aq_dequantize": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_int, c_f, c_vp]),
    "aq_fp4mm_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64]),
    "aq_fp4mm": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "aq_fp4mm_mx": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "aq_quantize_mx": (c_int, [c_vp, c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp]),
    "aq_dequantize_mx": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_int, c_vp]),
    "aq_e8m0_codes": (c_int, [c_vp, c_int, c_i64, c_vp, c_vp, c_vp]),
    "aq_round_codes": (c_int, [c_vp, c_int, c_i64, c_int, c_vp, c_vp, c_vp]),
    "aq_attn_fwd_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64, c_i64, c_int, c_int]),
    "aq_attn_fwd": (c_int, [ctypes.POINTER(AqFwdArgs), c_vp]),
    "aq_attn_fwd_kv4": (c_int, [ctypes.POINTER(AqFwdArgs), c_vp, c_vp, c_vp, c_vp, c_vp]),
    "aq_attn_fwd_plain": (c_int, [ctypes.POINTER(AqFwdArgs), c_int, c_vp]),
    "aq_attn_fwd_mx": (c_int, [ctypes.POINTER(AqFwdArgs), c_vp]),
    "aq_attn_bwd_mx": (c_int, [ctypes.POINTER(AqBwdArgs), c_vp]),
    "aq_attn_bwd_plain": (c_int, [ctypes.POINTER(AqBwdArgs), c_int, c_vp]),
    "aq_attn_fwd_sage3_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64, c_i64, c_i64, c_i64]),
    "aq_attn_fwd_sage3": (c_int, [ctypes.POINTER(AqSage3Args), c_vp]),
    "aq_attn_bwd_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64, c_i64]),
    "aq_attn_bwd": (c_int, [ctypes.POINTER(AqBwdArgs), c_vp]),
    "aq_probe_mma_peak": (c_int, [c_int, c_int, c_int, c_vp]),
    "aq_probe_mma_flops": (ctypes.c_double, [c_int, c_int, c_int]),
    "aq_debug_fwd_profile": (c_int, [ctypes.POINTER(ctypes.c_ulonglong), c_int]),
    "aq_debug_bwd_profile": (c_int, [ctypes.POINTER(ctypes.c_ulonglong), c_int]),
    "aq_debug_bwd_timeline": (c_int, [ctypes.POINTER(ctypes.c_ulonglong), c_int]),
}

_lib = None


def load():
    """Load the library (no GPU needed to load; compute calls need one)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2603_00040_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("the attnqat B200 path needs a CUDA (sm_100a) device; there is no CPU fallback")
    load()


def check(status: int):
    if status == 0:
        return
    msg = load().aq_status_string(status).decode()
    cls = {1: errors.ShapeError, 2: errors.TileError, 3: errors.InvalidValue,
           4: errors.MissingOPrime}.get(status, RuntimeError)
    raise cls(f"attnqat_b200: {msg}")


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())
