"""``quantized=False``: plain (unquantized) attention, the reference's bf16 mode.

flash_forward_training / flash_backward with quantized=False skip every fake
quantization (flash.py:195-200, 344-349): O = O' = softmax(QK^T/sqrt(d)) V and
the textbook backward. The reference harness uses it for its "bf16" training
and evaluation mode (harness.py:40, 333-335). Both directions run on the
hand-written sm_100a kernels (no library attention):

* forward (``aq_attn_fwd_plain``): the K4 skeleton with 16-bit operands -- Q /
  K / V staged as fp16 (or bf16 when a value leaves fp16's range) T8x8 tiles,
  S and P^ V on ``kind::f16`` MMAs with fp32 accumulation, the two-pass
  softmax of the FP4 path (L final before the P V pass, 1/l in the epilogue);
* backward (``aq_attn_bwd_plain``): the K7 skeleton with S recomputed from
  Q / K tiles in the forward's 16-bit format on ``kind::f16`` (so S and L
  agree), P = exp(S - L) unquantized for dV and dS, D = rowsum(dO . O)
  (flash.py:333-351), every operand in that format (fp16 with an exact
  power-of-two gain on dO, or bf16); dQ / dK / dV in TMEM, deterministic;
* head dims other than 64 / 128 (any d <= 128, e.g. the reference tests' 16 /
  24 / 32) are zero-padded to the next kernel width -- exact: zero Q / K
  columns add nothing to S, zero V columns give zero O columns -- with the
  softmax scale kept at 1/sqrt(d).
"""

from __future__ import annotations

import math

import torch

from .errors import InvalidValue, ShapeError


def _compute_dtype(*ts):
    """16-bit operand format of the forward for float32 Q / K / V: fp16
    (11-bit significand) when the largest magnitude sits inside its normal
    range with headroom (2^-10 <= amax < 6e4), else bf16 (fp32's exponent
    range). bf16 / fp16 inputs keep their format."""
    dt = ts[0].dtype
    if dt in (torch.float16, torch.bfloat16):
        return dt
    if dt != torch.float32:
        raise InvalidValue("plain attention takes float32 / bfloat16 / float16 operands")
    amax = max(float(t.abs().max()) for t in ts if t.numel())
    return torch.float16 if 2.0 ** -10 <= amax < 6.0e4 else torch.bfloat16


def _kernel_d(d):
    if d <= 0 or d > 128:
        raise InvalidValue(f"plain attention supports head dims up to 128 (got {d})")
    return 64 if d <= 64 else 128


def _pad(t, dk):
    return t if t.shape[-1] == dk else torch.nn.functional.pad(t, (0, dk - t.shape[-1]))


def _operands(*ts):
    from . import _lib
    in_dt = ts[0].dtype
    if in_dt not in _lib.DT_CODE or any(t.dtype != in_dt for t in ts):
        ts = tuple(t.float() for t in ts)
    return tuple(t.contiguous() for t in ts)


def _plain_forward_b200(q3, k3, v3, causal, dt):
    """The hand-written forward (aq_attn_fwd_plain) on [heads, n, d] operands,
    d padded to the kernel width -> (O in q's dtype, L fp32)."""
    from . import _lib
    lib = _lib.load()
    heads, n_q, d = q3.shape
    n_k = k3.shape[1]
    D = _kernel_d(d)
    q3, k3, v3 = (_pad(t, D) for t in _operands(q3, k3, v3))
    in_dt = q3.dtype
    ws = torch.empty(lib.aq_attn_fwd_workspace_bytes(heads, n_q, n_k, D, 1, 1), dtype=torch.uint8, device=q3.device)
    o = torch.empty((heads, n_q, D), dtype=in_dt, device=q3.device)
    lse = torch.empty((heads, n_q), dtype=torch.float32, device=q3.device)
    args = _lib.AqFwdArgs(q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[in_dt],
                          heads=heads, n_q=n_q, n_k=n_k, d=D, causal=int(causal), train=1,
                          o=o.data_ptr(), o_dtype=_lib.DT_CODE[o.dtype], o_hp=None, o_hp_dtype=0,
                          lse=lse.data_ptr(), workspace=ws.data_ptr(), keep_for_bwd=1, operands_staged=0,
                          softmax_scale=1.0 / math.sqrt(d))
    _lib.check(lib.aq_attn_fwd_plain(args, 0 if dt == torch.float16 else 1, _lib.stream_ptr()))
    return (o if D == d else o[..., :d].contiguous()), lse


def plain_forward(q3, k3, v3, causal):
    """q3 [heads, n_q, d], k3 / v3 [heads, n_k, d] CUDA -> (O [heads, n_q, d] in q's dtype, L fp32)."""
    if causal and q3.shape[1] > k3.shape[1]:
        raise ShapeError("causal attention requires N_q <= N_k")
    o, lse = _plain_forward_b200(q3, k3, v3, causal, _compute_dtype(q3, k3, v3))
    return o.to(q3.dtype) if o.dtype != q3.dtype else o, lse


def _fp16_gain(do3, v3, o3, d):
    """Exact power-of-two gain for dO in the fp16 backward: every fp16 operand
    it feeds stays in range -- dO itself and dS = P (dP - D) / sqrt(d), with
    |dS| <= sqrt(d) |dO| (|V| + |O|) -- while small values keep fp16's
    precision. The gradients are linear in dO, so dividing them by the gain is
    exact."""
    a_do = float(do3.abs().max()) if do3.numel() else 0.0
    if not (a_do > 0.0) or not math.isfinite(a_do):
        return 1.0
    a_vo = max(float(v3.abs().max()) + float(o3.abs().max()), 1e-30)
    k = min(math.floor(math.log2(2.0 ** 15 / (math.sqrt(d) * a_do * a_vo))), math.floor(math.log2(2.0 ** 15 / a_do)))
    return 2.0 ** max(-60, min(60, k))


def plain_backward(q3, k3, v3, do3, o_ref3, lse2, causal, grad_dtype=None):
    """Unquantized attention backward -> (dQ, dK, dV) [heads, n, d]
    (flash.py:317-390 with quantized=False) on aq_attn_bwd_plain, in the
    forward's 16-bit format (_compute_dtype on the same Q / K / V): fp16
    operands with an exact power-of-two gain on dO, or bf16."""
    from . import _lib
    lib = _lib.load()
    heads, n_q, d = q3.shape
    n_k = k3.shape[1]
    if causal and n_q > n_k:
        raise ShapeError("causal attention requires N_q <= N_k")
    fp16 = _compute_dtype(q3, k3, v3) == torch.float16
    gain = _fp16_gain(do3, v3, o_ref3, d) if fp16 else 1.0
    if gain != 1.0:
        do3 = do3.float() * gain
    D = _kernel_d(d)
    q3, k3, v3 = (_pad(t, D) for t in _operands(q3, k3, v3))
    do3, o_ref3 = (_pad(t, D) for t in _operands(do3, o_ref3))
    lse = lse2.reshape(heads, n_q).to(torch.float32).contiguous()
    g = grad_dtype or q3.dtype
    if gain != 1.0:
        g_out, g = g, torch.float32   # divide the gain out in fp32, then round once
    if g not in _lib.DT_CODE:
        raise InvalidValue(f"grad dtype {g} is not float32 / bfloat16 / float16")
    dq = torch.empty((heads, n_q, D), dtype=g, device=q3.device)
    dk = torch.empty((heads, n_k, D), dtype=g, device=q3.device)
    dv = torch.empty((heads, n_k, D), dtype=g, device=q3.device)
    ws = torch.empty(lib.aq_attn_bwd_workspace_bytes(heads, n_q, n_k, D), dtype=torch.uint8, device=q3.device)
    args = _lib.AqBwdArgs(
        q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[q3.dtype],
        d_o=do3.data_ptr(), do_dtype=_lib.DT_CODE[do3.dtype], o=o_ref3.data_ptr(), o_hp=None,
        o_dtype=_lib.DT_CODE[o_ref3.dtype], lse=lse.data_ptr(), heads=heads, n_q=n_q, n_k=n_k, d=D,
        causal=int(causal), variant=0, dq=dq.data_ptr(), dk=dk.data_ptr(), dv=dv.data_ptr(),
        g_dtype=_lib.DT_CODE[g], workspace=ws.data_ptr(), fwd_workspace=None, softmax_scale=1.0 / math.sqrt(d))
    _lib.check(lib.aq_attn_bwd_plain(args, 0 if fp16 else 1, _lib.stream_ptr()))
    if D != d:
        dq, dk, dv = (t[..., :d].contiguous() for t in (dq, dk, dv))
    if gain != 1.0:
        dq, dk, dv = ((t * (1.0 / gain)).to(g_out) for t in (dq, dk, dv))
    return dq, dk, dv
