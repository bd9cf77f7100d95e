"""``quantized=False``: plain (unquantized) attention, the reference's bf16 mode.

flash_forward_training / flash_backward with quantized=False skip every fake
quantization (flash.py:195-200, 344-349): O = O' = softmax(QK^T/sqrt(d)) V and
the textbook backward. The reference harness uses it for its "bf16" training
and evaluation mode (harness.py:40, 333-335).

* forward, d in {64, 128}: the hand-written K4 skeleton with 16-bit operands
  (``aq_attn_fwd_plain``): Q / K / V staged as fp16 (or bf16 when a value
  exceeds the fp16 range) T8x8 tiles, S and P^ V on ``kind::f16`` MMAs with
  fp32 accumulation, the two-pass softmax of the FP4 path (L final before the
  P V pass, 1/l in the epilogue);
* other head dims, and the backward: FlashAttention-2 (flash_attn 2.8, library
  kernels like cuBLAS). FA2's causal mask is bottom-right aligned for
  n_q != n_k, the reference's right-aligned mask (oracle.py:62-75); its LSE is
  the natural-log L of flash.py:217, so the backward consumes the forward's O
  and L directly; D = rowsum(dO . O_ref) from the ``out`` it is given
  (flash.py:333-351); deterministic mode, no atomics in dQ.
"""

from __future__ import annotations

import math

import torch

from .errors import InvalidValue, ShapeError

_fa = None


def _flash():
    global _fa
    if _fa is None:
        try:
            from flash_attn import flash_attn_interface as fa
        except ImportError as e:  # pragma: no cover - image ships flash_attn
            raise RuntimeError("quantized=False needs the flash_attn package (FlashAttention-2)") from e
        _fa = fa
    return _fa


def _compute_dtype(*ts):
    """16-bit operand format for float32 Q / K / V: fp16 (11-bit significand)
    when the largest magnitude sits inside its normal range with headroom
    (2^-10 <= amax < 6e4), else bf16 (fp32's exponent range). The forward and
    the backward call this on the same Q / K / V, so they agree."""
    dt = ts[0].dtype
    if dt in (torch.float16, torch.bfloat16):
        return dt
    if dt != torch.float32:
        raise InvalidValue("plain attention takes float32 / bfloat16 / float16 operands")
    amax = max(float(t.abs().max()) for t in ts if t.numel())
    return torch.float16 if 2.0 ** -10 <= amax < 6.0e4 else torch.bfloat16


def _pow2_gain(t, dt, target=2.0 ** 10):
    """Exact power-of-two gain that moves t's largest magnitude near ``target``
    when t is cast to fp16 (dO of a mean loss is often far below fp16's normal
    range); gradients are linear in dO, so dividing them by the gain is exact."""
    if dt != torch.float16 or t.numel() == 0:
        return 1.0
    amax = float(t.abs().max())
    if not (amax > 0.0) or not math.isfinite(amax):
        return 1.0
    return 2.0 ** max(-60, min(60, math.floor(math.log2(target / amax))))


def _fa_view(t, dt):
    # [heads, n, d] -> [heads, n, 1, d] (FA2 batch = heads, one head each)
    return t.to(dt).unsqueeze(2).contiguous()


def _plain_forward_b200(q3, k3, v3, causal, dt):
    """The hand-written path (aq_attn_fwd_plain): K4's skeleton with 16-bit
    operands, S and P^V on kind::f16 MMAs, fp32 softmax statistics."""
    from . import _lib
    lib = _lib.load()
    heads, n_q, d = q3.shape
    n_k = k3.shape[1]
    in_dt = q3.dtype
    if in_dt not in _lib.DT_CODE or k3.dtype != in_dt or v3.dtype != in_dt:
        q3, k3, v3 = q3.float(), k3.float(), v3.float()
        in_dt = torch.float32
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    ws = torch.empty(lib.aq_attn_fwd_workspace_bytes(heads, n_q, n_k, d, 1, 1), dtype=torch.uint8, device=q3.device)
    o = torch.empty((heads, n_q, d), dtype=q3.dtype, device=q3.device)
    lse = torch.empty((heads, n_q), dtype=torch.float32, device=q3.device)
    args = _lib.AqFwdArgs(q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[in_dt],
                          heads=heads, n_q=n_q, n_k=n_k, d=d, causal=int(causal), train=1,
                          o=o.data_ptr(), o_dtype=_lib.DT_CODE[o.dtype], o_hp=None, o_hp_dtype=0,
                          lse=lse.data_ptr(), workspace=ws.data_ptr(), keep_for_bwd=1, operands_staged=0)
    _lib.check(lib.aq_attn_fwd_plain(args, 0 if dt == torch.float16 else 1, _lib.stream_ptr()))
    return o, lse


def plain_forward(q3, k3, v3, causal):
    """q3 [heads, n_q, d], k3 / v3 [heads, n_k, d] CUDA -> (O [heads, n_q, d] in q's dtype, L fp32).

    Head dims 64 / 128 run on the hand-written sm_100a kernel; other head dims
    (multiples of 8 up to 256) on FlashAttention-2."""
    if causal and q3.shape[1] > k3.shape[1]:
        raise ShapeError("causal attention requires N_q <= N_k")
    if q3.shape[-1] in (64, 128):
        return _plain_forward_b200(q3, k3, v3, causal, _compute_dtype(q3, k3, v3))
    if q3.shape[-1] % 8 or q3.shape[-1] > 256:
        raise InvalidValue("plain attention supports head dims that are multiples of 8, up to 256")
    fa = _flash()
    dt = _compute_dtype(q3, k3, v3)
    scale = 1.0 / math.sqrt(q3.shape[-1])
    out, lse, _, _ = fa._flash_attn_forward(_fa_view(q3, dt), _fa_view(k3, dt), _fa_view(v3, dt), 0.0, scale,
                                             bool(causal), -1, -1, 0.0, None, False)
    return out.squeeze(2).to(q3.dtype), lse.squeeze(1).float()


def plain_backward(q3, k3, v3, do3, o_ref3, lse2, causal, grad_dtype=None):
    """Unquantized attention backward -> (dQ, dK, dV) [heads, n, d] (flash.py:317-390, quantized=False)."""
    fa = _flash()
    dt = _compute_dtype(q3, k3, v3)   # the forward's choice (same Q / K / V)
    gain = _pow2_gain(do3, dt)
    q, k, v, o = (_fa_view(t, dt) for t in (q3, k3, v3, o_ref3))
    do = _fa_view(do3 * gain if gain != 1.0 else do3, dt)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    scale = 1.0 / math.sqrt(q3.shape[-1])
    lse = lse2.float().unsqueeze(1).contiguous()
    fa._flash_attn_backward(do, q, k, v, o, lse, dq, dk, dv, 0.0, scale, bool(causal), -1, -1, 0.0, None, True)
    g = grad_dtype or q3.dtype
    inv = 1.0 / gain
    return tuple((t.squeeze(2).float() * inv).to(g) if gain != 1.0 else t.squeeze(2).to(g) for t in (dq, dk, dv))
