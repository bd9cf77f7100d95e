"""``quantized=False``: plain (unquantized) attention, the reference's bf16 mode.

flash_forward_training / flash_backward with quantized=False skip every fake
quantization (flash.py:195-200, 344-349): O = O' = softmax(QK^T/sqrt(d)) V and
the textbook backward. The reference harness uses it for its "bf16" training
and evaluation mode (harness.py:40, 333-335). It is not the NVFP4 hot path, so
it runs on a library kernel -- FlashAttention-2 (flash_attn 2.8, like calling
cuBLAS) -- rather than on the hand-written tcgen05 kernels:

  * layout: our [heads, n, d] operands are viewed as FA2's [batch=heads, n,
    1 head, d] without a copy;
  * masking: FA2's causal mask is bottom-right aligned for n_q != n_k, which
    is the reference's right-aligned mask (oracle.py:62-75);
  * L: FA2's softmax LSE is the natural-log L of flash.py:217;
  * dtypes: FA2 computes in fp16 / bf16 with fp32 accumulation; fp32 inputs run
    in fp16 when they fit its range (else bf16) and results come back in the
    caller's dtype;
  * backward: D = rowsum(dO . O_ref) is computed by FA2 from the ``out`` it is
    given, so O_ref (O or O', identical here) is passed there
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
    dt = ts[0].dtype
    if dt in (torch.float16, torch.bfloat16):
        return dt
    if dt != torch.float32:
        raise InvalidValue("plain attention takes float32 / bfloat16 / float16 operands")
    amax = max(float(t.abs().max()) for t in ts if t.numel())
    return torch.float16 if amax < 6.0e4 else torch.bfloat16


def _fa_view(t, dt):
    # [heads, n, d] -> [heads, n, 1, d] (FA2 batch = heads, one head each)
    return t.to(dt).unsqueeze(2).contiguous()


def plain_forward(q3, k3, v3, causal):
    """q3 [heads, n_q, d], k3 / v3 [heads, n_k, d] CUDA -> (O [heads, n_q, d] in q's dtype, L fp32)."""
    if q3.shape[-1] % 8 or q3.shape[-1] > 256:
        raise InvalidValue("plain attention supports head dims that are multiples of 8, up to 256")
    if causal and q3.shape[1] > k3.shape[1]:
        raise ShapeError("causal attention requires N_q <= N_k")
    fa = _flash()
    dt = _compute_dtype(q3, k3, v3)
    scale = 1.0 / math.sqrt(q3.shape[-1])
    out, lse, _, _ = fa._flash_attn_forward(_fa_view(q3, dt), _fa_view(k3, dt), _fa_view(v3, dt), 0.0, scale,
                                             bool(causal), -1, -1, 0.0, None, False)
    return out.squeeze(2).to(q3.dtype), lse.squeeze(1).float()


def plain_backward(q3, k3, v3, do3, o_ref3, lse2, causal, grad_dtype=None):
    """Unquantized attention backward -> (dQ, dK, dV) [heads, n, d] (flash.py:317-390, quantized=False)."""
    fa = _flash()
    dt = _compute_dtype(q3, k3, v3, do3)
    q, k, v, do, o = (_fa_view(t, dt) for t in (q3, k3, v3, do3, o_ref3))
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    scale = 1.0 / math.sqrt(q3.shape[-1])
    lse = lse2.float().unsqueeze(1).contiguous()
    fa._flash_attn_backward(do, q, k, v, o, lse, dq, dk, dv, 0.0, scale, bool(causal), -1, -1, 0.0, None, True)
    g = grad_dtype or q3.dtype
    return dq.squeeze(2).to(g), dk.squeeze(2).to(g), dv.squeeze(2).to(g)
