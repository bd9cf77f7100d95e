"""``torch.autograd.Function`` for NVFP4 Attn-QAT attention on [..., N, d] CUDA tensors.

Forward = flash_forward_training (O is the FP4-path output that flows to the
next layer; O' and L are saved). Backward = flash_backward with the chosen
BwdVariant: D = rowsum(dO . O'), P recomputed at forward precision and
re-quantized for dV, straight-through gradients for Q/K/V (flash.py:317-390).
The quantized operands staged by the forward are kept in a workspace and
reused by the backward instead of re-quantizing.
"""

from __future__ import annotations

import torch

from .flash import BwdVariant, attn_backward, attn_forward, attn_forward_mx, check_nonfinite


class AttnQATFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, causal=False, variant=BwdVariant.CORRECT, quantized=True, mx=False, scales=None,
                check_finite=False):
        scales = dict(scales or {})
        if quantized and mx:   # MXFP4: the staged operands are kept for the backward too
            o, lse, o_hp, ws = attn_forward_mx(q, k, v, causal=causal, train=True, keep_for_bwd=True)
        else:
            o, lse, o_hp, ws = attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True,
                                            quantized=quantized, **scales)
        if check_finite and quantized and not mx:
            check_nonfinite(q.device)  # one host read: NaN / Inf in Q, K or V raise InvalidValue
        ctx.save_for_backward(q, k, v, o, o_hp, lse, ws)
        ctx.causal = causal
        ctx.variant = variant
        ctx.quantized = quantized
        ctx.mx = quantized and mx
        ctx.scales = scales
        return o

    @staticmethod
    def backward(ctx, d_o):
        q, k, v, o, o_hp, lse, ws = ctx.saved_tensors
        extra = ctx.scales if (ctx.quantized and not ctx.mx) else {}
        dq, dk, dv = attn_backward(q, k, v, d_o.contiguous(), o, o_hp, lse, causal=ctx.causal,
                                   variant=ctx.variant, grad_dtype=q.dtype,
                                   fwd_workspace=ws, quantized=ctx.quantized, mx=ctx.mx, **extra)
        return dq, dk, dv, None, None, None, None, None, None


def attn_qat(q, k, v, causal=False, variant=BwdVariant.CORRECT, quantized=True, spec=None, softmax_scale=None,
             q_scale=None, k_scale=None, v_scale=None, p_scale=None, check_finite=False):
    """NVFP4 QAT attention: O = softmax_fq(Q^F K^F^T / sqrt(d)) V^F with the Attn-QAT backward.
    ``spec=MXFP4`` runs the MXFP4 format (UE8M0 scales per 32 elements);
    ``quantized=False`` is the reference's bf16 mode (plain attention, plain.py).
    The optional scales are attn_forward's two-level NVFP4 extension (None =
    the reference's semantics); 'auto' tensor scales are resolved once here so
    the backward reuses the forward's values. ``check_finite`` raises
    InvalidValue on NaN / Inf operands (one host read per call)."""
    from .codec import MXFP4, auto_tensor_scale
    scales = {}
    for name, val, t in (("q_scale", q_scale, q), ("k_scale", k_scale, k), ("v_scale", v_scale, v)):
        if val is not None:
            scales[name] = auto_tensor_scale(t) if isinstance(val, str) and val == "auto" else float(val)
    if softmax_scale is not None:
        scales["softmax_scale"] = float(softmax_scale)
    if p_scale is not None:
        scales["p_scale"] = float(p_scale)
    return AttnQATFunction.apply(q, k, v, causal, variant, quantized, spec == MXFP4, scales, check_finite)
