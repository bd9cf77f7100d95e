"""SageAttention3-style outlier heuristics as toggles (reference: attnqat/sage3.py).

``sage3_forward`` is the reference's real-quant tiled attention with

* Q / K smoothing: gamma_q = Q - (per-b_q-tile token mean), gamma_k = K -
  (global token mean) (sage3.py:45-60); only the zero-mean residuals pass
  through FP4;
* the exact score decomposition S = fp4(gamma_q) fp4(gamma_k)^T + q_bar
  gamma_k^T + [q_bar k_bar + gamma_q k_bar] (sage3.py:74-88), the two
  correction terms added to the scores in fp32 and never quantized;
* two-level P: every row of every b_k key segment is rescaled onto
  [0, 448*6] before NVFP4 block quantization and the product divided back
  (sage3.py:98-110, 186-190).

On the B200 the pre-processing (means in fp64, centring, the delta / bias
terms) runs in csrc/sage3.cu and the attention in the K4 kernel's SAGE
instances (csrc/attn_fwd.cu): the delta / bias terms are added to the S tile
after the FP4 MMA in both passes; two-level P quantizes P * r in registers and
accumulates dequant(P^F) * l / r through the f16 MMA (the per-segment 1/r is
applied before the accumulation). Segment maxima: in registers for b_k in
{16, 32, 64} and via a shared-memory exchange for 128; from the exact pass-1
row max when b_k == n_k; otherwise pass 1 reduces them per (row, segment)
into an HBM scratch with atomicMax. ``quantized=False`` is plain attention (the heuristics are exact no-ops
in exact arithmetic, sage3.py:117-120) and runs on the plain path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .codec import to_device
from .errors import InvalidValue, ShapeError
from .flash import AttnOutputs, _check_attention_shapes, _check_cfg, _heads_view, _np_out, _plain_forward

P_RESCALE_MAX = 448.0 * 6.0  # sage3.py:27 (max E4M3 scale x max FP4 value)


# ----------------------------------------------------------------------------
# the reference's composable pieces (sage3.py:30-110), as device ops; NumPy in
# gives NumPy out. The fused forward below does not call them -- it computes
# the same quantities inside csrc/sage3.cu and the K4 SAGE instance.
# ----------------------------------------------------------------------------

@dataclass
class SmoothedPair:
    """Token-mean-removed Q and K plus the removed means (sage3.py:30-42):
    q_bar one mean row per query tile (t_q, d), k_bar the global key mean (d,)."""

    gamma_q: object
    gamma_k: object
    q_bar: object
    k_bar: object
    b_q: int


def _dev64(x):
    as_np = not isinstance(x, torch.Tensor)
    t = torch.as_tensor(np.asarray(x)) if as_np else x
    return t.to("cuda"), as_np


def _host_like(t, as_np):
    return t.cpu().numpy() if as_np else t


def smooth(Q, K, b_q):
    """Subtract token-dimension means: per b_q tile from Q, globally from K
    (sage3.py:45-60). Means in float64 on the device; gamma keeps the promoted
    dtype of (input, float64 mean) as NumPy does."""
    _lib.require_cuda()
    q, as_np = _dev64(Q)
    k, _ = _dev64(K)
    if q.dim() != 2 or k.dim() != 2 or q.shape[1] != k.shape[1]:
        raise ShapeError("smooth expects 2-D Q and K with matching head dim")
    if b_q <= 0 or q.shape[0] % b_q:
        raise ShapeError(f"b_q ({b_q}) must divide N_q ({q.shape[0]})")
    t_q = q.shape[0] // b_q
    q_bar = q.reshape(t_q, b_q, -1).to(torch.float64).mean(dim=1)
    k_bar = k.to(torch.float64).mean(dim=0)
    gamma_q = q - q_bar.repeat_interleave(b_q, dim=0)
    gamma_k = k - k_bar
    return SmoothedPair(gamma_q=_host_like(gamma_q, as_np), gamma_k=_host_like(gamma_k, as_np),
                        q_bar=_host_like(q_bar, as_np), k_bar=_host_like(k_bar, as_np), b_q=b_q)


@dataclass
class ScoreDecomposition:
    """S_ij = main + delta_s + bias, exactly in exact arithmetic (sage3.py:63-71)."""

    main: object     # gamma(Q_i) gamma(K_j)^T, the only FP4-bound term
    delta_s: object  # q_bar_i gamma(K_j)^T, (1, b_k), broadcast down the rows
    bias: object     # q_bar_i k_bar^T + gamma(Q_i) k_bar^T, (b_q, 1)

    def reconstruct(self):
        return self.main + self.delta_s + self.bias


def decompose_scores(pair, i, j, b_k, accum_width=64):
    """Score decomposition for query tile i against key tile j (sage3.py:74-88),
    the products on the device in the accumulation width (tensors.matmul)."""
    from .tensors import matmul
    gq = pair.gamma_q[i * pair.b_q:(i + 1) * pair.b_q]
    gk = pair.gamma_k[j * b_k:(j + 1) * b_k]
    if min(int(np.prod(gq.shape)), int(np.prod(gk.shape))) == 0:
        raise ShapeError("tile indices out of range")
    qb = pair.q_bar[i]
    main = matmul(gq, gk.T, accum_width)
    delta_s = matmul(qb[None, :], gk.T, accum_width)
    bias = matmul(qb[None, :], pair.k_bar[:, None], accum_width) + matmul(gq, pair.k_bar[:, None], accum_width)
    return ScoreDecomposition(main=main, delta_s=delta_s, bias=bias)


@dataclass
class TwoLevelP:
    """Row-rescaled quantized probabilities plus the per-row factor (sage3.py:91-95)."""

    codes: object  # QuantTensor of quantize_padded(P * r)
    row_factor: object


def quantize_p_two_level(P_tile, spec=None):
    """Rescale each row of P onto [0, 448*6], then block-quantize with the GPU
    codec (sage3.py:98-110); rows of zeros keep factor 1. The scaled tile is
    rounded to float32 before the codec (codec.to_device), which only matters
    for values within one fp32 ulp of an E2M1 / E4M3 rounding midpoint."""
    from .codec import NVFP4, quantize_padded
    spec = spec or NVFP4
    _lib.require_cuda()
    p, as_np = _dev64(P_tile)
    p = p.to(torch.float64)
    if p.dim() != 2:
        raise ShapeError("quantize_p_two_level expects a 2-D tile")
    if bool((p < 0).any()):
        raise InvalidValue("two-level quantization expects non-negative P")
    rowmax = p.max(dim=1).values
    r = torch.where(rowmax > 0, P_RESCALE_MAX / torch.where(rowmax > 0, rowmax, torch.ones_like(rowmax)),
                    torch.ones_like(rowmax))
    scaled = torch.clamp(p * r[:, None], max=P_RESCALE_MAX).to(torch.float32)
    qt = quantize_padded(scaled.cpu().numpy() if as_np else scaled, spec)
    return TwoLevelP(codes=qt, row_factor=_host_like(r, as_np))


def attn_forward_sage3(q, k, v, causal=False, b_q=128, b_k=128, smooth_q=True, smooth_k=True, two_level_p=True,
                       quantized=True, out_dtype=None, workspace=None):
    """sage3_forward on CUDA tensors [..., N, d] -> (O, L)."""
    _lib.require_cuda()
    if not quantized:
        o, lse, _, _ = _plain_forward(q, k, v, causal, False, out_dtype)
        return o, lse
    q3, n_q, d = _heads_view(q)
    k3, n_k, dk = _heads_view(k)
    v3, n_v, dv = _heads_view(v)
    if dk != d or dv != d or n_v != n_k or k3.shape[0] != q3.shape[0] or v3.shape[0] != q3.shape[0]:
        raise ShapeError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} V{tuple(v.shape)}")
    dt = q.dtype
    if k.dtype != dt or v.dtype != dt or dt not in _lib.DT_CODE:
        raise InvalidValue("q, k, v must share a float32 / bfloat16 / float16 dtype")
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    heads = q3.shape[0]
    out_dtype = out_dtype or dt
    lib = _lib.load()
    ws_bytes = lib.aq_attn_fwd_sage3_workspace_bytes(heads, n_q, n_k, d, b_q, b_k) if b_q > 0 and n_q % b_q == 0 else 0
    if ws_bytes <= 0 and d in (64, 128) and n_q > 0 and n_k > 0:
        ws_bytes = 256  # the entry point reports the tile error
    if ws_bytes <= 0:
        raise InvalidValue(f"unsupported shape (heads {heads}, n_q {n_q}, n_k {n_k}, d {d})")
    ws = workspace if workspace is not None and workspace.numel() >= ws_bytes else \
        torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    o = torch.empty((heads, n_q, d), dtype=out_dtype, device=q.device)
    lse = torch.empty((heads, n_q), dtype=torch.float32, device=q.device)
    args = _lib.AqSage3Args(
        q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[dt],
        heads=heads, n_q=n_q, n_k=n_k, d=d, causal=int(causal), b_q=b_q, b_k=b_k,
        smooth_q=int(smooth_q), smooth_k=int(smooth_k), two_level_p=int(two_level_p),
        o=o.data_ptr(), o_dtype=_lib.DT_CODE[out_dtype], lse=lse.data_ptr(), workspace=ws.data_ptr())
    _lib.check(lib.aq_attn_fwd_sage3(args, _lib.stream_ptr()))
    lead = q.shape[:-2]
    return o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q)


def sage3_forward(Q, K, V, cfg, smooth_q=True, smooth_k=True, two_level_p=True, quantized=True):
    """Real-quant tiled attention with the outlier heuristics (sage3.py:113-194)
    -> AttnOutputs(O, L, O_prime=None). NumPy in, NumPy out; CUDA tensors stay
    on the device."""
    n_q, n_k, d = _check_attention_shapes(Q, K, V)
    _check_cfg(cfg, n_q, n_k, d, quantized)
    if cfg.b_q <= 0 or n_q % cfg.b_q:
        raise ShapeError(f"b_q ({cfg.b_q}) must divide N_q ({n_q})")  # sage3.py:50-53
    if quantized:
        from .flash import _check_finite
        _check_finite(Q, K, V)
    q, as_np = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    o, lse = attn_forward_sage3(q, k, v, causal=cfg.causal, b_q=cfg.b_q, b_k=cfg.b_k, smooth_q=smooth_q,
                                smooth_k=smooth_k, two_level_p=two_level_p, quantized=quantized,
                                out_dtype=torch.float32 if as_np else None)
    if as_np:
        import numpy as np
        return AttnOutputs(O=_np_out(o, True), L=_np_out(lse, True, np.float64), O_prime=None)
    return AttnOutputs(O=o, L=lse, O_prime=None)
