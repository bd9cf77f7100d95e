"""Fused NVFP4 Attn-QAT attention, mirroring ``attnqat.flash`` (flash.py:50-390).

``flash_forward_training`` / ``flash_forward_inference`` / ``flash_backward``
keep the reference names, arguments, return types and exceptions. Besides the
reference's 2-D per-head (N, d) operands they accept batched [..., N, d]
torch tensors (leading dims are flattened into heads, every head independent).

Differences from the CPU reference, by design of the B200 path:
  * tiles are fixed at 128 x 128 inside the kernels; ``TileConfig`` is still
    validated exactly as the reference does (results are tiling-invariant,
    test_flash.py:72-84) and b_q / b_k are otherwise ignored;
  * accumulation is fp32 on the tensor cores (``accum_width=64`` raises
    InvalidValue); ``threads`` is accepted and ignored; ``instrument`` records
    are rebuilt from the kernels' P^F dump (see _instrument_*).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .codec import NVFP4, BlockSpec, to_device
from .host import default_chunk, run_pipelined
from .plain import plain_backward, plain_forward
from .errors import InvalidValue, MissingOPrime, ShapeError, TileError


@dataclass(frozen=True)
class TileConfig:
    """Tile row counts plus the numeric knobs (flash.py:50-71)."""

    b_q: int
    b_k: int
    causal: bool = False
    accum_width: int = 32
    spec: BlockSpec = NVFP4

    def validate(self, n_q, n_k, quantized):
        if self.b_q <= 0 or self.b_k <= 0:
            raise TileError("tile sizes must be positive")
        if n_q % self.b_q or n_k % self.b_k:
            raise TileError(f"tiles ({self.b_q}, {self.b_k}) must divide ({n_q}, {n_k})")
        if quantized and n_k > self.b_k and self.b_k % self.spec.block_size:
            raise TileError("b_k must be a multiple of the block size so probability blocks align across tiles")


@dataclass
class AttnOutputs:
    """O and the log-sum-exp L; O_prime only in training mode (flash.py:74-80)."""

    O: object
    L: object
    O_prime: object = None


@dataclass
class RowState:
    """Online-softmax state after one key tile (flash.py:98-114), instrumented mode."""

    i_tile: int
    j_tile: int
    m: np.ndarray
    l: np.ndarray

    def to_json_dict(self):
        return {"kind": "row_state", "i_tile": self.i_tile, "j_tile": self.j_tile,
                "m": self.m.tolist(), "l": self.l.tolist()}


@dataclass
class PTileRecord:
    """Quantized probability tile captured by instrumented runs (flash.py:117-124)."""

    phase: str  # "forward" or "backward"
    i_tile: int
    j_tile: int
    P_fq: np.ndarray


@dataclass
class AttnGrads:
    """oracle.py:134-138."""

    dQ: object
    dK: object
    dV: object


class BwdVariant(Enum):
    """flash.py:83-95."""

    CORRECT = "correct"
    LOW_PREC_O = "lowpreco"
    NO_FAKE_QUANT_P = "nofqp"
    NAIVE_BF16_BWD = "naive-bf16-bwd"

    @property
    def uses_o_prime(self):
        return self in (BwdVariant.CORRECT, BwdVariant.NO_FAKE_QUANT_P)

    @property
    def fake_quantizes_p(self):
        return self in (BwdVariant.CORRECT, BwdVariant.LOW_PREC_O)

    @property
    def code(self):
        return {BwdVariant.CORRECT: 0, BwdVariant.LOW_PREC_O: 1,
                BwdVariant.NO_FAKE_QUANT_P: 2, BwdVariant.NAIVE_BF16_BWD: 3}[self]


# ----------------------------------------------------------------------------
# batched device entry points (what the autograd Function and benches call)
# ----------------------------------------------------------------------------

def _heads_view(t):
    if t.dim() < 2:
        raise ShapeError("attention operands need at least 2 dims (n, d)")
    n, d = t.shape[-2:]
    return t.reshape(-1, n, d), n, d


def kernel_head_dim(d):
    """Head dim the sm_100a kernels run for a given d: 64 / 128 natively, any
    other multiple of 16 below 128 zero-padded up (flash.py:185-188 accepts any
    d % 16 == 0). Padding is exact: zero Q/K columns add 0 to S, zero V
    columns give zero O columns, and the softmax scale stays 1/sqrt(d)."""
    if d in (64, 128):
        return d
    if d % 16 == 0 and 0 < d < 128:
        return 64 if d < 64 else 128
    raise InvalidValue(f"unsupported head dim {d} (the B200 kernels take d % 16 == 0, d <= 128)")


def _pad_d(t, dk):
    return t if t.shape[-1] == dk else torch.nn.functional.pad(t, (0, dk - t.shape[-1]))


_NONFINITE = {}


def nonfinite_flag(device=None):
    """Per-device int32 flag the quantizers OR with 1 on NaN / Inf input
    (codec.py:313-314); attn_forward / attn_backward pass it by default."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    f = _NONFINITE.get(dev.index)
    if f is None:
        f = _NONFINITE[dev.index] = torch.zeros(1, dtype=torch.int32, device=dev)
    return f


def check_nonfinite(device=None, reset=True):
    """Raise InvalidValue if any quantizer on ``device`` saw NaN / Inf since the
    last check (the reference raises at quantize time, codec.py:313-314). Reads
    one int from the device (a host synchronisation)."""
    f = nonfinite_flag(device)
    bad = bool(f.item())
    if reset and bad:
        f.zero_()
    if bad:
        raise InvalidValue("quantize requires finite input (NaN / Inf in Q, K or V)")


def _scale(x, what):
    if x is None:
        return 0.0  # the C ABI's "1.0 / reference semantics"
    x = float(x)
    if not (x > 0 and np.isfinite(x)):
        raise InvalidValue(f"{what} must be positive and finite, got {x}")
    return x


def _resolve_tensor_scales(q, k, v, q_scale, k_scale, v_scale):
    from .codec import auto_tensor_scale
    out = []
    for t, s in ((q, q_scale), (k, k_scale), (v, v_scale)):
        out.append(auto_tensor_scale(t) if isinstance(s, str) and s == "auto" else s)
    return out


def _check_out(t, shape, dtype, device, what):
    """caller-supplied outputs must match what the kernel writes."""
    if t is None:
        return
    if tuple(t.shape) != tuple(shape) and t.numel() != int(np.prod(shape)):
        raise ShapeError(f"{what} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise InvalidValue(f"{what} has dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise InvalidValue(f"{what} must be contiguous")
    if t.device != device:
        raise InvalidValue(f"{what} is on {t.device}, expected {device}")


def _check_pf_out(pf_out, heads, n_q, n_k):
    if pf_out is None:
        return None, None
    n16 = -(-n_k // 16) * 16
    pf_c, pf_s = pf_out
    if pf_c.dtype != torch.uint8 or pf_s.dtype != torch.uint8 or pf_c.numel() != heads * n_q * n16 // 2 \
            or pf_s.numel() != heads * n_q * n16 // 16 or not (pf_c.is_contiguous() and pf_s.is_contiguous()):
        raise ShapeError("pf_out must be contiguous uint8 (codes [heads, n_q, n16/2], scales [heads, n_q, n16/16])")
    return pf_c, pf_s


def pf_buffers(heads, n_q, n_k, device=None):
    """Zeroed (codes, scales) buffers for ``pf_out``: P^F of every row in the
    reference's quantize_padded(P) layout; unvisited (fully masked) blocks stay 0."""
    n16 = -(-n_k // 16) * 16
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return (torch.zeros((heads, n_q, n16 // 2), dtype=torch.uint8, device=dev),
            torch.zeros((heads, n_q, n16 // 16), dtype=torch.uint8, device=dev))


def attn_forward(q, k, v, causal=False, train=True, out_dtype=None, keep_for_bwd=False, lse_out=None,
                 workspace=None, operands_staged=False, out=None, o_hp_out=None, quantized=True,
                 softmax_scale=None, q_scale=None, k_scale=None, v_scale=None, p_scale=None, nonfinite=None,
                 pf_out=None):
    """Fused forward on CUDA tensors [..., N, d] -> (O, L, O_hp or None, workspace).

    ``train=True`` is flash_forward_training (O, L, O'), ``False`` is
    flash_forward_inference (O, L). O is the FP4-path output, O' the
    high-precision output the QAT backward needs (flash.py:176-246).
    ``quantized=False`` is plain attention (O' = O; plain.py).

    Beyond the reference (all default to its semantics, bit for bit):
    ``softmax_scale`` (default 1/sqrt(d)); ``q_scale`` / ``k_scale`` /
    ``v_scale`` per-tensor FP32 scales of the two-level NVFP4 format (a float
    or 'auto' = amax / 2688); ``p_scale`` the P tensor scale (e.g. 1/2688 keeps
    long rows above the E4M3 floor; not parity); ``nonfinite`` an int32 device
    flag (default: the per-device one, see check_nonfinite); ``pf_out`` =
    (codes [.., n_q, n16/2] u8, scales [.., n_q, n16/16] u8) receives P^F of
    every row in the reference's quantize_padded(P) layout (instrument)."""
    _lib.require_cuda()
    if q.device.type == "cuda" and q.device.index is not None and q.device.index != torch.cuda.current_device():
        with torch.cuda.device(q.device):  # launch on (and with the current stream of) q's device
            return attn_forward(q, k, v, causal, train, out_dtype, keep_for_bwd, lse_out, workspace,
                                operands_staged, out, o_hp_out, quantized, softmax_scale, q_scale, k_scale,
                                v_scale, p_scale, nonfinite, pf_out)
    if not quantized:
        return _plain_forward(q, k, v, causal, train, out_dtype)
    q3, n_q, d = _heads_view(q)
    k3, n_k, dk_ = _heads_view(k)
    v3, n_v, dv_ = _heads_view(v)
    if dk_ != d or dv_ != d or n_v != n_k or k3.shape[0] != q3.shape[0] or v3.shape[0] != q3.shape[0]:
        raise ShapeError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} V{tuple(v.shape)}")
    if d % 16:
        raise ShapeError("d must be a multiple of the block size when quantizing")
    if causal and n_q > n_k:
        raise ShapeError("causal attention requires N_q <= N_k")
    dt = q.dtype
    if k.dtype != dt or v.dtype != dt or dt not in _lib.DT_CODE:
        raise InvalidValue("q, k, v must share a float32 / bfloat16 / float16 dtype")
    D = kernel_head_dim(d)
    heads = q3.shape[0]
    out_dtype = out_dtype or dt
    if out_dtype not in _lib.DT_CODE:
        raise InvalidValue(f"out_dtype must be float32 / bfloat16 / float16, got {out_dtype}")
    _check_out(out, (heads, n_q, d), out_dtype, q.device, "out")
    _check_out(o_hp_out, (heads, n_q, d), out_dtype, q.device, "o_hp_out")
    _check_out(lse_out, (heads, n_q), torch.float32, q.device, "lse_out")
    if softmax_scale is None and D != d:
        softmax_scale = 1.0 / float(np.sqrt(d))
    q_scale, k_scale, v_scale = _resolve_tensor_scales(q, k, v, q_scale, k_scale, v_scale)
    q3, k3, v3 = (_pad_d(t.contiguous(), D) for t in (q3, k3, v3))
    lib = _lib.load()
    ws_bytes = lib.aq_attn_fwd_workspace_bytes(heads, n_q, n_k, D, int(train), int(keep_for_bwd))
    if ws_bytes <= 0:
        raise InvalidValue(f"unsupported attention shape (heads={heads}, n_q={n_q}, n_k={n_k}, d={d})")
    if workspace is not None:
        if workspace.numel() < ws_bytes:
            raise ShapeError("workspace too small")
        ws = workspace
    else:
        if operands_staged:
            raise InvalidValue("operands_staged needs the workspace that holds them")
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    padded = D != d
    o = out.view(heads, n_q, d) if (out is not None and not padded) else \
        torch.empty((heads, n_q, D), dtype=out_dtype, device=q.device)
    o_hp = None
    if train:
        o_hp = o_hp_out.view(heads, n_q, d) if (o_hp_out is not None and not padded) else \
            torch.empty((heads, n_q, D), dtype=out_dtype, device=q.device)
    lse = lse_out.view(heads, n_q) if lse_out is not None else \
        torch.empty((heads, n_q), dtype=torch.float32, device=q.device)
    pf_c, pf_s = _check_pf_out(pf_out, heads, n_q, n_k)
    flag = nonfinite if nonfinite is not None else nonfinite_flag(q.device)
    args = _lib.AqFwdArgs(
        q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[dt],
        heads=heads, n_q=n_q, n_k=n_k, d=D, causal=int(causal), train=int(train),
        o=o.data_ptr(), o_dtype=_lib.DT_CODE[out_dtype],
        o_hp=o_hp.data_ptr() if o_hp is not None else None, o_hp_dtype=_lib.DT_CODE[out_dtype],
        lse=lse.data_ptr(), workspace=ws.data_ptr(), keep_for_bwd=int(keep_for_bwd),
        operands_staged=int(operands_staged),
        softmax_scale=_scale(softmax_scale, "softmax_scale"), q_scale=_scale(q_scale, "q_scale"),
        k_scale=_scale(k_scale, "k_scale"), v_scale=_scale(v_scale, "v_scale"), p_scale=_scale(p_scale, "p_scale"),
        nonfinite=flag.data_ptr(), pf_codes=pf_c.data_ptr() if pf_c is not None else None,
        pf_scales=pf_s.data_ptr() if pf_s is not None else None)
    _lib.check(lib.aq_attn_fwd(args, _lib.stream_ptr()))
    ws._aq_meta = ("nvfp4", bool(keep_for_bwd), heads, n_q, n_k, D)
    if padded:
        o = o[..., :d]
        o_hp = o_hp[..., :d] if o_hp is not None else None
        if out is not None:
            out.view(heads, n_q, d).copy_(o)
            o = out
        else:
            o = o.contiguous()
        if o_hp is not None:
            if o_hp_out is not None:
                o_hp_out.view(heads, n_q, d).copy_(o_hp)
                o_hp = o_hp_out
            else:
                o_hp = o_hp.contiguous()
    lead = q.shape[:-2]
    return (o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q),
            o_hp.reshape(*lead, n_q, d) if o_hp is not None else None, ws)


def attn_backward(q, k, v, d_o, o, o_hp, lse, causal=False, variant=BwdVariant.CORRECT, grad_dtype=None,
                  fwd_workspace=None, workspace=None, grads_out=None, quantized=True, mx=False,
                  softmax_scale=None, q_scale=None, k_scale=None, v_scale=None, p_scale=None, nonfinite=None,
                  pf_out=None):
    """Fused QAT backward on CUDA tensors -> (dQ, dK, dV) (flash.py:317-390).
    The scale arguments must repeat the forward's; ``pf_out`` (as for
    attn_forward) receives the backward's own recomputed P^F (instrument)."""
    _lib.require_cuda()
    if q.device.type == "cuda" and q.device.index is not None and q.device.index != torch.cuda.current_device():
        with torch.cuda.device(q.device):
            return attn_backward(q, k, v, d_o, o, o_hp, lse, causal, variant, grad_dtype, fwd_workspace,
                                 workspace, grads_out, quantized, mx, softmax_scale, q_scale, k_scale, v_scale,
                                 p_scale, nonfinite, pf_out)
    q3, n_q, d = _heads_view(q)
    k3, n_k, dk_ = _heads_view(k)
    v3, n_v, dv_ = _heads_view(v)
    heads = q3.shape[0]
    if dk_ != d or dv_ != d or n_v != n_k or k3.shape[0] != heads or v3.shape[0] != heads:
        raise ShapeError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} V{tuple(v.shape)}")
    if causal and n_q > n_k:
        raise ShapeError("causal attention requires N_q <= N_k")
    if tuple(d_o.shape) != tuple(q.shape):
        raise ShapeError(f"dO shape {tuple(d_o.shape)} does not match Q {tuple(q.shape)}")
    if variant.uses_o_prime and o_hp is None:
        raise MissingOPrime(f"variant {variant.value} needs O_prime; run the training forward")
    o_ref = o_hp if variant.uses_o_prime else o
    if o_ref is None:
        raise ShapeError("the forward output O is required")
    for t, what in ((o, "O"), (o_hp, "O_prime")):
        if t is not None and t.numel() != heads * n_q * d:
            raise ShapeError(f"{what} has the wrong shape {tuple(t.shape)}")
    if lse.numel() != heads * n_q:
        raise ShapeError("outs.L has the wrong shape")
    dt = q.dtype
    if k.dtype != dt or v.dtype != dt or dt not in _lib.DT_CODE:
        raise InvalidValue("q, k, v must share a float32 / bfloat16 / float16 dtype")
    if d_o.dtype not in _lib.DT_CODE:
        raise InvalidValue(f"dO dtype {d_o.dtype} is not float32 / bfloat16 / float16")
    grad_dtype = grad_dtype or q.dtype
    if not quantized:
        # every variant reduces to the plain backward (flash.py:344-349, 357)
        g = plain_backward(q3.contiguous(), k3.contiguous(), v3.contiguous(), d_o.reshape(heads, n_q, d),
                           o_ref.reshape(heads, n_q, d), lse.reshape(heads, n_q), causal, grad_dtype)
        return (g[0].reshape(q.shape[:-2] + (n_q, d)), g[1].reshape(k.shape[:-2] + (n_k, d)),
                g[2].reshape(v.shape[:-2] + (n_k, d)))
    if d % 16:
        raise ShapeError("d must be a multiple of the block size when quantizing")
    D = kernel_head_dim(d)
    if softmax_scale is None and D != d:
        softmax_scale = 1.0 / float(np.sqrt(d))
    lib = _lib.load()
    if fwd_workspace is not None:
        meta = getattr(fwd_workspace, "_aq_meta", None)
        want = ("mxfp4" if mx else "nvfp4", True, heads, n_q, n_k, D)
        if meta is not None and meta != want:
            raise InvalidValue(f"fwd_workspace was staged as {meta}, this backward needs {want} "
                               "(run the forward with keep_for_bwd=True and the same format)")
        if fwd_workspace.numel() < lib.aq_attn_fwd_workspace_bytes(heads, n_q, n_k, D, 0, 1):
            raise ShapeError("fwd_workspace too small (needs a keep_for_bwd=True forward workspace)")
    ws_bytes = lib.aq_attn_bwd_workspace_bytes(heads, n_q, n_k, D)
    if workspace is not None:
        if workspace.numel() < ws_bytes:
            raise ShapeError("backward workspace too small")
        ws = workspace
    else:
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    padded = D != d
    if grads_out is not None:
        dq, dk, dv = (g.reshape(heads, -1, d) for g in grads_out)
        if dq.dtype != grad_dtype or dk.dtype != grad_dtype or dv.dtype != grad_dtype:
            raise InvalidValue("grads_out dtypes must match grad_dtype")
        if dq.shape[1] != n_q or dk.shape[1] != n_k or dv.shape[1] != n_k:
            raise ShapeError("grads_out shapes must match Q / K / V")
    if grads_out is None or padded:
        dq_k = torch.empty((heads, n_q, D), dtype=grad_dtype, device=q.device)
        dk_k = torch.empty((heads, n_k, D), dtype=grad_dtype, device=q.device)
        dv_k = torch.empty((heads, n_k, D), dtype=grad_dtype, device=q.device)
    else:
        dq_k, dk_k, dv_k = dq, dk, dv
    d_o3 = _pad_d(d_o.reshape(heads, n_q, d).contiguous(), D)
    o_c = _pad_d(o.reshape(heads, n_q, d).contiguous(), D) if o is not None else None
    o_hp_c = _pad_d(o_hp.reshape(heads, n_q, d).contiguous(), D) if o_hp is not None else None
    o_dt = (o_hp_c if o_hp_c is not None else o_c).dtype
    if o_c is not None and o_hp_c is not None and o_c.dtype != o_hp_c.dtype:
        o_c = o_c.to(o_dt)
    if o_dt not in _lib.DT_CODE:
        raise InvalidValue(f"O dtype {o_dt} is not float32 / bfloat16 / float16")
    lse_c = lse.reshape(heads, n_q).to(torch.float32).contiguous()
    q3, k3, v3 = (_pad_d(t.contiguous(), D) for t in (q3, k3, v3))
    q_scale, k_scale, v_scale = _resolve_tensor_scales(q, k, v, q_scale, k_scale, v_scale)
    flag = nonfinite if nonfinite is not None else nonfinite_flag(q.device)
    pf_c, pf_s = _check_pf_out(pf_out, heads, n_q, n_k)
    args = _lib.AqBwdArgs(
        q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(),
        in_dtype=_lib.DT_CODE[q.dtype], d_o=d_o3.data_ptr(), do_dtype=_lib.DT_CODE[d_o3.dtype],
        o=o_c.data_ptr() if o_c is not None else None,
        o_hp=o_hp_c.data_ptr() if o_hp_c is not None else None, o_dtype=_lib.DT_CODE[o_dt],
        lse=lse_c.data_ptr(), heads=heads, n_q=n_q, n_k=n_k, d=D, causal=int(causal),
        variant=variant.code, dq=dq_k.data_ptr(), dk=dk_k.data_ptr(), dv=dv_k.data_ptr(),
        g_dtype=_lib.DT_CODE[grad_dtype], workspace=ws.data_ptr(),
        fwd_workspace=fwd_workspace.data_ptr() if fwd_workspace is not None else None,
        softmax_scale=_scale(softmax_scale, "softmax_scale"), q_scale=_scale(q_scale, "q_scale"),
        k_scale=_scale(k_scale, "k_scale"), v_scale=_scale(v_scale, "v_scale"), p_scale=_scale(p_scale, "p_scale"),
        nonfinite=flag.data_ptr(), pf_codes=pf_c.data_ptr() if pf_c is not None else None,
        pf_scales=pf_s.data_ptr() if pf_s is not None else None)
    _lib.check((lib.aq_attn_bwd_mx if mx else lib.aq_attn_bwd)(args, _lib.stream_ptr()))
    if grads_out is None:
        dq, dk, dv = dq_k, dk_k, dv_k
        if padded:
            dq, dk, dv = (g[..., :d].contiguous() for g in (dq, dk, dv))
    elif padded:
        dq.copy_(dq_k[..., :d])
        dk.copy_(dk_k[..., :d])
        dv.copy_(dv_k[..., :d])
    return (dq.reshape(q.shape[:-2] + (n_q, d)), dk.reshape(k.shape[:-2] + (n_k, d)),
            dv.reshape(v.shape[:-2] + (n_k, d)))


def _plain_forward(q, k, v, causal, train, out_dtype):
    q3, n_q, d = _heads_view(q)
    k3, n_k, dk = _heads_view(k)
    v3, n_v, dv = _heads_view(v)
    if dk != d or dv != d or n_v != n_k or k3.shape[0] != q3.shape[0] or v3.shape[0] != q3.shape[0]:
        raise ShapeError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} V{tuple(v.shape)}")
    o, lse = plain_forward(q3.contiguous(), k3.contiguous(), v3.contiguous(), causal)
    if out_dtype is not None:
        o = o.to(out_dtype)
    lead = q.shape[:-2]
    o = o.reshape(*lead, n_q, d)
    return o, lse.reshape(*lead, n_q), (o.clone() if train else None), None


# ----------------------------------------------------------------------------
# host-buffer entry points (the reference's host-in / host-out contract, with
# H2D, kernels and D2H overlapped across head chunks -- host.py)
# ----------------------------------------------------------------------------

def _host_heads(t):
    if t.device.type != "cpu":
        raise InvalidValue("host entry points take CPU tensors (pinned for overlapped copies)")
    return _heads_view(t)


def _host_empty(shape, dtype, like=None):
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def attn_forward_host(q, k, v, causal=False, train=False, out=None, lse_out=None, o_hp_out=None,
                      out_dtype=None, chunk_heads=None, sync=True):
    """Forward from host tensors [..., N, d] into host outputs -> (O, L, O' or None).

    Same math as ``attn_forward`` (train selects flash_forward_training vs
    flash_forward_inference); the head axis is streamed through the GPU in
    chunks so uploads, kernels and downloads overlap."""
    _lib.require_cuda()
    q3, n_q, d = _host_heads(q)
    k3, n_k, _ = _host_heads(k)
    v3, _, _ = _host_heads(v)
    heads = q3.shape[0]
    # the device output slots take the host output's dtype (a bf16 `out`
    # with fp32 inputs must not receive 4-byte elements)
    out_dtype = out.dtype if out is not None else (out_dtype or q.dtype)
    o = out.reshape(heads, n_q, d) if out is not None else _host_empty((heads, n_q, d), out_dtype)
    lse = lse_out.reshape(heads, n_q) if lse_out is not None else _host_empty((heads, n_q), torch.float32)
    outs = [o, lse]
    if train:
        o_hp = o_hp_out.reshape(heads, n_q, d) if o_hp_out is not None else _host_empty((heads, n_q, d), out_dtype)
        outs.append(o_hp)
    per_head = (q3[0].numel() + 2 * k3[0].numel()) * q3.element_size()
    chunk = chunk_heads or default_chunk(heads, per_head, items_per_head=-(-n_q // 128))
    lib = _lib.load()
    D = kernel_head_dim(d)
    ws_bytes = lambda h: (lib.aq_attn_fwd_workspace_bytes(h, n_q, n_k, D, int(train), 0),)  # noqa: E731
    if ws_bytes(1)[0] <= 0:
        raise InvalidValue(f"unsupported attention shape (n_q={n_q}, n_k={n_k}, d={d})")

    def fn(dev, res, scr):
        attn_forward(dev[0], dev[1], dev[2], causal=causal, train=train, out_dtype=out_dtype, out=res[0],
                     lse_out=res[1], o_hp_out=res[2] if train else None, workspace=scr[0])
    run_pipelined(fn, [q3, k3, v3], outs, chunk, scratch=[("fwd_ws", ws_bytes, torch.uint8)], sync=sync)
    lead = q.shape[:-2]
    return (o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q),
            outs[2].reshape(*lead, n_q, d) if train else None)


def attn_qat_host(q, k, v, d_o, causal=False, variant=BwdVariant.CORRECT, out=None, grads_out=None,
                  chunk_heads=None, sync=True):
    """One QAT attention training step from host tensors: forward (O, O', L) and
    backward (dQ, dK, dV) per head chunk, H2D / kernels / D2H overlapped.
    Returns (O, dQ, dK, dV) in host memory."""
    _lib.require_cuda()
    q3, n_q, d = _host_heads(q)
    k3, n_k, _ = _host_heads(k)
    v3, _, _ = _host_heads(v)
    do3, _, _ = _host_heads(d_o)
    heads = q3.shape[0]
    dt = q.dtype
    o = out.reshape(heads, n_q, d) if out is not None else _host_empty((heads, n_q, d), dt)
    if grads_out is not None:
        dq, dk, dv = (g.reshape(heads, -1, d) for g in grads_out)
    else:
        dq = _host_empty((heads, n_q, d), dt)
        dk, dv = (_host_empty((heads, n_k, d), dt) for _ in range(2))
    per_head = (2 * q3[0].numel() + 2 * k3[0].numel()) * q3.element_size()
    chunk = chunk_heads or default_chunk(heads, per_head, items_per_head=-(-n_q // 128))
    lib = _lib.load()
    D = kernel_head_dim(d)
    if lib.aq_attn_fwd_workspace_bytes(1, n_q, n_k, D, 1, 1) <= 0:
        raise InvalidValue(f"unsupported attention shape (n_q={n_q}, n_k={n_k}, d={d})")
    scratch = [("fwd_ws", lambda h: (lib.aq_attn_fwd_workspace_bytes(h, n_q, n_k, D, 1, 1),), torch.uint8),
               ("bwd_ws", lambda h: (lib.aq_attn_bwd_workspace_bytes(h, n_q, n_k, D),), torch.uint8),
               ("o_hp", lambda h: (h, n_q, d), dt), ("lse", lambda h: (h, n_q), torch.float32)]

    def fn(dev, res, scr):
        qd, kd, vd, dod = dev
        n = qd.shape[0]
        o_hp_d, lse_d = scr[2][:n], scr[3][:n]
        attn_forward(qd, kd, vd, causal=causal, train=True, keep_for_bwd=True, out=res[0], o_hp_out=o_hp_d,
                     lse_out=lse_d, workspace=scr[0])
        attn_backward(qd, kd, vd, dod, res[0], o_hp_d, lse_d, causal=causal, variant=variant, grad_dtype=dt,
                      fwd_workspace=scr[0], workspace=scr[1], grads_out=res[1:])
    run_pipelined(fn, [q3, k3, v3, do3], [o, dq, dk, dv], chunk, scratch=scratch, sync=sync)
    lead = q.shape[:-2]
    return (o.reshape(*lead, n_q, d), dq.reshape(*lead, n_q, d), dk.reshape(*lead, n_k, d),
            dv.reshape(*lead, n_k, d))


# ----------------------------------------------------------------------------
# reference-API shims (2-D per-head numpy or torch operands)
# ----------------------------------------------------------------------------

def _check_attention_shapes(Q, K, V):
    """oracle.py:96-103."""
    if Q.ndim < 2 or K.ndim < 2 or V.ndim < 2:
        raise ShapeError("attention operands must be 2-D (one head at a time)")
    n_q, d = Q.shape[-2:]
    n_k, d_k = K.shape[-2:]
    if d_k != d or tuple(V.shape[-2:]) != (n_k, d):
        raise ShapeError(f"inconsistent shapes Q{tuple(Q.shape)} K{tuple(K.shape)} V{tuple(V.shape)}")
    return n_q, n_k, d


def _check_cfg(cfg, n_q, n_k, d, quantized, allow_mx=False):
    cfg.validate(n_q, n_k, quantized)
    if cfg.accum_width not in (32, 64):
        raise ShapeError(f"accum_width must be 32 or 64, got {cfg.accum_width}")
    if cfg.accum_width != 32:
        raise InvalidValue("the B200 path accumulates in fp32 (tensor cores); accum_width=64 is CPU-only")
    from .codec import MXFP4
    if cfg.spec != NVFP4 and not (allow_mx and cfg.spec == MXFP4):
        raise InvalidValue("the B200 attention path implements NVFP4 (and MXFP4 for the inference forward)")
    if quantized and d % cfg.spec.block_size:
        raise ShapeError("d must be a multiple of the block size when quantizing")
    if cfg.causal and n_q > n_k:
        raise ShapeError("causal attention requires N_q <= N_k")


def _check_finite(*xs):
    """The quantizing reference functions reject non-finite operands
    (codec.py:313-314 via fake_quantize / quantize in flash.py:195-198, 265-267)."""
    for x in xs:
        ok = bool(torch.isfinite(x).all()) if isinstance(x, torch.Tensor) else bool(np.all(np.isfinite(np.asarray(x))))
        if not ok:
            raise InvalidValue("quantize requires finite input")


def _is_host(x):
    return not isinstance(x, torch.Tensor)


# ----------------------------------------------------------------------------
# instrument= (flash.py:98-124; appended at flash.py:167-168, 237-238, 386-387)
# ----------------------------------------------------------------------------

def _visited_tiles(n_q, n_k, cfg):
    """(i, j) key tiles the reference visits: fully masked tiles are skipped (flash.py:127-132, 154)."""
    offset = n_k - n_q if cfg.causal else 0
    for i in range(n_q // cfg.b_q):
        for j in range(n_k // cfg.b_k):
            if cfg.causal and j * cfg.b_k > (i * cfg.b_q + cfg.b_q - 1) + offset:
                continue
            yield i, j


def _instrument_row_states(instrument, q, k, cfg):
    """Sweep-1 snapshots RowState(i, j, m, l) after every key tile (flash.py:145-168).
    The fused kernel keeps (m, l) in registers only, so instrumented runs rebuild
    them on the GPU from S = fp4mm(Q, K) / sqrt(d) -- the block-scaled tcgen05
    GEMM (aq_fp4mm), the same products as the kernels' S MMAs -- with the
    recurrence in float64. Debug-only: one small launch per tile."""
    from .codec import quantize
    from .tensors import fp4mm
    n_q, d = q.shape
    n_k = k.shape[0]
    S = fp4mm(quantize(q), quantize(k)) / torch.tensor(float(np.sqrt(d)), dtype=torch.float32)
    if cfg.causal:
        r = torch.arange(n_q, device=S.device)[:, None]
        c = torch.arange(n_k, device=S.device)[None, :]
        S = S.masked_fill(c > r + (n_k - n_q), float("-inf"))
    S64 = S.double()
    last = {}
    for i, j in _visited_tiles(n_q, n_k, cfg):
        rows = slice(i * cfg.b_q, (i + 1) * cfg.b_q)
        m, l = last.get(i, (torch.full((cfg.b_q,), float("-inf"), dtype=torch.float64, device=S.device),
                            torch.zeros(cfg.b_q, dtype=torch.float64, device=S.device)))
        t = S64[rows, j * cfg.b_k:(j + 1) * cfg.b_k]
        m_new = torch.maximum(m, t.max(dim=1).values)
        dead = torch.isneginf(m_new)
        alpha = torch.where(dead, torch.zeros_like(m), torch.exp(m - torch.where(dead, torch.zeros_like(m_new), m_new)))
        p = torch.exp(t - torch.where(dead, torch.zeros_like(m_new), m_new)[:, None])
        p = torch.where(dead[:, None], torch.zeros_like(p), p)
        l = alpha * l + p.sum(dim=1)
        last[i] = (m_new, l)
        instrument.append(RowState(i, j, m_new.cpu().numpy(), l.cpu().numpy()))


def _instrument_p_tiles(instrument, phase, pf, n_q, n_k, cfg):
    """PTileRecord(phase, i, j, P^F) for every visited tile, from the kernels' P^F dump
    (codes / scales in the quantize_padded(P) layout) decoded by aq_dequantize."""
    from .codec import QuantTensor, dequantize
    codes, scales = pf
    n16 = codes.shape[-1] * 2
    vals = dequantize(QuantTensor(n_q, n16, NVFP4, codes.reshape(n_q, n16 // 2), scales.reshape(n_q, n16 // 16)),
                      torch.float32)
    vals = vals[:, :n_k].double().cpu().numpy()
    for i, j in _visited_tiles(n_q, n_k, cfg):
        instrument.append(PTileRecord(phase, i, j,
                                      vals[i * cfg.b_q:(i + 1) * cfg.b_q, j * cfg.b_k:(j + 1) * cfg.b_k].copy()))


def _host_f32(x):
    """NumPy operand -> float32 CPU tensor (float64 rounds to float32, as on upload)."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))


def _np_out(t, as_np, dtype=np.float32):
    return t.float().cpu().numpy().astype(dtype) if as_np else t


def flash_forward_training(Q, K, V, cfg, quantized=True, instrument=None, threads=1):
    """Training forward: O, L and the auxiliary O' (flash.py:176-246); NVFP4, or
    MXFP4 per cfg.spec."""
    from .codec import MXFP4
    n_q, n_k, d = _check_attention_shapes(Q, K, V)
    _check_cfg(cfg, n_q, n_k, d, quantized, allow_mx=True)
    if quantized and (_is_host(Q) or cfg.spec == MXFP4):
        _check_finite(Q, K, V)  # device NVFP4 operands: the quantizers' flag, checked below
    if quantized and cfg.spec == MXFP4:
        q, as_np = to_device(Q)
        k, _ = to_device(K)
        v, _ = to_device(V)
        o, lse, o_hp = attn_forward_mx(q, k, v, causal=cfg.causal, out_dtype=torch.float32 if as_np else None,
                                       train=True)
        return AttnOutputs(O=_np_out(o, as_np), L=_np_out(lse, as_np, np.float64), O_prime=_np_out(o_hp, as_np))
    if not quantized:
        q, as_np = to_device(Q)
        k, _ = to_device(K)
        v, _ = to_device(V)
        o, lse, o_hp, _ = attn_forward(q, k, v, causal=cfg.causal, train=True, quantized=False)
        return AttnOutputs(O=_np_out(o, as_np), L=_np_out(lse, as_np, np.float64), O_prime=_np_out(o_hp, as_np))
    if _is_host(Q) and instrument is None:
        # host in, host out (the reference's contract): streamed through host.py
        o, lse, o_hp = attn_forward_host(*(_host_f32(x) for x in (Q, K, V)), causal=cfg.causal, train=True,
                                         out_dtype=torch.float32)
        return AttnOutputs(O=o.numpy(), L=lse.numpy().astype(np.float64), O_prime=o_hp.numpy())
    q, as_np = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    pf = pf_buffers(1, n_q, n_k, q.device) if instrument is not None else None
    o, lse, o_hp, _ = attn_forward(q, k, v, causal=cfg.causal, train=True, pf_out=pf,
                                   out_dtype=torch.float32 if as_np else None)
    if not as_np:
        check_nonfinite(q.device)
    if instrument is not None:
        _instrument_row_states(instrument, q.reshape(n_q, d), k.reshape(n_k, d), cfg)
        _instrument_p_tiles(instrument, "forward", pf, n_q, n_k, cfg)
    return AttnOutputs(O=_np_out(o, as_np), L=_np_out(lse, as_np, np.float64), O_prime=_np_out(o_hp, as_np))


def attn_forward_mx(q, k, v, causal=False, out_dtype=None, train=False, keep_for_bwd=False):
    """MXFP4 forward on CUDA tensors [..., N, d] -> (O, L), or (O, L, O') with
    train=True (flash.py:176-314 with cfg.spec = MXFP4; aq_attn_fwd_mx)."""
    _lib.require_cuda()
    q3, n_q, d = _heads_view(q)
    k3, n_k, _ = _heads_view(k)
    v3, _, _ = _heads_view(v)
    dt = q.dtype
    if k.dtype != dt or v.dtype != dt or dt not in _lib.DT_CODE:
        raise InvalidValue("q, k, v must share a float32 / bfloat16 / float16 dtype")
    q3, k3, v3 = q3.contiguous(), k3.contiguous(), v3.contiguous()
    heads = q3.shape[0]
    out_dtype = out_dtype or dt
    lib = _lib.load()
    ws_bytes = lib.aq_attn_fwd_workspace_bytes(heads, n_q, n_k, d, int(train), int(keep_for_bwd))
    if ws_bytes <= 0:
        raise InvalidValue(f"unsupported head dim {d} (the B200 kernels take d in {{64, 128}})")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    o = torch.empty((heads, n_q, d), dtype=out_dtype, device=q.device)
    o_hp = torch.empty((heads, n_q, d), dtype=out_dtype, device=q.device) if train else None
    lse = torch.empty((heads, n_q), dtype=torch.float32, device=q.device)
    args = _lib.AqFwdArgs(
        q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[dt],
        heads=heads, n_q=n_q, n_k=n_k, d=d, causal=int(causal), train=int(train),
        o=o.data_ptr(), o_dtype=_lib.DT_CODE[out_dtype], o_hp=o_hp.data_ptr() if train else None,
        o_hp_dtype=_lib.DT_CODE[out_dtype], lse=lse.data_ptr(), workspace=ws.data_ptr(),
        keep_for_bwd=int(keep_for_bwd), operands_staged=0)
    _lib.check(lib.aq_attn_fwd_mx(args, _lib.stream_ptr()))
    ws._aq_meta = ("mxfp4", bool(keep_for_bwd), heads, n_q, n_k, d)
    lead = q.shape[:-2]
    outs = (o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q))
    if train:
        outs = outs + (o_hp.reshape(*lead, n_q, d),)
    return outs + (ws,) if keep_for_bwd else outs


def flash_forward_inference(Q, K, V, cfg, instrument=None, threads=1):
    """Inference forward on real FP4 codes: O, L (flash.py:249-314); NVFP4 or
    MXFP4 per cfg.spec."""
    from .codec import MXFP4
    n_q, n_k, d = _check_attention_shapes(Q, K, V)
    _check_cfg(cfg, n_q, n_k, d, True, allow_mx=True)
    if _is_host(Q) or cfg.spec == MXFP4:
        _check_finite(Q, K, V)
    if cfg.spec == MXFP4:
        q, as_np = to_device(Q)
        k, _ = to_device(K)
        v, _ = to_device(V)
        o, lse = attn_forward_mx(q, k, v, causal=cfg.causal, out_dtype=torch.float32 if as_np else None)
        return AttnOutputs(O=_np_out(o, as_np), L=_np_out(lse, as_np, np.float64), O_prime=None)
    if _is_host(Q):
        o, lse, _ = attn_forward_host(*(_host_f32(x) for x in (Q, K, V)), causal=cfg.causal, train=False,
                                      out_dtype=torch.float32)
        if instrument is not None:  # sweep-1 snapshots only, as the reference (flash.py:287-288)
            _instrument_row_states(instrument, to_device(Q)[0], to_device(K)[0], cfg)
        return AttnOutputs(O=o.numpy(), L=lse.numpy().astype(np.float64), O_prime=None)
    q, _ = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    o, lse, _, _ = attn_forward(q, k, v, causal=cfg.causal, train=False)
    check_nonfinite(q.device)
    if instrument is not None:
        _instrument_row_states(instrument, q.reshape(n_q, d), k.reshape(n_k, d), cfg)
    return AttnOutputs(O=o, L=lse, O_prime=None)


def flash_backward(Q, K, V, dO, outs, cfg, variant=BwdVariant.CORRECT, quantized=True, instrument=None):
    """Recompute-and-requantize QAT backward (flash.py:317-390)."""
    from .codec import MXFP4
    n_q, n_k, d = _check_attention_shapes(Q, K, V)
    _check_cfg(cfg, n_q, n_k, d, quantized, allow_mx=True)
    if tuple(dO.shape) != tuple(Q.shape):
        raise ShapeError(f"dO shape {tuple(dO.shape)} does not match Q {tuple(Q.shape)}")
    if tuple(outs.L.shape) != tuple(Q.shape[:-1]):
        raise ShapeError("outs.L has the wrong shape")
    if variant.uses_o_prime and outs.O_prime is None:
        raise MissingOPrime(f"variant {variant.value} needs O_prime; run the training forward")
    if quantized and (_is_host(Q) or cfg.spec == MXFP4):
        _check_finite(Q, K, V)
    q, as_np = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    d_o, _ = to_device(dO)
    o = to_device(outs.O)[0] if outs.O is not None else None
    o_hp = to_device(outs.O_prime)[0] if outs.O_prime is not None else None
    lse = to_device(outs.L)[0]
    g_dt = torch.float32 if as_np else None
    mx = quantized and cfg.spec == MXFP4
    want_pf = instrument is not None and quantized and not mx and variant.fake_quantizes_p
    pf = pf_buffers(1, n_q, n_k, q.device) if want_pf else None
    dq, dk, dv = attn_backward(q, k, v, d_o.to(q.dtype) if d_o.dtype != q.dtype and not as_np else d_o,
                               o, o_hp, lse, causal=cfg.causal, variant=variant, grad_dtype=g_dt,
                               quantized=quantized, mx=mx, pf_out=pf)
    if quantized and not as_np and not mx:
        check_nonfinite(q.device)
    if want_pf:  # flash.py:386-387: records in the backward's loop order (key tile outer)
        recs = []
        _instrument_p_tiles(recs, "backward", pf, n_q, n_k, cfg)
        instrument.extend(sorted(recs, key=lambda r: (r.j_tile, r.i_tile)))
    return AttnGrads(dQ=_np_out(dq, as_np), dK=_np_out(dk, as_np), dV=_np_out(dv, as_np))
