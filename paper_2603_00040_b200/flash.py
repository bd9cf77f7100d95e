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
    InvalidValue); ``instrument`` and ``threads`` are accepted and ignored.
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


def attn_forward(q, k, v, causal=False, train=True, out_dtype=None, keep_for_bwd=False, lse_out=None,
                 workspace=None, operands_staged=False, out=None, o_hp_out=None, quantized=True):
    """Fused forward on CUDA tensors [..., N, d] -> (O, L, O_hp or None, workspace).

    ``train=True`` is flash_forward_training (O, L, O'), ``False`` is
    flash_forward_inference (O, L). O is the FP4-path output, O' the
    high-precision output the QAT backward needs (flash.py:176-246).
    ``quantized=False`` is plain attention (O' = O; plain.py)."""
    _lib.require_cuda()
    if q.device.type == "cuda" and q.device.index is not None and q.device.index != torch.cuda.current_device():
        with torch.cuda.device(q.device):  # launch on (and with the current stream of) q's device
            return attn_forward(q, k, v, causal, train, out_dtype, keep_for_bwd, lse_out, workspace,
                                operands_staged, out, o_hp_out, quantized)
    if not quantized:
        return _plain_forward(q, k, v, causal, train, out_dtype)
    q3, n_q, d = _heads_view(q)
    k3, n_k, dk = _heads_view(k)
    v3, n_v, dv = _heads_view(v)
    if dk != d or dv != d or n_v != n_k or k3.shape[0] != q3.shape[0] or v3.shape[0] != q3.shape[0]:
        raise ShapeError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} V{tuple(v.shape)}")
    if d % 16:
        raise ShapeError("d must be a multiple of the block size when quantizing")
    if causal and n_q > n_k:
        raise ShapeError("causal attention requires N_q <= N_k")
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
    if workspace is not None:
        if workspace.numel() < ws_bytes:
            raise ShapeError("workspace too small")
        ws = workspace
    else:
        if operands_staged:
            raise InvalidValue("operands_staged needs the workspace that holds them")
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    o = out if out is not None else torch.empty((heads, n_q, d), dtype=out_dtype, device=q.device)
    o_hp = None
    if train:
        o_hp = o_hp_out if o_hp_out is not None else torch.empty((heads, n_q, d), dtype=out_dtype, device=q.device)
    lse = lse_out if lse_out is not None else torch.empty((heads, n_q), dtype=torch.float32, device=q.device)
    args = _lib.AqFwdArgs(
        q=q3.data_ptr(), k=k3.data_ptr(), v=v3.data_ptr(), in_dtype=_lib.DT_CODE[dt],
        heads=heads, n_q=n_q, n_k=n_k, d=d, causal=int(causal), train=int(train),
        o=o.data_ptr(), o_dtype=_lib.DT_CODE[out_dtype],
        o_hp=o_hp.data_ptr() if o_hp is not None else None, o_hp_dtype=_lib.DT_CODE[out_dtype],
        lse=lse.data_ptr(), workspace=ws.data_ptr(), keep_for_bwd=int(keep_for_bwd),
        operands_staged=int(operands_staged))
    _lib.check(lib.aq_attn_fwd(args, _lib.stream_ptr()))
    lead = q.shape[:-2]
    return (o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q),
            o_hp.reshape(*lead, n_q, d) if o_hp is not None else None, ws)


def attn_backward(q, k, v, d_o, o, o_hp, lse, causal=False, variant=BwdVariant.CORRECT, grad_dtype=None,
                  fwd_workspace=None, workspace=None, grads_out=None, quantized=True, mx=False):
    """Fused QAT backward on CUDA tensors -> (dQ, dK, dV) (flash.py:317-390)."""
    _lib.require_cuda()
    if q.device.type == "cuda" and q.device.index is not None and q.device.index != torch.cuda.current_device():
        with torch.cuda.device(q.device):
            return attn_backward(q, k, v, d_o, o, o_hp, lse, causal, variant, grad_dtype, fwd_workspace,
                                 workspace, grads_out, quantized, mx)
    q3, n_q, d = _heads_view(q)
    k3, n_k, _ = _heads_view(k)
    v3, _, _ = _heads_view(v)
    heads = q3.shape[0]
    if tuple(d_o.shape) != tuple(q.shape):
        raise ShapeError(f"dO shape {tuple(d_o.shape)} does not match Q {tuple(q.shape)}")
    if variant.uses_o_prime and o_hp is None:
        raise MissingOPrime(f"variant {variant.value} needs O_prime; run the training forward")
    o_ref = o_hp if variant.uses_o_prime else o
    if o_ref is None:
        raise ShapeError("the forward output O is required")
    if lse.numel() != heads * n_q:
        raise ShapeError("outs.L has the wrong shape")
    grad_dtype = grad_dtype or q.dtype
    if not quantized:
        # every variant reduces to the plain backward (flash.py:344-349, 357)
        g = plain_backward(q3.contiguous(), k3.contiguous(), v3.contiguous(), d_o.reshape(heads, n_q, d),
                           o_ref.reshape(heads, n_q, d), lse.reshape(heads, n_q), causal, grad_dtype)
        return (g[0].reshape(q.shape[:-2] + (n_q, d)), g[1].reshape(k.shape[:-2] + (n_k, d)),
                g[2].reshape(v.shape[:-2] + (n_k, d)))
    lib = _lib.load()
    ws_bytes = lib.aq_attn_bwd_workspace_bytes(heads, n_q, n_k, d)
    if workspace is not None:
        if workspace.numel() < ws_bytes:
            raise ShapeError("backward workspace too small")
        ws = workspace
    else:
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    if grads_out is not None:
        dq, dk, dv = (g.reshape(heads, -1, d) for g in grads_out)
        if dq.dtype != grad_dtype or dk.dtype != grad_dtype or dv.dtype != grad_dtype:
            raise InvalidValue("grads_out dtypes must match grad_dtype")
    else:
        dq = torch.empty((heads, n_q, d), dtype=grad_dtype, device=q.device)
        dk = torch.empty((heads, n_k, d), dtype=grad_dtype, device=q.device)
        dv = torch.empty((heads, n_k, d), dtype=grad_dtype, device=q.device)
    d_o3 = d_o.reshape(heads, n_q, d).contiguous()
    o_c = o.reshape(heads, n_q, d).contiguous() if o is not None else None
    o_hp_c = o_hp.reshape(heads, n_q, d).contiguous() if o_hp is not None else None
    o_dt = (o_hp_c if o_hp_c is not None else o_c).dtype
    if o_c is not None and o_hp_c is not None and o_c.dtype != o_hp_c.dtype:
        o_c = o_c.to(o_dt)
    lse_c = lse.reshape(heads, n_q).to(torch.float32).contiguous()
    args = _lib.AqBwdArgs(
        q=q3.contiguous().data_ptr(), k=k3.contiguous().data_ptr(), v=v3.contiguous().data_ptr(),
        in_dtype=_lib.DT_CODE[q.dtype], d_o=d_o3.data_ptr(), do_dtype=_lib.DT_CODE[d_o3.dtype],
        o=o_c.data_ptr() if o_c is not None else None,
        o_hp=o_hp_c.data_ptr() if o_hp_c is not None else None, o_dtype=_lib.DT_CODE[o_dt],
        lse=lse_c.data_ptr(), heads=heads, n_q=n_q, n_k=n_k, d=d, causal=int(causal),
        variant=variant.code, dq=dq.data_ptr(), dk=dk.data_ptr(), dv=dv.data_ptr(),
        g_dtype=_lib.DT_CODE[grad_dtype], workspace=ws.data_ptr(),
        fwd_workspace=fwd_workspace.data_ptr() if fwd_workspace is not None else None)
    _lib.check((lib.aq_attn_bwd_mx if mx else lib.aq_attn_bwd)(args, _lib.stream_ptr()))
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
    out_dtype = out_dtype or q.dtype
    o = out.reshape(heads, n_q, d) if out is not None else _host_empty((heads, n_q, d), out_dtype)
    lse = lse_out.reshape(heads, n_q) if lse_out is not None else _host_empty((heads, n_q), torch.float32)
    outs = [o, lse]
    if train:
        o_hp = o_hp_out.reshape(heads, n_q, d) if o_hp_out is not None else _host_empty((heads, n_q, d), out_dtype)
        outs.append(o_hp)
    per_head = (q3[0].numel() + 2 * k3[0].numel()) * q3.element_size()
    chunk = chunk_heads or default_chunk(heads, per_head, items_per_head=-(-n_q // 128))
    lib = _lib.load()
    ws_bytes = lambda h: (lib.aq_attn_fwd_workspace_bytes(h, n_q, n_k, d, int(train), 0),)  # noqa: E731
    if ws_bytes(1)[0] <= 0:
        raise InvalidValue(f"unsupported head dim {d} (the B200 kernels take d in {{64, 128}})")

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
    if lib.aq_attn_fwd_workspace_bytes(1, n_q, n_k, d, 1, 1) <= 0:
        raise InvalidValue(f"unsupported head dim {d} (the B200 kernels take d in {{64, 128}})")
    scratch = [("fwd_ws", lambda h: (lib.aq_attn_fwd_workspace_bytes(h, n_q, n_k, d, 1, 1),), torch.uint8),
               ("bwd_ws", lambda h: (lib.aq_attn_bwd_workspace_bytes(h, n_q, n_k, d),), torch.uint8),
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
    if quantized:
        _check_finite(Q, K, V)
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
    if _is_host(Q):
        # host in, host out (the reference's contract): streamed through host.py
        o, lse, o_hp = attn_forward_host(*(_host_f32(x) for x in (Q, K, V)), causal=cfg.causal, train=True,
                                         out_dtype=torch.float32)
        return AttnOutputs(O=o.numpy(), L=lse.numpy().astype(np.float64), O_prime=o_hp.numpy())
    q, _ = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    o, lse, o_hp, _ = attn_forward(q, k, v, causal=cfg.causal, train=True)
    return AttnOutputs(O=o, L=lse, O_prime=o_hp)


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
        return AttnOutputs(O=o.numpy(), L=lse.numpy().astype(np.float64), O_prime=None)
    q, _ = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    o, lse, _, _ = attn_forward(q, k, v, causal=cfg.causal, train=False)
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
    if quantized:
        _check_finite(Q, K, V)
    q, as_np = to_device(Q)
    k, _ = to_device(K)
    v, _ = to_device(V)
    d_o, _ = to_device(dO)
    o = to_device(outs.O)[0] if outs.O is not None else None
    o_hp = to_device(outs.O_prime)[0] if outs.O_prime is not None else None
    lse = to_device(outs.L)[0]
    g_dt = torch.float32 if as_np else None
    dq, dk, dv = attn_backward(q, k, v, d_o.to(q.dtype) if d_o.dtype != q.dtype and not as_np else d_o,
                               o, o_hp, lse, causal=cfg.causal, variant=variant, grad_dtype=g_dt,
                               quantized=quantized, mx=quantized and cfg.spec == MXFP4)
    return AttnGrads(dQ=_np_out(dq, as_np), dK=_np_out(dk, as_np), dV=_np_out(dv, as_np))
