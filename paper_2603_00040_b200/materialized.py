"""The reference's materialized O(N^2) attention oracle on the GPU
(attnqat/oracle.py:27-161): ``QuantPoints``, ``OracleTrace``,
``oracle_forward``, ``oracle_backward``.

This is the reference's debugging / test oracle, not the fused hot path: it
materializes S, P and P^F for one head, so it is meant for small N. The fake
quantization at the chosen points runs on the NVFP4 / MXFP4 quantizer kernels
(csrc/quantize.cu); the matmuls run in the requested accumulation width (fp32
or fp64) on the GPU's BLAS, not in the reference's fixed left-to-right order
(tensors.py:32-51), so results agree with the reference to rounding, not bit
for bit. P is the fp64 row softmax (oracle.py:78-93); P^F is quantized from
P rounded to fp32 (the quantizer kernels read fp32).

NumPy inputs give NumPy outputs; CUDA tensors stay on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .codec import NVFP4, fake_quantize, fake_quantize_cols, fake_quantize_padded
from .errors import ShapeError
from .flash import AttnGrads


@dataclass(frozen=True)
class QuantPoints:
    """Which attention operands get fake-quantized (oracle.py:27-46)."""

    q: bool = True
    k: bool = True
    v: bool = True
    p: bool = True

    @classmethod
    def all_on(cls):
        return cls(True, True, True, True)

    @classmethod
    def all_off(cls):
        return cls(False, False, False, False)

    @property
    def any(self):
        return self.q or self.k or self.v or self.p


@dataclass
class OracleTrace:
    """Everything the materialized forward produces (oracle.py:49-58)."""

    S: object
    P: object
    P_fq: object
    L: object
    O: object
    O_prime: object
    causal: bool


def _dt(accum_width):
    if accum_width not in (32, 64):
        raise ShapeError(f"accum_width must be 32 or 64, got {accum_width}")
    return torch.float32 if accum_width == 32 else torch.float64


def _dev(x):
    """(cuda tensor, came_from_numpy), keeping float64 (the unquantized points
    run in the accumulation width, like the reference)."""
    from . import _lib
    _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t, was_np = x, False
    else:
        t, was_np = torch.from_numpy(np.ascontiguousarray(np.asarray(x))), True
    if not t.is_floating_point():
        t = t.to(torch.float32)
    return t.to("cuda"), was_np


def _np(t, as_np):
    return t.cpu().numpy() if as_np else t


def oracle_forward(Q, K, V, spec=NVFP4, points=QuantPoints(), causal=False, accum_width=32):
    """Reference attention forward with fake quantization at the chosen points
    (oracle.py:106-131)."""
    q, as_np = _dev(Q)
    k, _ = _dev(K)
    v, _ = _dev(V)
    if q.dim() != 2 or k.dim() != 2 or v.dim() != 2:
        raise ShapeError("attention operands must be 2-D (one head at a time)")
    n_q, d = q.shape
    n_k, d_k = k.shape
    if d_k != d or tuple(v.shape) != (n_k, d):
        raise ShapeError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} V{tuple(v.shape)}")
    if points.any and d % spec.block_size:
        raise ShapeError("d must be a multiple of the block size when quantizing")
    if causal and n_q > n_k:
        raise ShapeError("causal attention requires N_q <= N_k")
    dt = _dt(accum_width)
    qf = fake_quantize(q.float(), spec) if points.q else q
    kf = fake_quantize(k.float(), spec) if points.k else k
    vf = fake_quantize_cols(v.float(), spec) if points.v else v
    S = (qf.to(dt) @ kf.to(dt).t()) / torch.sqrt(torch.tensor(float(d), dtype=dt, device=q.device))
    if causal:
        rows = torch.arange(n_q, device=q.device)[:, None]
        cols = torch.arange(n_k, device=q.device)[None, :]
        S = S.masked_fill(cols > rows + (n_k - n_q), float("-inf"))
    S64 = S.double()
    m = S64.max(dim=1).values
    if torch.isneginf(m).any():
        raise ShapeError("fully masked rows are rejected")
    L = m + torch.log(torch.exp(S64 - m[:, None]).sum(dim=1))
    P = torch.exp(S64 - L[:, None])
    P_fq = fake_quantize_padded(P.float(), spec).double() if points.p else P
    O = P_fq.to(dt) @ vf.to(dt)
    O_prime = P.to(dt) @ vf.to(dt)
    return OracleTrace(S=_np(S, as_np), P=_np(P, as_np), P_fq=_np(P_fq, as_np), L=_np(L, as_np),
                       O=_np(O, as_np), O_prime=_np(O_prime, as_np), causal=causal)


def oracle_backward(trace, Qf, Kf, Vf, dO, accum_width=32):
    """Gradients through the explicit softmax Jacobian (oracle.py:141-161):
    dS = P * (dP - delta) / sqrt(d), delta_i = P_i . dP_i."""
    qf, as_np = _dev(Qf)
    kf, _ = _dev(Kf)
    vf, _ = _dev(Vf)
    do, _ = _dev(dO)
    n_q, d = qf.shape
    if tuple(do.shape) != (n_q, d):
        raise ShapeError(f"dO shape {tuple(do.shape)} does not match Q {tuple(qf.shape)}")
    P = _dev(trace.P)[0].double()
    P_fq = _dev(trace.P_fq)[0].double()
    if tuple(P.shape) != (n_q, kf.shape[0]):
        raise ShapeError("trace does not match the provided operands")
    dt = _dt(accum_width)
    dV = P_fq.to(dt).t() @ do.to(dt)
    dP = do.to(dt) @ vf.to(dt).t()
    delta = (P * dP.double()).sum(dim=1)
    dS = (dP - delta.to(dt)[:, None]) * P.to(dt) / torch.sqrt(torch.tensor(float(d), dtype=dt, device=qf.device))
    dQ = dS @ kf.to(dt)
    dK = dS.t() @ qf.to(dt)
    return AttnGrads(dQ=_np(dQ, as_np), dK=_np(dK, as_np), dV=_np(dV, as_np))


def fd_attention_grads(Q, K, V, dO, causal=False, step=1e-3):
    """Central finite differences of <dO, O> on the unquantized path
    (oracle.py:164-194): an independent fp64 gradient check, O(params)
    materialized forwards -- tiny shapes only."""
    q, as_np = _dev(Q)
    k, _ = _dev(K)
    v, _ = _dev(V)
    do = _dev(dO)[0].double()
    base = [t.double() for t in (q, k, v)]
    off = QuantPoints.all_off()

    def loss(args):
        tr = oracle_forward(*args, points=off, causal=causal, accum_width=64)
        return float((do * tr.O).sum())

    grads = []
    for which in range(3):
        g = torch.zeros_like(base[which])
        flat = base[which].view(-1)
        for i in range(flat.numel()):
            keep = float(flat[i])
            flat[i] = keep + step
            up = loss(base)
            flat[i] = keep - step
            down = loss(base)
            flat[i] = keep
            g.view(-1)[i] = (up - down) / (2 * step)
        grads.append(g)
    return AttnGrads(dQ=_np(grads[0], as_np), dK=_np(grads[1], as_np), dV=_np(grads[2], as_np))
