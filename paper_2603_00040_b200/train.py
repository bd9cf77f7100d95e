"""Data-parallel QAT training driver on B200 (the caller of the hot path).

Mirrors the reference toy harness (attnqat/harness.py:49-344) at GPU scale:
projections W_q / W_k / W_v / W_o stay high precision (bf16 weights, fp32
master copy in AdamW), quantization happens only inside the attention operator
(``attn_qat``: NVFP4 two-pass forward + QAT backward, harness.py:195-248). The
loss is the associative-recall MSE on the last token (harness.py:214-217).

Multi-GPU: one process per GPU (torchrun), the global batch is sharded over
ranks, each rank runs forward/backward on its shard and the parameter
gradients are all-reduced with NCCL. The all-reduce of W_o starts as soon as
its gradient is final (post-accumulate hook), so it overlaps the attention
backward; W_q/W_k/W_v follow once the projection backward finishes. The
attention path itself has no communication.

Divergence handling follows harness.py:291-321: a non-finite or > 1e6 loss,
or non-finite parameters, raise StabilityError with the step index.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from .autograd import attn_qat
from .errors import InvalidValue, StabilityError
from .flash import BwdVariant

# attention modes of the reference harness (harness.py:39-45): (quantized, variant)
ATTN_MODES = {
    "bf16": (False, BwdVariant.CORRECT),
    "fp4-qat": (True, BwdVariant.CORRECT),
    "fp4-qat/lowpreco": (True, BwdVariant.LOW_PREC_O),
    "fp4-qat/nofqp": (True, BwdVariant.NO_FAKE_QUANT_P),
    "fp4-qat/naive-bf16-bwd": (True, BwdVariant.NAIVE_BF16_BWD),
    # the MXFP4 format (UE8M0 scales per 32 elements) with the correct backward
    "mxfp4-qat": (True, BwdVariant.CORRECT),
}
TASK_COMMON_GAIN = 12.0  # harness.py:37
DIVERGENCE_LOSS = 1e6


@dataclass
class TrainConfig:
    """harness.py:93-127, widened to multi-head B200 shapes."""

    steps: int = 100
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    weight_decay: float = 0.0
    seed: int = 0
    seq_len: int = 256
    batch: int = 8           # global batch (sharded over ranks)
    d_model: int = 256
    n_heads: int = 2
    head_dim: int = 64
    causal: bool = False
    attn_mode: str = "fp4-qat"
    compute_dtype: str = "bf16"   # projection / attention operand dtype ("bf16" | "fp32")

    def validate(self, world=1):
        problems = []
        if self.steps < 1:
            problems.append("steps must be >= 1")
        if not self.lr > 0:
            problems.append("lr must be > 0")
        if not 0 <= self.beta1 < 1 or not 0 <= self.beta2 < 1:
            problems.append("betas must lie in [0, 1)")
        if self.seq_len < 4:
            problems.append("seq_len must be >= 4")
        if self.batch < 1 or self.batch % world:
            problems.append(f"batch must be >= 1 and divisible by the world size {world}")
        if self.attn_mode not in ATTN_MODES:
            problems.append(f"attn_mode must be one of {sorted(ATTN_MODES)}")
        if self.head_dim % 16 or not 0 < self.head_dim <= 128:
            problems.append("head_dim must be a multiple of 16 up to 128 (B200 kernels; < 128 is zero-padded)")
        if self.d_model % 2:
            problems.append("d_model must be even")
        if self.compute_dtype not in ("bf16", "fp32"):
            problems.append("compute_dtype must be bf16 or fp32")
        return problems


@dataclass
class TrainLog:
    losses: list = field(default_factory=list)
    grad_norms: list = field(default_factory=list)
    wall_ms: list = field(default_factory=list)

    def append(self, loss, gnorm, ms):
        self.losses.append(float(loss))
        self.grad_norms.append(float(gnorm))
        self.wall_ms.append(float(ms))


def make_task(seed, seq_len, d_model, batch):
    """Associative recall batch (harness.py:161-182): the last token repeats one
    memory token; the target is that token. Returns float32 numpy arrays."""
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    n_mem = seq_len - 1
    d_key = d_model // 2
    u = np.ones(d_key) / np.sqrt(d_key)
    keys = TASK_COMMON_GAIN * u + rng.standard_normal((batch, n_mem, d_key))
    payload = rng.standard_normal((batch, n_mem, d_model - d_key))
    X = np.zeros((batch, seq_len, d_model))
    X[:, :n_mem, :d_key] = keys
    X[:, :n_mem, d_key:] = payload
    match = rng.integers(0, n_mem, size=batch)
    rows = X[np.arange(batch), match]
    X[:, -1] = rows
    return X.astype(np.float32), rows.astype(np.float32)


class AttnLayer(torch.nn.Module):
    """Multi-head attention with learned projections (harness.py:49-76)."""

    def __init__(self, d_model, n_heads, head_dim, seed=0, device="cuda", attn_fn=None):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        inner = n_heads * head_dim
        s = 1.0 / math.sqrt(d_model)
        self.w_q = torch.nn.Parameter((torch.randn(d_model, inner, generator=g) * s).to(device))
        self.w_k = torch.nn.Parameter((torch.randn(d_model, inner, generator=g) * s).to(device))
        self.w_v = torch.nn.Parameter((torch.randn(d_model, inner, generator=g) * s).to(device))
        self.w_o = torch.nn.Parameter((torch.randn(d_model, inner, generator=g) * s).to(device))
        self.n_heads, self.head_dim = n_heads, head_dim
        self.attn_fn = attn_fn or attn_qat   # tests inject a CPU reference attention

    def forward(self, x, causal=False, variant=BwdVariant.CORRECT, dtype=torch.bfloat16, quantized=True):
        B, N, _ = x.shape
        H, d = self.n_heads, self.head_dim
        xc = x.to(dtype)

        def proj(w):
            return (xc @ w.to(dtype)).view(B, N, H, d).transpose(1, 2)
        qkv = (proj(self.w_q), proj(self.w_k), proj(self.w_v))
        if quantized:
            o = self.attn_fn(*qkv, causal, variant)
        else:   # the harness's "bf16" mode: plain attention (flash.py quantized=False)
            o = self.attn_fn(*qkv, causal, variant, False)
        o = o.transpose(1, 2).reshape(B, N, H * d)
        return o @ self.w_o.to(dtype).t()


def random_prediction_baseline(targets):
    """Mean loss of predicting zero: the target second moment (harness.py:185-187)."""
    t = targets.float() if isinstance(targets, torch.Tensor) else torch.from_numpy(np.asarray(targets)).float()
    return float((t ** 2).mean())


@torch.no_grad()
def evaluate(layer, X, targets, eval_mode="bf16", causal=False, dtype=torch.bfloat16):
    """Deterministic last-token MSE under the chosen attention precision
    (harness.py:326-344): "bf16" the unquantized forward, "fp4" the real-quant
    inference kernel (K5), "fp4-fake" the training forward (K4) -- the two FP4
    paths give the same O bit for bit, so "fp4" and "fp4-fake" agree exactly."""
    from .flash import attn_forward
    dev = layer.w_q.device
    x = (X if isinstance(X, torch.Tensor) else torch.from_numpy(np.asarray(X))).to(dev)
    t = (targets if isinstance(targets, torch.Tensor) else torch.from_numpy(np.asarray(targets))).to(dev)
    if eval_mode == "bf16":
        y = layer(x, causal, dtype=dtype, quantized=False)
    elif eval_mode in ("fp4", "fp4-fake"):
        train = eval_mode == "fp4-fake"

        def fwd(q, k, v, causal_, variant, quantized=True):
            return attn_forward(q, k, v, causal=causal_, train=train)[0]
        saved = layer.attn_fn
        layer.attn_fn = fwd
        try:
            y = layer(x, causal, dtype=dtype)
        finally:
            layer.attn_fn = saved
    else:
        raise InvalidValue(f"unknown eval_mode {eval_mode!r}")
    return float(((y[:, -1].float() - t.float()) ** 2).mean())


def qat_matmul(A, B, spec=None, accum_width=64):
    """C = fq(A) fq(B) (harness.py:356-358): both operands fake-quantized along
    their last axis on the GPU quantizers, the product in the accumulation width."""
    from .codec import NVFP4, fake_quantize
    spec = spec or NVFP4
    dt = torch.float64 if accum_width == 64 else torch.float32
    a = torch.as_tensor(fake_quantize(A, spec))
    b = torch.as_tensor(fake_quantize(B, spec))
    out = a.to("cuda", dt) @ b.to("cuda", dt)
    return out.cpu().numpy() if not isinstance(A, torch.Tensor) else out


def qat_matmul_backward(A, B, dC, spec=None, accum_width=64):
    """Straight-through gradients (harness.py:361-369): dA = dC fq(B)^T,
    dB = fq(A)^T dC -- exactly, an identity of the estimator."""
    from .codec import NVFP4, fake_quantize
    spec = spec or NVFP4
    dt = torch.float64 if accum_width == 64 else torch.float32
    a = torch.as_tensor(fake_quantize(A, spec)).to("cuda", dt)
    b = torch.as_tensor(fake_quantize(B, spec)).to("cuda", dt)
    dc = torch.as_tensor(dC if isinstance(dC, torch.Tensor) else np.asarray(dC)).to("cuda", dt)
    dA, dB = dc @ b.t(), a.t() @ dc
    if not isinstance(A, torch.Tensor):
        return dA.cpu().numpy(), dB.cpu().numpy()
    return dA, dB


class GradAllReduce:
    """NCCL all-reduce of parameter gradients, each launched asynchronously the
    moment its gradient is final, averaged over ranks."""

    def __init__(self, params, world):
        self.world = world
        self.handles = []
        if world > 1:
            for p in params:
                p.register_post_accumulate_grad_hook(self._hook)

    def _hook(self, p):
        p.grad.div_(self.world)
        self.handles.append(dist.all_reduce(p.grad, op=dist.ReduceOp.SUM, async_op=True))

    def wait(self):
        for h in self.handles:
            h.wait()
        self.handles.clear()


def shard(batch_arrays, rank, world):
    """Contiguous batch shard of this rank (SURVEY §8e partitioning)."""
    out = []
    for a in batch_arrays:
        per = a.shape[0] // world
        out.append(a[rank * per:(rank + 1) * per])
    return out


def train(cfg: TrainConfig, device=None, attn_fn=None, log_every=0):
    """Run the data-parallel QAT loop; returns (layer, TrainLog)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    problems = cfg.validate(world)
    if problems:
        raise InvalidValue("; ".join(problems))
    device = device or ("cuda" if torch.cuda.is_available() else "cpu")
    if attn_fn is None and cfg.attn_mode == "mxfp4-qat":
        from .codec import MXFP4

        def attn_fn(q, k, v, causal, variant, quantized=True):
            return attn_qat(q, k, v, causal, variant, quantized, spec=MXFP4)
    layer = AttnLayer(cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.seed, device, attn_fn)
    opt = torch.optim.AdamW(layer.parameters(), lr=cfg.lr, betas=(cfg.beta1, cfg.beta2),
                            weight_decay=cfg.weight_decay)
    ar = GradAllReduce(layer.parameters(), world)
    quantized, variant = ATTN_MODES[cfg.attn_mode]
    log = TrainLog()
    for step in range(cfg.steps):
        t0 = time.perf_counter()
        X, T = make_task(cfg.seed * 1_000_003 + step, cfg.seq_len, cfg.d_model, cfg.batch)
        X, T = shard((X, T), rank, world)
        x = torch.from_numpy(X).to(device)
        t = torch.from_numpy(T).to(device)
        opt.zero_grad(set_to_none=True)
        y = layer(x, cfg.causal, variant,
                  dtype=torch.bfloat16 if cfg.compute_dtype == "bf16" else torch.float32, quantized=quantized)
        loss = torch.mean((y[:, -1].float() - t) ** 2)
        loss.backward()
        ar.wait()
        lv = loss.detach()
        if world > 1:
            dist.all_reduce(lv, op=dist.ReduceOp.SUM)
            lv = lv / world
        lval = float(lv)
        if not math.isfinite(lval) or lval > DIVERGENCE_LOSS:
            raise StabilityError(f"loss diverged to {lval}", step=step)
        gnorm = math.sqrt(sum(float((p.grad.float() ** 2).sum()) for p in layer.parameters()))
        opt.step()
        for name, p in layer.named_parameters():
            if not torch.isfinite(p).all():
                raise StabilityError(f"parameter {name} became non-finite", step=step)
        log.append(lval, gnorm, (time.perf_counter() - t0) * 1e3)
        if log_every and rank == 0 and step % log_every == 0:
            print(f"step {step} loss {lval:.4f} gnorm {gnorm:.3f}", flush=True)
    return layer, log
