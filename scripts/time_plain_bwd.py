"""Time the quantized=False backward (aq_attn_bwd_plain) at the C4 shape next to
FlashAttention-2's backward on the same operands (comparator only). GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

B, H, N, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 32, 4096, 128)))
causal = True
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(B, H, N, d, generator=g, device="cuda").bfloat16() for _ in range(4))
o, lse, ohp, _ = aq.attn_forward(q, k, v, causal=causal, train=True, quantized=False)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


ours = timed(lambda: aq.attn_backward(q, k, v, do, o, ohp, lse, causal=causal, quantized=False))
fwd = timed(lambda: aq.attn_forward(q, k, v, causal=causal, train=True, quantized=False))
flops = 4.0 * B * H * N * N * d * ((N + 1) / (2 * N) if causal else 1.0)
line = f"plain B{B} H{H} N{N} d{d} causal: fwd {fwd:.3f} ms ({flops / fwd / 1e9:.0f} TF/s), bwd {ours:.3f} ms " \
       f"({2.5 * flops / ours / 1e9:.0f} TF/s)"
try:
    from flash_attn import flash_attn_func
    qf, kf, vf = (t.transpose(1, 2).contiguous().requires_grad_() for t in (q, k, v))
    of = flash_attn_func(qf, kf, vf, causal=causal)
    dof = do.transpose(1, 2).contiguous()
    fa = timed(lambda: torch.autograd.grad(of, (qf, kf, vf), dof, retain_graph=True))
    line += f"; flash_attn 2.8 bwd {fa:.3f} ms ({2.5 * flops / fa / 1e9:.0f} TF/s)"
except Exception as e:  # noqa: BLE001
    line += f"; flash_attn comparator unavailable ({str(e)[:60]})"
print(line, flush=True)
