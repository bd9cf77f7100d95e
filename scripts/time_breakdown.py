"""Per-kernel breakdown of one training step (fwd + bwd) at a given shape (GPU).

    python scripts/time_breakdown.py B H N d [causal]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

B, H, N, d = (int(x) for x in sys.argv[1:5])
causal = len(sys.argv) < 6 or sys.argv[5] != "nc"
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(B, H, N, d, generator=g, device="cuda").bfloat16() for _ in range(4))


def t(fn, reps=5):
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


o, lse, ohp, ws = aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True)
full_fwd = t(lambda: aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True, workspace=ws))
kern_fwd = t(lambda: aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True, workspace=ws,
                                     operands_staged=True))
bwd = t(lambda: aq.attn_backward(q, k, v, do, o, ohp, lse, causal=causal, fwd_workspace=ws))
f = 4.0 * B * H * N * N * d * ((N + 1) / (2 * N) if causal else 1.0)
print(f"B{B} H{H} N{N} d{d} causal={causal}: fwd full {full_fwd:.3f} ms (kernel {kern_fwd:.3f}, quantizers "
      f"{full_fwd - kern_fwd:.3f}), bwd {bwd:.3f} ms ({2.5 * f / bwd / 1e9:.0f} TF/s); step {full_fwd + bwd:.3f} ms "
      f"= {3.5 * f / (full_fwd + bwd) / 1e9:.0f} TF/s")
