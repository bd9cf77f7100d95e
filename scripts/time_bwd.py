"""Time the fused backward alone on the C4 shape (GPU)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

B, H, N, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 32, 4096, 128)))
causal = True
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(B, H, N, d, generator=g, device="cuda").bfloat16() for _ in range(4))
o, lse, ohp, ws = aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True)


def f():
    aq.attn_backward(q, k, v, do, o, ohp, lse, causal=causal, fwd_workspace=ws)


for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    f()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 5
fl = 2.5 * 4.0 * B * H * N * N * d * (N + 1) / (2 * N)
print(f"bwd B{B} H{H} N{N} d{d}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TF/s (alg, bwd = 2.5 x fwd)")
