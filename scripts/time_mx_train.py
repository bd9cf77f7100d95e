"""C4-shape MXFP4 QAT step (attn_qat(spec=MXFP4) forward + backward) vs NVFP4."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

B, H, N, D = 8, 32, 4096, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, D, generator=g, device="cuda").bfloat16().requires_grad_() for _ in range(3))
d_o = torch.randn(B, H, N, D, generator=g, device="cuda").bfloat16()
f = 14.0 * B * H * N * N * D * (N + 1) / (2 * N)
for name, spec in (("NVFP4", None), ("MXFP4", aq.MXFP4)):
    def step():
        o = aq.attn_qat(q, k, v, causal=True, spec=spec)
        o.backward(d_o)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"C4 {name} QAT step (autograd fwd+bwd): {ms:.3f} ms = {f / ms / 1e9:.0f} TF/s")
