"""One C4-shape QAT step, NVFP4 then MXFP4 (for an ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(8, 32, 4096, 128, generator=g, device="cuda").bfloat16().requires_grad_() for _ in range(3))
d_o = torch.randn(8, 32, 4096, 128, generator=g, device="cuda").bfloat16()
for spec in (None, aq.MXFP4):
    aq.attn_qat(q, k, v, causal=True, spec=spec).backward(d_o)
torch.cuda.synchronize()
