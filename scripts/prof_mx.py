"""One C2-shape MXFP4 inference forward (for an ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(4, 32, 8192, 128, generator=g, device="cuda").bfloat16() for _ in range(3))
aq.attn_forward_mx(q, k, v, causal=True)
torch.cuda.synchronize()
