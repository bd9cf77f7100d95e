"""C2-shape K4 / K5 / sage3 variants, one call each (for an ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(4, 32, 8192, 128, generator=g, device="cuda").bfloat16() for _ in range(3))
aq.attn_forward(q, k, v, causal=True, train=True)                   # K4 training
aq.attn_forward(q, k, v, causal=True, train=False)                  # K5 (or K4 with AQ_FWD_INFER=0)
for kw in [dict(smooth_q=False, smooth_k=False, two_level_p=False), dict(two_level_p=False),
           dict(smooth_q=False, smooth_k=False, two_level_p=True), dict(two_level_p=True)]:
    aq.attn_forward_sage3(q, k, v, causal=True, b_q=128, b_k=128, **kw)
torch.cuda.synchronize()
