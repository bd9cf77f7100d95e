"""One C2-shape quantized=False forward (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00040_b200 import plain  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(128, 8192, 128, generator=g, device="cuda").bfloat16() for _ in range(3))
for _ in range(2):
    plain._plain_forward_b200(q, k, v, True, torch.bfloat16)
torch.cuda.synchronize()
