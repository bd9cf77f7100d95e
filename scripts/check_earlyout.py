"""K5's exact pass-2 early-out vs K4 (which never skips): O and L bitwise equal
on inputs where few / some / most 16-key P blocks fall below 2^-11. GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

for n, causal in ((4096, False), (4000, True), (32760, False)):
    for qs in (0.1, 0.3, 0.6, 1.0):
        g = torch.Generator(device="cuda").manual_seed(7)
        q, k, v = (torch.randn(1, 2, n, 128, generator=g, device="cuda") for _ in range(3))
        q = (q * qs).bfloat16()
        k, v = k.bfloat16(), v.bfloat16()
        o_t, l_t, _, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
        o_i, l_i, _, _ = aq.attn_forward(q, k, v, causal=causal, train=False)
        print(f"n={n} causal={causal} q*{qs}: O equal {torch.equal(o_t, o_i)}  L equal {torch.equal(l_t, l_i)}  "
              f"max|dO| {(o_t.float() - o_i.float()).abs().max().item():.3e}", flush=True)
