"""MXFP4 inference forward: errors vs the reference goldens and time at C2's shape."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from oracle import nvfp4_attn_oracle as orc  # noqa: E402

mx = np.load("tests/golden/mxattn.npz")
for name in ("m64", "m128c", "mrag"):
    n_q, n_k, d, causal, b_q, b_k = (int(x) for x in mx[f"{name}_meta"])
    o = aq.flash_forward_inference(mx[f"{name}_Q"], mx[f"{name}_K"], mx[f"{name}_V"],
                                   aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal), spec=aq.MXFP4))
    print(f"{name}: O rel-L2 {orc.rel_l2(o.O, mx[name + '_O']):.2e}  L max {np.max(np.abs(o.L - mx[name + '_L'])):.1e}")
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(4, 32, 8192, 128, generator=g, device="cuda").bfloat16() for _ in range(3))
f = 4.0 * 4 * 32 * 8192 * 8192 * 128 * (8193 / 16384)
for _ in range(2):
    aq.attn_forward_mx(q, k, v, causal=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    aq.attn_forward_mx(q, k, v, causal=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"C2 MXFP4 inference fwd (full op incl. quantizers): {ms:.3f} ms = {f / ms / 1e9:.0f} TF/s")
