"""Per-segment cycle breakdown of the backward compute warps (library built with -DAQ_BWD_PROFILE)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from paper_2603_00040_b200 import _lib  # noqa: E402

B, H, N, d = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 32, 4096, 128)
lib = _lib.load()
q, k, v, do = (torch.randn(B, H, N, d, device="cuda").bfloat16() for _ in range(4))
o, lse, ohp, ws = aq.attn_forward(q, k, v, causal=True, train=True, keep_for_bwd=True)
aq.attn_backward(q, k, v, do, o, ohp, lse, causal=True, fwd_workspace=ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
lib.aq_debug_bwd_profile(buf, 1)
aq.attn_backward(q, k, v, do, o, ohp, lse, causal=True, fwd_workspace=ws)
torch.cuda.synchronize()
lib.aq_debug_bwd_profile(buf, 0)
v = list(buf)
kv = ["S wait+ld", "P exp", "PF_FREE wait", "P^F write+arrive", "dP wait+ld", "DS_FREE wait", "dS write+arrive"]
qn = ["S wait+ld", "P exp", "dP wait+ld", "DS_EMPTY wait", "dS write+arrive"]
print("KV role, cycles per warp-tile:")
for i, n in enumerate(kv):
    print(f"  {n:18s} {v[i] / max(1, v[14]):9.1f}")
print("Q role, cycles per warp-tile:")
for i, n in enumerate(qn):
    print(f"  {n:18s} {v[8 + i] / max(1, v[15]):9.1f}")
