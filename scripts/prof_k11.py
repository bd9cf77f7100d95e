"""Wait breakdown of the split-pass forwards' softmax groups: K11 (training,
built with -DAQ_FWDQ_PROFILE) or, with AQ_PROF_INFER=1, K5 (inference,
-DAQ_FWDI_PROFILE); AQ_FWD_DEBUG=32. GPU.
    python scripts/prof_k11.py [B H N d causal]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from paper_2603_00040_b200 import _lib  # noqa: E402

lib = _lib.load()
infer = os.environ.get("AQ_PROF_INFER", "0") == "1"
fn = lib.aq_debug_fwdi_profile if infer else lib.aq_debug_fwdq_profile
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
a = sys.argv[1:]
B, H, N, d = (int(x) for x in a[:4]) if len(a) >= 4 else (8, 32, 4096, 128)
causal = (a[4] != "0") if len(a) > 4 else True
q, k, v = (torch.randn(B, H, N, d, device="cuda").bfloat16() for _ in range(3))
o, lse, _, ws = aq.attn_forward(q, k, v, causal=causal, train=not infer)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
fn(buf, 1)
aq.attn_forward(q, k, v, causal=causal, train=not infer, workspace=ws, operands_staged=True)
torch.cuda.synchronize()
fn(buf, 0)
v = list(buf)
ta, tb = v[3] or 1, v[13] or 1
print(f"B{B} H{H} N{N} d{d} causal={causal}: per warp-tile cycles")
print(f"  group A: total {v[2] / ta:.0f}  S_A wait {v[0] / ta:.0f}  L_EMPTY wait {v[1] / ta:.0f}")
print(f"  group B: total {v[14] / tb:.0f}  S_B wait {v[8] / tb:.0f}  L_FULL wait {v[9] / tb:.0f}  "
      f"P_EMPTY wait {v[10] / tb:.0f}  O_FULL wait {v[11] / tb:.0f}")
