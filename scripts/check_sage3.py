"""Print the sage3 GPU path's errors vs the reference goldens and time it at C2 shape."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from oracle import nvfp4_attn_oracle as orc  # noqa: E402

sg = np.load("tests/golden/sage3.npz")
for name in ["s16", "s64c", "s128", "s32", "srow", "srowc", "noTL", "kOnly", "qOnly", "none", "s48", "s256c", "s80c"]:
    n_q, n_k, d, causal, b_q, b_k, sq, sk, tl, qz = (int(x) for x in sg[f"{name}_meta"])
    Q, K, V = sg[f"{name}_Q"], sg[f"{name}_K"], sg[f"{name}_V"]
    o = aq.sage3_forward(Q, K, V, aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal)), smooth_q=bool(sq),
                         smooth_k=bool(sk), two_level_p=bool(tl))
    plain = aq.flash_forward_inference(Q, K, V, aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal))).O
    ref = orc.oracle_forward(Q, K, V, causal=bool(causal), width=64, points=(False,) * 4)["O"]
    print(f"{name:6s} O rel-L2 vs reference sage3 {orc.rel_l2(o.O, sg[name + '_O']):.2e}  "
          f"L max {np.max(np.abs(o.L - sg[name + '_L'])):.1e}   err vs exact: sage3 {orc.rel_l2(o.O, ref):.3e} "
          f"plain fp4 {orc.rel_l2(plain, ref):.3e}")

B, H, N, D = 4, 32, 8192, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, D, generator=g, device="cuda").bfloat16() for _ in range(3))
flops = 4 * B * H * N * N * D * (N + 1) / (2 * N)
for tl, bk in [(True, 128), (True, 16), (False, 128)]:
    for _ in range(3):
        aq.attn_forward_sage3(q, k, v, causal=True, b_q=128, b_k=bk, two_level_p=tl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        aq.attn_forward_sage3(q, k, v, causal=True, b_q=128, b_k=bk, two_level_p=tl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"C2 sage3 two_level={tl} b_k={bk}: {ms:.3f} ms = {flops / ms / 1e9:.0f} TF/s (full op incl. smoothing)")
