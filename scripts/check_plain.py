"""quantized=False forward: the hand-written kernel vs FlashAttention-2 (agreement and time)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00040_b200 import plain  # noqa: E402


def t(fn, reps=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (B, H, N, d, causal, dt) in [(1, 2, 384, 64, True, torch.bfloat16), (2, 3, 200, 128, False, torch.float16),
                                 (4, 32, 8192, 128, True, torch.bfloat16), (4, 32, 8192, 64, True, torch.bfloat16)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(B * H, N, d, generator=g, device="cuda").to(dt) for _ in range(3))
    o1, l1 = plain._plain_forward_b200(q, k, v, causal, dt)
    fa = plain._flash()
    sc = 1.0 / math.sqrt(d)
    out, lse, _, _ = fa._flash_attn_forward(q.unsqueeze(2), k.unsqueeze(2), v.unsqueeze(2), 0.0, sc, causal, -1, -1,
                                            0.0, None, False)
    o2, l2 = out.squeeze(2), lse.squeeze(1)
    err = float((o1.float() - o2.float()).norm() / o2.float().norm())
    lerr = float((l1 - l2).abs().max())
    line = f"B{B} H{H} N{N} d{d} causal={causal} {dt}: O rel-L2 vs FA2 {err:.2e}, L max {lerr:.1e}"
    if N >= 4096:
        f = 4.0 * B * H * N * N * d * ((N + 1) / (2 * N) if causal else 1.0)
        ta = t(lambda: plain._plain_forward_b200(q, k, v, causal, dt))
        tb = t(lambda: fa._flash_attn_forward(q.unsqueeze(2), k.unsqueeze(2), v.unsqueeze(2), 0.0, sc, causal, -1, -1,
                                              0.0, None, False))
        line += f"; ours {ta:.3f} ms = {f / ta / 1e9:.0f} TF/s, FA2 {tb:.3f} ms = {f / tb / 1e9:.0f} TF/s"
    print(line, flush=True)
