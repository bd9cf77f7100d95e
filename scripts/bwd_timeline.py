"""Per-CTA timeline of the fused backward at C4 (library built with -DAQ_BWD_PROFILE, AQ_LIB_PATH).

Splits each SM's busy time into: CTA start -> first S tile in registers (ramp),
the tile loop, loop end -> CTA exit (epilogue), and the gaps between one CTA's
exit and the next CTA's entry on the same SM (launch), plus the grid tail."""
import ctypes
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from paper_2603_00040_b200 import _lib  # noqa: E402

B, H, N, d = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 32, 4096, 128)
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(B, H, N, d, generator=g, device="cuda").bfloat16() for _ in range(4))
o, lse, ohp, ws = aq.attn_forward(q, k, v, causal=True, train=True, keep_for_bwd=True)
for _ in range(3):
    aq.attn_backward(q, k, v, do, o, ohp, lse, causal=True, fwd_workspace=ws)
torch.cuda.synchronize()
heads = B * H
T = (N + 127) // 128
ctas = heads * (T // 2 + T) if (T % 2 == 0 and os.environ.get("AQ_TL_PAIRED", "1") == "1") else heads * 2 * T
buf = (ctypes.c_ulonglong * (5 * ctas))()
assert lib.aq_debug_bwd_timeline(buf, ctas) == 0, "not a -DAQ_BWD_PROFILE build"
a = np.frombuffer(buf, dtype=np.uint64).reshape(ctas, 5).astype(np.int64)
t0 = a[:, 0].min()
a[:, :4] -= t0
sm = a[:, 4] & 0xFFFF
kv = (a[:, 4] >> 16) & 1
span = a[:, 3].max()
ramp = a[:, 1] - a[:, 0]
loop = a[:, 2] - a[:, 1]
epi = a[:, 3] - a[:, 2]
print(f"kernel span {span / 1e3:.1f} us, {ctas} CTAs on {len(set(sm.tolist()))} SMs")
for name, m in (("KV", kv == 1), ("Q", kv == 0)):
    print(f"{name:2s} role: {m.sum():5d} CTAs  ramp {ramp[m].mean() / 1e3:6.2f} us  loop {loop[m].mean() / 1e3:6.2f} us  "
          f"epilogue {epi[m].mean() / 1e3:6.2f} us  (sums: ramp {ramp[m].sum() / 1e6:.2f} ms-SM, loop "
          f"{loop[m].sum() / 1e6:.2f}, epi {epi[m].sum() / 1e6:.2f})")
gaps, tails, heads_ = 0, 0, 0
per_sm = defaultdict(list)
for i in range(ctas):
    per_sm[int(sm[i])].append((a[i, 0], a[i, 3]))
for s_, lst in per_sm.items():
    lst.sort()
    heads_ += lst[0][0]
    for (s0, e0), (s1, e1) in zip(lst, lst[1:]):
        gaps += max(0, s1 - e0)
    tails += span - lst[-1][1]
nsm = len(per_sm)
tot = span * nsm
print(f"per-SM average: busy loop {loop.sum() / nsm / 1e3:.1f} us, ramp {ramp.sum() / nsm / 1e3:.1f}, "
      f"epilogue {epi.sum() / nsm / 1e3:.1f}, inter-CTA gaps {gaps / nsm / 1e3:.1f}, start {heads_ / nsm / 1e3:.1f}, "
      f"tail {tails / nsm / 1e3:.1f} (span {span / 1e3:.1f})")
