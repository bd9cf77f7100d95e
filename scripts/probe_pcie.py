"""PCIe copy-rate probe and host-pipeline chunk sweep (GPU)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

B, H, N, d = 4, 32, 8192, 128
hq, hk, hv = (torch.randn(B, H, N, d).bfloat16().pin_memory() for _ in range(3))
ho = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
hl = torch.empty(B, H, N, dtype=torch.float32).pin_memory()
dq, dk, dv = (torch.empty(B, H, N, d, dtype=torch.bfloat16, device="cuda") for _ in range(3))


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


nb = hq.numel() * 2
t = timed(lambda: [x.copy_(h, non_blocking=True) for x, h in ((dq, hq), (dk, hk), (dv, hv))])
print(f"H2D 3 x {nb/1e6:.0f} MB one stream: {t:.2f} ms  {3*nb/t/1e6:.1f} GB/s")
t = timed(lambda: ho.copy_(dq, non_blocking=True))
print(f"D2H 1 x {nb/1e6:.0f} MB: {t:.2f} ms  {nb/t/1e6:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        for x, h in ((dq, hq), (dk, hk), (dv, hv)):
            x.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(dq, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(both)
print(f"H2D 805MB || D2H 268MB: {t:.2f} ms  {4*nb/t/1e6:.1f} GB/s total")
for ch in (128, 64, 32, 16, 8):
    t = timed(lambda: aq.attn_forward_host(hq, hk, hv, causal=True, train=False, out=ho, lse_out=hl, chunk_heads=ch))
    print(f"attn_forward_host chunk_heads={ch}: {t:.2f} ms")

# bench-style host buffers: generated on the device, copied back, pinned
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, d, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
bq, bk, bv = (x.cpu().pin_memory() for x in (q, k, v))
for ch in (16, 8):
    t = timed(lambda: aq.attn_forward_host(bq, bk, bv, causal=True, train=False, out=ho, lse_out=hl, chunk_heads=ch))
    print(f"bench-style buffers attn_forward_host chunk_heads={ch}: {t:.2f} ms")
print("pinned:", bq.is_pinned(), hq.is_pinned(), bq.data_ptr() % 4096, bq.is_contiguous())
t = timed(lambda: [x.copy_(h, non_blocking=True) for x, h in ((dq, bq), (dk, bk), (dv, bv))])
print(f"H2D bench-style 3 x {nb/1e6:.0f} MB one stream: {t:.2f} ms  {3*nb/t/1e6:.1f} GB/s")
