"""e2e (host buffers) C2 inference time vs head-chunk count (GPU)."""
import os
import sys
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
B, H, N, d = 4, 32, 8192, 128
hq, hk, hv = (torch.randn(B * H, N, d).bfloat16().pin_memory() for _ in range(3))
ho = torch.empty(B * H, N, d, dtype=torch.bfloat16).pin_memory()
hl = torch.empty(B * H, N, dtype=torch.float32).pin_memory()
flops = 4.0 * B * H * N * N * d * (N + 1) / (2 * N)
for ch in (None, 4, 8, 16, 32):
    f = lambda: aq.attn_forward_host(hq, hk, hv, causal=True, train=False, out=ho, lse_out=hl, chunk_heads=ch)  # noqa
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"chunk_heads={ch}: {ms:.2f} ms  {flops / ms / 1e9:.0f} TF/s  H2D {3 * hq.numel() * 2 / ms / 1e6:.1f} GB/s")
# raw PCIe H2D / D2H copy rates for reference
dbuf = torch.empty_like(hq, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    dbuf.copy_(hq, non_blocking=True)
torch.cuda.synchronize()
print(f"raw H2D {hq.numel() * 2 * 5 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
