"""Same-box BF16 FlashAttention comparators on the BASELINE shapes (GPU)."""
import json
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel


def bench(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def run(B, H, N, d, causal, train=False):
    q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16, requires_grad=train) for _ in range(3))
    f = 4.0 * B * H * N * N * d * ((N + 1) / (2 * N) if causal else 1.0) * (3.5 if train else 1.0)
    out = {"shape": [B, H, N, d], "causal": causal, "train": train}
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel(be):
                if train:
                    do = torch.randn_like(q)
                    def step():
                        o = F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                        o.backward(do)
                else:
                    def step():
                        F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                ms = bench(step)
            out[name] = {"ms": ms, "tflops": f / ms / 1e9}
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": str(e)[:120]}
    try:
        from flash_attn import flash_attn_func
        qt, kt, vt = (x.detach().transpose(1, 2).contiguous() for x in (q, k, v))
        ms = bench(lambda: flash_attn_func(qt, kt, vt, causal=causal)) if not train else None
        if ms:
            out["flash_attn_2.8"] = {"ms": ms, "tflops": f / ms / 1e9}
    except Exception as e:  # noqa: BLE001
        out["flash_attn_2.8"] = {"error": str(e)[:120]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    run(4, 32, 8192, 128, True)
    run(1, 40, 32760, 128, False)
    run(8, 32, 4096, 128, True, train=True)
    run(4, 32, 8192, 64, True)
