"""Time the fused attention kernel alone (pre-staged operands) and the full forward. GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402


def run(B, H, N, d, causal, train, reps=10):
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(B, H, N, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    o, lse, ohp, ws = aq.attn_forward(q, k, v, causal=causal, train=train)
    torch.cuda.synchronize()

    def t(fn):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps
    full = t(lambda: aq.attn_forward(q, k, v, causal=causal, train=train, workspace=ws))
    kern = t(lambda: aq.attn_forward(q, k, v, causal=causal, train=train, workspace=ws, operands_staged=True))
    f = 4.0 * B * H * N * N * d * ((N + 1) / (2 * N) if causal else 1.0)
    print(f"B{B} H{H} N{N} d{d} causal={causal} train={train}: full {full:.3f} ms ({f/full/1e9:.0f} TF/s)  "
          f"kernel {kern:.3f} ms ({f/kern/1e9:.0f} TF/s)", flush=True)


CASES = [(4, 32, 8192, 128, True, False), (1, 40, 32760, 128, False, False), (8, 32, 4096, 128, True, True),
         (4, 32, 8192, 64, True, False), (8, 32, 4096, 128, True, False), (4, 32, 8192, 128, True, True)]

if __name__ == "__main__":
    sel = [int(a) for a in sys.argv[1:]] or range(len(CASES))
    for i in sel:
        run(*CASES[i], reps=3 if i == 1 else 10)
