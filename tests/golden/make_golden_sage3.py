"""Golden outputs of the REFERENCE's sage3_forward (smoothing + two-level P).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_sage3.py

sage3_forward(Q, K, V, cfg, smooth_q, smooth_k, two_level_p, quantized)
(sage3.py:113-194) on bf16-representable inputs with a +3 common mode and 2 %
10x key outliers (the heavy-tailed setup of test_sage3.py:158-178), fp32
accumulation, over the toggle / tile / mask combinations the GPU path takes.
Writes sage3.npz next to this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
# name: (n_q, n_k, d, causal, b_q, b_k, smooth_q, smooth_k, two_level_p, quantized)
CASES = {
    "s16": (256, 256, 64, False, 16, 16, True, True, True, True),
    "s64c": (256, 256, 64, True, 64, 64, True, True, True, True),
    "s128": (256, 256, 128, False, 128, 128, True, True, True, True),
    "s32": (256, 256, 128, False, 64, 32, True, True, True, True),
    "srow": (256, 256, 64, False, 32, 256, True, True, True, True),
    "srowc": (256, 384, 64, True, 128, 384, True, True, True, True),
    "noTL": (256, 256, 64, False, 64, 32, True, True, False, True),
    "kOnly": (128, 256, 128, True, 128, 128, False, True, True, True),
    "qOnly": (256, 256, 64, False, 16, 64, True, False, True, True),
    "none": (256, 256, 64, True, 128, 128, False, False, False, True),
    "s48": (256, 384, 64, False, 64, 48, True, True, True, True),
    "s256c": (512, 512, 128, True, 128, 256, True, True, True, True),
    "s80c": (160, 320, 64, True, 32, 80, True, False, True, True),
}


def bf16(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().double().numpy()


def main():
    sys.path.insert(0, REF)
    from attnqat.flash import TileConfig
    from attnqat.sage3 import sage3_forward

    out = {}
    for i, (name, (n_q, n_k, d, causal, b_q, b_k, sq, sk, tl, qz)) in enumerate(CASES.items()):
        g = np.random.default_rng(300 + i)
        Q = bf16(g.standard_normal((n_q, d)) + 3.0)
        K = g.standard_normal((n_k, d)) + 3.0
        K = bf16(np.where(g.uniform(size=(n_k, d)) < 0.02, K * 10.0, K))
        V = bf16(g.standard_normal((n_k, d)))
        cfg = TileConfig(b_q=b_q, b_k=b_k, causal=causal, accum_width=32)
        o = sage3_forward(Q, K, V, cfg, smooth_q=sq, smooth_k=sk, two_level_p=tl, quantized=qz)
        for k_, v_ in dict(Q=Q, K=K, V=V, O=o.O, L=o.L).items():
            out[f"{name}_{k_}"] = v_
        out[f"{name}_meta"] = np.array([n_q, n_k, d, int(causal), b_q, b_k, int(sq), int(sk), int(tl), int(qz)])
        print(name, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "sage3.npz"), **out)
    print("wrote sage3.npz")


if __name__ == "__main__":
    main()
