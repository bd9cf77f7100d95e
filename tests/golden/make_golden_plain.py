"""Golden outputs of the REFERENCE's quantized=False (plain attention) path.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_plain.py

flash_forward_training(..., quantized=False) and flash_backward(...,
quantized=False) (flash.py:176-246, 317-390) on bf16-representable inputs,
fp64 accumulation, for a non-causal, a causal and a right-aligned causal
(n_q < n_k) case. Writes plain.npz next to this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {"p64": (256, 256, 64, False), "p128c": (256, 256, 128, True), "poffc": (128, 384, 64, True)}


def bf16(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().double().numpy()


def main():
    sys.path.insert(0, REF)
    import attnqat as A

    out = {}
    for i, (name, (n_q, n_k, d, causal)) in enumerate(CASES.items()):
        g = np.random.default_rng(100 + i)
        Q, dO = bf16(g.standard_normal((n_q, d))), bf16(g.standard_normal((n_q, d)))
        K, V = bf16(g.standard_normal((n_k, d))), bf16(g.standard_normal((n_k, d)))
        cfg = A.TileConfig(b_q=n_q, b_k=n_k, causal=causal, accum_width=64)
        o = A.flash_forward_training(Q, K, V, cfg, quantized=False)
        gr = A.flash_backward(Q, K, V, dO, o, cfg, quantized=False)
        for k_, v_ in dict(Q=Q, K=K, V=V, dO=dO, O=o.O, L=o.L, Op=o.O_prime, dQ=gr.dQ, dK=gr.dK, dV=gr.dV).items():
            out[f"{name}_{k_}"] = v_
        out[f"{name}_meta"] = np.array([n_q, n_k, d, int(causal)])
    np.savez_compressed(os.path.join(HERE, "plain.npz"), **out)
    print("wrote plain.npz")


if __name__ == "__main__":
    main()
