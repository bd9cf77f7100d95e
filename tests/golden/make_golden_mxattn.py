"""Golden outputs of the REFERENCE's MXFP4 inference / training forwards and backward.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_mxattn.py

flash_forward_inference / flash_forward_training(Q, K, V, TileConfig(...,
spec=MXFP4)) (flash.py:176-314 with the MXFP4 codec, codec.py:123-203) on bf16-representable inputs, fp32
accumulation. Writes mxattn.npz next to this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
# name: (n_q, n_k, d, causal, b_q, b_k)
CASES = {"m64": (256, 256, 64, False, 128, 128), "m128c": (256, 384, 128, True, 128, 128),
         "mrag": (200, 200, 64, True, 200, 200)}


def bf16(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().double().numpy()


def main():
    sys.path.insert(0, REF)
    from attnqat.codec import MXFP4
    from attnqat.flash import TileConfig, flash_backward, flash_forward_inference, flash_forward_training

    out = {}
    for i, (name, (n_q, n_k, d, causal, b_q, b_k)) in enumerate(CASES.items()):
        g = np.random.default_rng(500 + i)
        Q, K, V = (bf16(g.standard_normal((n, d))) for n in (n_q, n_k, n_k))
        cfg = TileConfig(b_q=b_q, b_k=b_k, causal=causal, accum_width=32, spec=MXFP4)
        o = flash_forward_inference(Q, K, V, cfg)
        t = flash_forward_training(Q, K, V, cfg)
        dO = bf16(g.standard_normal((n_q, d)))
        gr = flash_backward(Q, K, V, dO, t, cfg)
        for k_, v_ in dict(Q=Q, K=K, V=V, O=o.O, L=o.L, Otr=t.O, Ltr=t.L, Op=t.O_prime, dO=dO, dQ=gr.dQ, dK=gr.dK,
                           dV=gr.dV).items():
            out[f"{name}_{k_}"] = v_
        out[f"{name}_meta"] = np.array([n_q, n_k, d, int(causal), b_q, b_k])
        print(name, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "mxattn.npz"), **out)
    print("wrote mxattn.npz")


if __name__ == "__main__":
    main()
