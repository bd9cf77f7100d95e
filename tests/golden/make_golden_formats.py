"""Golden ATNQ / ATQ4 files and an FP4 KV cache written by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_formats.py

Writes, next to this script:
  ref_t32.atnq, ref_t64.atnq   save_tensor of float32 3-D / float64 1-D tensors
  ref_q.atq4                   save_quant_tensor(quantize(randn(4, 48)))
  ref_kv.k.atq4, ref_kv.vt.atq4  a 2-head FP4 KV cache (n = 200, d = 64): K rows
                               quantize(K_h) stacked over heads, V^T rows
                               quantize_padded(V_h.T) stacked over heads
  formats.npz                  the source tensors, Q, and the reference
                               flash_forward_inference O / L per head
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def bf16(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().double().numpy()


def main():
    sys.path.insert(0, REF)
    import attnqat as A
    from attnqat.codec import quantize_padded

    rng = A.Rng(21)
    t32 = A.randn((3, 5, 7), rng).astype(np.float32)
    t64 = A.randn((11,), rng)
    A.save_tensor(t32, os.path.join(HERE, "ref_t32.atnq"))
    A.save_tensor(t64, os.path.join(HERE, "ref_t64.atnq"))
    qsrc = A.randn((4, 48), rng)
    A.save_quant_tensor(A.quantize(qsrc), os.path.join(HERE, "ref_q.atq4"))

    heads, n, d = 2, 200, 64
    g = np.random.default_rng(5)
    Q, K, V = (bf16(g.standard_normal((heads, n, d))) for _ in range(3))
    kq = [A.quantize(K[h]) for h in range(heads)]
    vq = [quantize_padded(np.ascontiguousarray(V[h].T)) for h in range(heads)]
    spec = kq[0].spec
    kall = A.QuantTensor(rows=heads * n, cols=d, spec=spec, codes=np.concatenate([x.codes for x in kq]),
                         scales=np.concatenate([x.scales for x in kq]))
    vall = A.QuantTensor(rows=heads * d, cols=vq[0].cols, spec=spec, codes=np.concatenate([x.codes for x in vq]),
                         scales=np.concatenate([x.scales for x in vq]))
    A.save_quant_tensor(kall, os.path.join(HERE, "ref_kv.k.atq4"))
    A.save_quant_tensor(vall, os.path.join(HERE, "ref_kv.vt.atq4"))
    cfg = A.TileConfig(b_q=n, b_k=n, causal=False)
    outs = [A.flash_forward_inference(Q[h], K[h], V[h], cfg) for h in range(heads)]
    np.savez_compressed(os.path.join(HERE, "formats.npz"), t32=t32, t64=t64, qsrc=qsrc, Q=Q, K=K, V=V,
                        O=np.stack([o.O for o in outs]), L=np.stack([o.L for o in outs]))
    print("wrote format fixtures to", HERE)


if __name__ == "__main__":
    main()
