"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``attnqat`` read-only from /root/reference/pkg/src, feeds it
bf16-representable inputs (so the GPU can receive bit-identical values) and
stores inputs + reference outputs as compressed .npz files next to this
script. The GPU box never reads /root/reference; the tests only read these
committed fixtures.
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


def adversarial_rows(rng):
    """Codec edge cases: midpoints +-1ulp, E4M3 midpoints x6, -0.0, tiny blocks,
    saturation, small negatives that round to the 0x8 nibble."""
    import attnqat.codec as C

    rows = []
    mids = (C._FP4_POS[:-1] + C._FP4_POS[1:]) / 2.0
    # FP4 midpoints under a unit scale (block max 6 -> scale exactly 1.0)
    for m in mids:
        for v in (m, np.nextafter(np.float32(m), 0), np.nextafter(np.float32(m), 10)):
            r = np.zeros(16)
            r[0] = 6.0
            r[1:8] = v
            r[8:15] = -v
            r[15] = -0.0
            rows.append(r)
    # E4M3 midpoints times 6 (scale rounding ties), +-1 ulp in fp32
    e4 = C._E4M3_MIDS
    for m in e4[::3]:
        for v in (6 * m, np.nextafter(np.float32(6 * m), 0), np.nextafter(np.float32(6 * m), 1e9)):
            r = np.linspace(-1, 1, 16) * float(v)
            r[3] = float(v)
            rows.append(r)
    # tiny blocks -> scale bump to 0x01 (test_codec.py:206-211)
    for t in (1e-6, 1e-5, 3e-4, 1e-3, 2.0 ** -12, 2.0 ** -11):
        rows.append(rng.standard_normal(16) * t)
    # saturation: block max beyond 448*6
    rows.append(np.linspace(-1e5, 1e5, 16))
    rows.append(np.full(16, 3000.0))
    # exact zeros / negative zeros / small negatives
    rows.append(np.zeros(16))
    r = np.zeros(16)
    r[0] = 6.0
    r[1] = -0.1
    r[2] = -0.0
    rows.append(r)
    r = np.full(16, -0.0)
    rows.append(r)
    arr = np.array(rows, dtype=np.float64)
    return arr.astype(np.float32).astype(np.float64)  # fp32-representable


def main():
    sys.path.insert(0, REF)
    import attnqat
    from attnqat import codec as C
    from attnqat.flash import (BwdVariant, TileConfig, flash_backward,
                               flash_forward_inference, flash_forward_training)
    from attnqat.oracle import QuantPoints, oracle_forward
    from attnqat.tensors import Rng, randn

    rng = np.random.default_rng(7)

    # ---- codec ----------------------------------------------------------
    x_randn = bf16(rng.standard_normal((256, 128)))
    x_wide = bf16(rng.standard_normal((64, 64)) * np.exp(rng.uniform(-12, 9, (64, 1))))
    x_adv = adversarial_rows(rng)
    # fp32-valued (non-bf16) inputs exercise the IEEE-division requirement
    x_f32 = rng.standard_normal((128, 64)).astype(np.float32).astype(np.float64)
    codec = {}
    for name, x in (("randn", x_randn), ("wide", x_wide), ("adv", x_adv), ("f32", x_f32)):
        qt = C.quantize(x)
        codec[f"{name}_x"] = x
        codec[f"{name}_codes"] = qt.codes
        codec[f"{name}_scales"] = qt.scales
        codec[f"{name}_fq"] = C.fake_quantize(x)
    # V operand: blocks along tokens, ragged token count (zero-padded tail)
    v = bf16(rng.standard_normal((200, 64)))
    vt = C.quantize_padded(np.ascontiguousarray(v.T))
    codec["vcols_x"] = v
    codec["vcols_codes"] = vt.codes
    codec["vcols_scales"] = vt.scales
    codec["vcols_fq"] = C.fake_quantize_cols(v)
    codec["golden_2p4375"] = C.fake_quantize(np.array([[2.5] + [0.0] * 15]))
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **codec)

    # ---- attention --------------------------------------------------------
    def gen(seed, n_q, n_k, d):
        r = Rng(seed)
        return (bf16(randn((n_q, d), r)), bf16(randn((n_k, d), r)),
                bf16(randn((n_k, d), r)))

    cases = {
        # C1 parity config (BASELINE.json configs[0]): B1 H2 N256 d64, both heads
        "c1h0": dict(seed=0, n_q=256, n_k=256, d=64, causal=False, bq=128, bk=128),
        "c1h1": dict(seed=100, n_q=256, n_k=256, d=64, causal=False, bq=128, bk=128),
        "c1h0c": dict(seed=0, n_q=256, n_k=256, d=64, causal=True, bq=128, bk=128),
        "d128": dict(seed=3, n_q=256, n_k=256, d=128, causal=False, bq=128, bk=128),
        "d128c": dict(seed=4, n_q=384, n_k=384, d=128, causal=True, bq=128, bk=128),
        # right-aligned causal with N_q < N_k
        "offc": dict(seed=5, n_q=128, n_k=256, d=64, causal=True, bq=64, bk=128),
        # ragged N (not a multiple of 16): single key tile, padded P/V blocks
        "ragged": dict(seed=6, n_q=200, n_k=200, d=64, causal=False, bq=200, bk=200),
    }
    att = {}
    for name, c in cases.items():
        Q, K, V = gen(c["seed"], c["n_q"], c["n_k"], c["d"])
        dO = bf16(randn((c["n_q"], c["d"]), Rng(c["seed"] + 1)))
        cfg = TileConfig(b_q=c["bq"], b_k=c["bk"], causal=c["causal"], accum_width=32)
        tr = flash_forward_training(Q, K, V, cfg)
        inf = flash_forward_inference(Q, K, V, cfg)
        att[f"{name}_Q"], att[f"{name}_K"], att[f"{name}_V"] = Q, K, V
        att[f"{name}_dO"] = dO
        att[f"{name}_meta"] = np.array([c["n_q"], c["n_k"], c["d"], int(c["causal"]), c["bq"], c["bk"]])
        att[f"{name}_O"], att[f"{name}_L"], att[f"{name}_Op"] = tr.O, tr.L, tr.O_prime
        att[f"{name}_Oinf"] = inf.O
        for var in BwdVariant:
            g = flash_backward(Q, K, V, dO, tr, cfg, variant=var)
            tag = var.value.replace("-", "_")
            att[f"{name}_{tag}_dQ"], att[f"{name}_{tag}_dK"], att[f"{name}_{tag}_dV"] = g.dQ, g.dK, g.dV
    # the reference oracle's own pinned instance (test_oracle.py:97-103)
    r = Rng(1234)
    Q, K, V = randn((8, 16), r), randn((8, 16), r), randn((8, 16), r)
    o = oracle_forward(Q, K, V, points=QuantPoints.all_on(), accum_width=64)
    att["g1234_Q"], att["g1234_K"], att["g1234_V"] = Q, K, V
    att["g1234_O"], att["g1234_L"], att["g1234_Op"] = o.O, o.L, o.O_prime
    att["ref_version"] = np.array(attnqat.__version__)
    # bf16-valued inputs are exact in float32; halve the fixture size
    for k in list(att):
        if k.endswith(("_Q", "_K", "_V", "_dO")) and not k.startswith("g1234"):
            att[k] = att[k].astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **att)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
