"""Golden MXFP4 (BlockSpec(32, E8M0)) codec vectors from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_mx.py

quantize / fake_quantize / fake_quantize_cols with MXFP4 and round_to_e8m0
(codec.py:123-203, 302-381) on float32-representable inputs, including the
power-of-two ties of the E8M0 rounding, zero blocks, -0.0 and saturation.
Writes mxfp4.npz next to this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def main():
    sys.path.insert(0, REF)
    import attnqat as A

    rng = np.random.default_rng(7)
    rows = [rng.standard_normal(64) * 10.0 ** rng.uniform(-6, 6) for _ in range(40)]
    for e in range(-20, 21, 5):                       # amax / 6 = 1.5 * 2^e exactly: ties go up
        r = rng.uniform(-1, 1, 64) * 9.0 * 2.0 ** e
        r[3] = 9.0 * 2.0 ** e
        r[40] = -9.0 * 2.0 ** e
        rows.append(r)
    z = np.zeros(64)
    z[5] = -0.0
    rows.append(z)                                    # all-zero blocks (code 0)
    s = np.zeros(64)
    s[:32] = np.linspace(-1e30, 1e30, 32)
    s[32:] = 1e-30
    rows.append(s)
    x = f32(np.stack(rows))
    qt = A.quantize(x, A.MXFP4)
    fq = A.fake_quantize(x, A.MXFP4)
    v = f32(rng.standard_normal((40, 8)) * 3)
    fqc = A.fake_quantize_cols(v, A.MXFP4)
    e8 = f32(np.concatenate([[3.0, 2.9, 3.1, 1.5, 1.0, 0.75, 6.0, 1e-30, 1e30, 2.0 ** -127, 2.0 ** 127],
                             np.abs(rng.standard_normal(200)) * 10.0 ** rng.uniform(-30, 30, 200)]))
    np.savez_compressed(os.path.join(HERE, "mxfp4.npz"), x=x, codes=qt.codes, scales=qt.scales, fq=fq, v=v, fqc=fqc,
                        e8_x=e8, e8_codes=A.round_to_e8m0(e8))
    print("wrote mxfp4.npz", x.shape)


if __name__ == "__main__":
    main()
