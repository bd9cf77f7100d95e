"""GPU materialized oracle (oracle_forward / oracle_backward with QuantPoints)
vs the CPU restatement of oracle.py."""

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
POINTS = [(True, True, True, True), (False, False, False, False), (True, True, True, False),
          (False, True, True, True), (True, False, False, True)]


def _bf16(x):
    # bf16-representable values: the device quantizers read fp32, the CPU oracle fp64
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).bfloat16().double().numpy()


@pytest.mark.parametrize("points", POINTS, ids=lambda p: "".join("qkvp"[i] if b else "-" for i, b in enumerate(p)))
@pytest.mark.parametrize("causal", [False, True])
def test_oracle_forward_backward(points, causal):
    Q, K, V = (_bf16(x) for x in orc.make_qkv(60 + sum(points), 96, 128, 64))
    dO = _bf16(orc.randn((96, 64), 61))
    tr = aq.oracle_forward(Q, K, V, points=aq.QuantPoints(*points), causal=causal)
    ref = orc.oracle_forward(Q, K, V, causal=causal, width=32, points=points)
    # BLAS vs fixed-order fp32 accumulation: S agrees to ~1e-6 relative, which
    # can flip a P^F code at a rounding midpoint (~1e-3 of O each)
    fin = np.isfinite(ref["S"])
    assert np.array_equal(np.isfinite(tr.S), fin)
    assert orc.rel_l2(np.where(fin, tr.S, 0), np.where(fin, ref["S"], 0)) <= 1e-5
    assert np.max(np.abs(tr.L - ref["L"])) <= 1e-5
    assert orc.rel_l2(tr.P, ref["P"]) <= 1e-5
    assert orc.rel_l2(tr.O, ref["O"]) <= (1e-2 if points[3] else 1e-5)
    assert orc.rel_l2(tr.O_prime, ref["O_prime"]) <= 1e-5
    assert tr.causal == causal
    g = aq.oracle_backward(tr, ref["Qf"], ref["Kf"], ref["Vf"], dO)
    dq, dk, dv = orc.oracle_backward(ref, dO, 32)
    assert orc.rel_l2(g.dQ, dq) <= 1e-4
    assert orc.rel_l2(g.dK, dk) <= 1e-4
    assert orc.rel_l2(g.dV, dv) <= (1e-2 if points[3] else 1e-5)


def test_oracle_forward_matches_flash_training():
    # all points on: O and O' are what the fused training forward computes
    Q, K, V = (_bf16(x) for x in orc.make_qkv(70, 256, 256, 128))
    tr = aq.oracle_forward(Q, K, V, causal=True)
    outs = aq.flash_forward_training(Q, K, V, aq.TileConfig(b_q=128, b_k=128, causal=True))
    assert orc.rel_l2(outs.O, tr.O) <= 1e-2
    assert orc.rel_l2(outs.O_prime, tr.O_prime) <= 2e-3
    assert np.max(np.abs(outs.L - tr.L)) <= 2e-5


def test_oracle_errors():
    Q = np.zeros((16, 24))
    with pytest.raises(aq.ShapeError):
        aq.oracle_forward(Q, Q, Q)                                  # d % 16 with quantization on
    aq.oracle_forward(Q + 1, Q, Q, points=aq.QuantPoints.all_off())  # fine without
    with pytest.raises(aq.ShapeError):
        aq.oracle_forward(np.zeros((32, 16)), np.zeros((16, 16)), np.zeros((16, 16)), causal=True)


def test_fused_forward_memory_is_linear_in_n():
    # the use the reference's tracker exists for: fused attention keeps O(N)
    # device memory (the materialized oracle is O(N^2))
    from paper_2603_00040_b200 import tracking
    peaks = []
    for n in (2048, 4096):
        q = torch.randn(1, 4, n, 128, device="cuda").bfloat16()
        with tracking.AllocationTracker() as t:
            aq.attn_forward(q, q, q, causal=True, train=True)
        peaks.append(t.peak)
    assert 1.5 <= peaks[1] / peaks[0] <= 2.5
    with tracking.AllocationTracker() as t:
        aq.oracle_forward(*(torch.randn(1024, 64, device="cuda") for _ in range(3)))
    assert t.peak >= 1024 * 1024 * 8      # S / P materialized


def test_fd_grads_match_oracle_backward():
    # oracle.py:164-194 vs the explicit Jacobian on the unquantized path
    from paper_2603_00040_b200.materialized import fd_attention_grads
    Q, K, V = orc.make_qkv(80, 6, 8, 16)
    dO = orc.randn((6, 16), 81)
    fd = fd_attention_grads(Q, K, V, dO, causal=True)
    tr = aq.oracle_forward(Q, K, V, points=aq.QuantPoints.all_off(), causal=True, accum_width=64)
    g = aq.oracle_backward(tr, Q, K, V, dO, accum_width=64)
    for a, b in ((fd.dQ, g.dQ), (fd.dK, g.dK), (fd.dV, g.dV)):
        assert np.max(np.abs(a - b)) <= 1e-5 * max(1.0, np.max(np.abs(b)))
