"""GPU fused forward vs the reference golden outputs (and the oracle)."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["c1h0", "c1h1", "c1h0c", "d128", "d128c", "offc", "ragged"]

# Tolerances (vs the reference, fp32 tensor-core accumulation vs fixed-order
# fp32): O rel-L2 <= 1e-2 (a single P^F code flip costs ~1e-3), O' <= 2e-3,
# L <= 2e-5 absolute.
TOL_O, TOL_OP, TOL_L = 1e-2, 2e-3, 2e-5


@pytest.fixture(scope="module")
def att():
    return np.load(os.path.join(GOLD, "attention.npz"))


def _case(att, name):
    n_q, n_k, d, causal, bq, bk = (int(x) for x in att[f"{name}_meta"])
    Q, K, V = (att[f"{name}_{t}"] for t in "QKV")
    return Q, K, V, bool(causal), bq, bk


@pytest.mark.parametrize("name", CASES)
def test_training_forward_matches_reference(att, name):
    Q, K, V, causal, bq, bk = _case(att, name)
    outs = aq.flash_forward_training(Q, K, V, aq.TileConfig(b_q=bq, b_k=bk, causal=causal))
    assert orc.rel_l2(outs.O, att[f"{name}_O"]) <= TOL_O
    assert orc.rel_l2(outs.O_prime, att[f"{name}_Op"]) <= TOL_OP
    assert np.max(np.abs(outs.L - att[f"{name}_L"])) <= TOL_L


@pytest.mark.parametrize("name", CASES)
def test_inference_forward_matches_reference(att, name):
    Q, K, V, causal, bq, bk = _case(att, name)
    outs = aq.flash_forward_inference(Q, K, V, aq.TileConfig(b_q=bq, b_k=bk, causal=causal))
    assert outs.O_prime is None
    assert orc.rel_l2(outs.O, att[f"{name}_Oinf"]) <= TOL_O
    assert np.max(np.abs(outs.L - att[f"{name}_L"])) <= TOL_L


@pytest.mark.parametrize("causal", [False, True])
def test_training_o_equals_inference_o_bitwise(causal):
    # analogue of test_flash.py:129-137: same MMA kinds and order -> same bits
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(2, 3, 512, 128, generator=g, device="cuda").bfloat16() for _ in range(3))
    o_t, l_t, _, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
    o_i, l_i, _, _ = aq.attn_forward(q, k, v, causal=causal, train=False)
    assert torch.equal(o_t, o_i)
    assert torch.equal(l_t, l_i)


def test_zero_v_gives_zero_o():
    # test_flash.py:63-70
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k = (torch.randn(1, 256, 64, generator=g, device="cuda") for _ in range(2))
    o, lse, o_hp, _ = aq.attn_forward(q, k, torch.zeros_like(q), train=True)
    assert torch.all(o == 0) and torch.all(o_hp == 0)
    _, lse2, _, _ = aq.attn_forward(q, k, torch.randn_like(q), train=True)
    assert torch.equal(lse, lse2)


@pytest.mark.parametrize("n,d,causal", [(1024, 128, False), (1000, 64, True), (2048, 128, True)])
def test_larger_vs_oracle(n, d, causal):
    g = np.random.default_rng(n + d)
    Q, K, V = (torch.from_numpy(g.standard_normal((n, d))).bfloat16().double().numpy() for _ in range(3))
    outs = aq.flash_forward_training(Q, K, V, aq.TileConfig(b_q=n, b_k=n, causal=causal))
    O, L, Op = orc.forward_training(Q, K, V, causal, 128 if n % 128 == 0 else n, 128 if n % 128 == 0 else n,
                                    32, ordered=False)
    assert orc.rel_l2(outs.O, O) <= TOL_O
    assert orc.rel_l2(outs.O_prime, Op) <= TOL_OP
    assert np.max(np.abs(outs.L - L)) <= 5e-5


def test_errors():
    q = np.zeros((128, 64))
    with pytest.raises(aq.TileError):
        aq.flash_forward_training(q, q, q, aq.TileConfig(b_q=100, b_k=128))
    with pytest.raises(aq.ShapeError):
        aq.flash_forward_training(np.zeros((128, 24)), np.zeros((128, 24)), np.zeros((128, 24)),
                                  aq.TileConfig(b_q=128, b_k=128))
    with pytest.raises(aq.ShapeError):
        aq.flash_forward_training(np.zeros((256, 64)), q, q, aq.TileConfig(b_q=128, b_k=128, causal=True))
