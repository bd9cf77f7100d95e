"""GPU sage3 forward (smoothing, score decomposition, two-level P) vs the
reference's sage3_forward goldens and the oracle."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NAMES = ["s16", "s64c", "s128", "s32", "srow", "srowc", "noTL", "kOnly", "qOnly", "none", "s48", "s256c", "s80c"]
# O rel-L2 <= 2e-3 vs the goldens (measured <= 1e-4: fp32 tensor-core
# accumulation vs fixed-order fp32, plus the f16 rounding of dequant(P^F) * l / r
# under two-level P; a single P^F code flip costs ~1e-3), L <= 5e-5 absolute
# (measured <= 2.1e-5; the smoothing means are fp64 on both sides, the delta /
# bias terms fp32 in the reference order). Larger cases vs the oracle: 1e-2.
TOL_O, TOL_L = 2e-3, 5e-5


@pytest.fixture(scope="module")
def sg():
    return np.load(os.path.join(GOLD, "sage3.npz"))


def case(sg, name):
    n_q, n_k, d, causal, b_q, b_k, sq, sk, tl, qz = (int(x) for x in sg[f"{name}_meta"])
    return (sg[f"{name}_Q"], sg[f"{name}_K"], sg[f"{name}_V"], aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal)),
            dict(smooth_q=bool(sq), smooth_k=bool(sk), two_level_p=bool(tl), quantized=bool(qz)))


@pytest.mark.parametrize("name", NAMES)
def test_sage3_matches_reference(sg, name):
    Q, K, V, cfg, kw = case(sg, name)
    outs = aq.sage3_forward(Q, K, V, cfg, **kw)
    assert outs.O_prime is None
    assert orc.rel_l2(outs.O, sg[f"{name}_O"]) <= TOL_O, name
    assert np.max(np.abs(outs.L - sg[f"{name}_L"])) <= TOL_L, name


def test_sage3_unquantized_is_plain_attention(sg):
    # test_sage3.py:137-144
    Q, K, V, cfg, _ = case(sg, "s64c")
    outs = aq.sage3_forward(Q, K, V, cfg, quantized=False)
    O, L = orc.sage3_forward(Q, K, V, cfg.causal, cfg.b_q, cfg.b_k, 64, quantized=False)
    assert orc.rel_l2(outs.O, O) <= 1e-2
    assert np.max(np.abs(outs.L - L)) <= 1e-2


def test_constant_k_gives_mean_of_v():
    # test_sage3.py:146-156: constant K -> uniform attention -> O = column mean of V^F
    g = np.random.default_rng(41)
    Q = g.standard_normal((128, 64))
    K = np.tile(g.standard_normal((1, 64)), (128, 1))
    V = g.standard_normal((128, 64))
    outs = aq.sage3_forward(Q, K, V, aq.TileConfig(b_q=128, b_k=128))
    want = np.tile(orc.fake_quantize_cols(V.astype(np.float32)).mean(axis=0), (128, 1))
    np.testing.assert_allclose(outs.O, want, atol=2e-3)


def test_sage3_beats_plain_fp4_on_heavy_tailed_inputs():
    # test_sage3.py:158-178 at GPU tile sizes: smoothing + two-level P should not lose
    wins = 0
    for seed in range(5):
        g = np.random.default_rng(seed + 100)
        n, d = 256, 64
        Q = g.standard_normal((n, d)) + 3.0
        K = g.standard_normal((n, d)) + 3.0
        K = np.where(g.uniform(size=(n, d)) < 0.02, K * 10.0, K)
        V = g.standard_normal((n, d))
        ref = orc.oracle_forward(Q, K, V, width=64, points=(False,) * 4)["O"]
        cfg = aq.TileConfig(b_q=128, b_k=128)
        plain = aq.flash_forward_inference(Q, K, V, cfg).O
        sage = aq.sage3_forward(Q, K, V, cfg).O
        wins += np.linalg.norm(sage - ref) <= np.linalg.norm(plain - ref)
    assert wins >= 4


@pytest.mark.parametrize("n,d,causal,b_k", [(1024, 128, True, 128), (640, 64, False, 32), (512, 128, False, 512)])
def test_sage3_larger_vs_oracle(n, d, causal, b_k):
    g = np.random.default_rng(n + d)
    Q, K, V = (torch.from_numpy(g.standard_normal((n, d)) + 1.0).bfloat16().double().numpy() for _ in range(3))
    cfg = aq.TileConfig(b_q=128, b_k=b_k, causal=causal)
    outs = aq.sage3_forward(Q, K, V, cfg)
    O, L = orc.sage3_forward(Q, K, V, causal, 128, b_k, 32)
    assert orc.rel_l2(outs.O, O) <= 1e-2
    assert np.max(np.abs(outs.L - L)) <= TOL_L


def test_sage3_batched_torch_api_matches_per_head():
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, v = (torch.randn(2, 3, 384, 128, generator=g, device="cuda").bfloat16() + 2 for _ in range(3))
    o, lse = aq.attn_forward_sage3(q, k, v, causal=True, b_q=128, b_k=64)
    assert o.shape == q.shape and lse.shape == q.shape[:-1]
    o1, l1 = aq.attn_forward_sage3(q[1, 2], k[1, 2], v[1, 2], causal=True, b_q=128, b_k=64)
    assert torch.equal(o[1, 2], o1) and torch.equal(lse[1, 2], l1)


def test_sage3_errors():
    q = torch.randn(512, 64, device="cuda")
    with pytest.raises(aq.TileError):
        aq.attn_forward_sage3(q, q, q, b_q=96, b_k=128)   # b_q must divide n_q
    with pytest.raises(aq.TileError):
        aq.attn_forward_sage3(q, q, q, b_q=128, b_k=48)   # b_k must divide n_k
    with pytest.raises(aq.TileError):
        aq.attn_forward_sage3(q, q, q, b_q=128, b_k=40)    # b_k must be a multiple of 16
    aq.attn_forward_sage3(q, q, q, b_q=128, b_k=256)       # segments spanning two kernel tiles


def test_sage3_input_dtypes_agree():
    # bf16-representable values given as bf16, fp16 (exact here) and fp32: same
    # centred operands, so the same bits out
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn(2, 256, 64, generator=g, device="cuda").bfloat16() for _ in range(3))
    ref = aq.attn_forward_sage3(q, k, v, causal=True, b_q=64, b_k=64, out_dtype=torch.float32)
    for dt in (torch.float32, torch.float16):
        o, l = aq.attn_forward_sage3(q.to(dt), k.to(dt), v.to(dt), causal=True, b_q=64, b_k=64,
                                     out_dtype=torch.float32)
        assert torch.equal(o, ref[0]) and torch.equal(l, ref[1]), dt


def test_sage3_helpers_match_oracle():
    """smooth / decompose_scores / quantize_p_two_level (sage3.py:45-110) on the
    device vs the oracle restatement: means and gammas to fp64 rounding, the
    decomposition reconstructs S, two-level codes byte-identical."""
    rng = np.random.default_rng(7)
    Q = rng.standard_normal((256, 64)) + 3.0
    K = rng.standard_normal((192, 64)) - 1.0
    pair = aq.smooth(Q, K, 128)
    gq, gk, qb, kb = orc.smooth(Q, K, 128)
    for got, want in ((pair.gamma_q, gq), (pair.gamma_k, gk), (pair.q_bar, qb), (pair.k_bar, kb)):
        assert isinstance(got, np.ndarray) and got.dtype == np.float64
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-13)
    dec = aq.decompose_scores(pair, 1, 1, 64)
    assert dec.main.shape == (128, 64) and dec.delta_s.shape == (1, 64) and dec.bias.shape == (128, 1)
    S = Q[128:256] @ K[64:128].T
    np.testing.assert_allclose(dec.reconstruct(), S, rtol=0, atol=1e-10)
    with pytest.raises(aq.ShapeError):
        aq.decompose_scores(pair, 5, 0, 64)
    with pytest.raises(aq.ShapeError):
        aq.smooth(Q, K, 100)
    # two-level P: a softmax-like tile with a zero row and a ragged width
    P = np.exp(rng.standard_normal((64, 200)) * 3.0)
    P /= P.sum(axis=1, keepdims=True)
    P[5] = 0.0
    tl = aq.quantize_p_two_level(P)
    scaled, r = orc.two_level_scale(P)
    codes, scales = orc.quantize_padded(scaled)
    np.testing.assert_allclose(tl.row_factor, r, rtol=1e-15)
    assert tl.row_factor[5] == 1.0
    assert np.array_equal(np.asarray(tl.codes.codes), codes) and np.array_equal(np.asarray(tl.codes.scales), scales)
    with pytest.raises(aq.InvalidValue):
        aq.quantize_p_two_level(-P)
