"""The oracle's SageAttention3 restatement vs the reference goldens (CPU)."""

import os

import numpy as np
import pytest

from oracle import nvfp4_attn_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sg():
    return np.load(os.path.join(GOLD, "sage3.npz"))


def case(sg, name):
    n_q, n_k, d, causal, b_q, b_k, sq, sk, tl, qz = (int(x) for x in sg[f"{name}_meta"])
    return (sg[f"{name}_Q"], sg[f"{name}_K"], sg[f"{name}_V"],
            dict(causal=bool(causal), b_q=b_q, b_k=b_k, smooth_q=bool(sq), smooth_k=bool(sk),
                 two_level_p=bool(tl), quantized=bool(qz)))


NAMES = ["s16", "s64c", "s128", "s32", "srow", "srowc", "noTL", "kOnly", "qOnly", "none", "s48", "s256c", "s80c"]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_sage3_matches_reference(sg, name):
    Q, K, V, kw = case(sg, name)
    O, L = orc.sage3_forward(Q, K, V, width=32, **kw)
    np.testing.assert_array_equal(O, sg[f"{name}_O"])
    np.testing.assert_array_equal(L, sg[f"{name}_L"])


def test_two_level_scale_properties():
    # test_sage3.py:101-118
    s, r = orc.two_level_scale(np.zeros((4, 16)))
    assert np.all(r == 1.0) and np.all(s == 0)
    P = np.zeros((1, 16))
    P[0, 0] = orc.P_RESCALE_MAX
    assert orc.two_level_scale(P)[1][0] == 1.0
    P = np.random.default_rng(22).uniform(0, 1, (8, 32))
    s, r = orc.two_level_scale(P)
    assert np.all(s.max(axis=1) <= orc.P_RESCALE_MAX)


def test_smooth_properties():
    # test_sage3.py:26-63
    g = np.random.default_rng(3)
    Q, K = g.standard_normal((64, 32)), g.standard_normal((80, 32))
    gq, gk, q_bar, k_bar = orc.smooth(Q, K, 16)
    assert np.max(np.abs(gk.mean(axis=0))) <= 1e-6
    assert np.max(np.abs(gq.reshape(4, 16, 32).mean(axis=1))) <= 1e-6
    np.testing.assert_allclose(gq + np.repeat(q_bar, 16, axis=0), Q, rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        orc.smooth(np.zeros((10, 8)), np.zeros((10, 8)), 3)


def test_sage3_api_validates_before_touching_the_gpu():
    # TileConfig.validate / accum_width checks run on the host (flash.py:60-71)
    import paper_2603_00040_b200 as aq
    Q = np.zeros((256, 64))
    with pytest.raises(aq.TileError):
        aq.sage3_forward(Q, Q, Q, aq.TileConfig(b_q=96, b_k=128))
    with pytest.raises(aq.InvalidValue):
        aq.sage3_forward(Q, Q, Q, aq.TileConfig(b_q=128, b_k=128, accum_width=64))
    assert aq.P_RESCALE_MAX == orc.P_RESCALE_MAX == 2688.0


def test_quant_points_semantics():
    # oracle.py:27-46
    import paper_2603_00040_b200 as aq
    assert aq.QuantPoints() == aq.QuantPoints.all_on()
    assert aq.QuantPoints.all_on().any and not aq.QuantPoints.all_off().any
    assert aq.QuantPoints(p=False).any and aq.QuantPoints(False, False, False, True).p


def test_tracking_api():
    # tracking.py:16-69: live / peak bookkeeping, scopes release their registrations
    from paper_2603_00040_b200 import tracking
    assert tracking.track(np.zeros(4)) is not None          # no tracker: a no-op
    with tracking.AllocationTracker() as t:
        tracking.track(np.zeros(100))                       # 800 bytes
        with tracking.scope():
            tracking.track(np.zeros(50))                    # 400 bytes, released on exit
        assert t.live == 800
    assert t.peak >= 1200


def test_reference_api_rejects_non_finite_before_the_gpu():
    # codec.py:313-314 through fake_quantize / quantize in the flash functions
    import paper_2603_00040_b200 as aq
    Q = np.zeros((128, 64))
    bad = Q.copy()
    bad[3, 5] = np.nan
    cfg = aq.TileConfig(b_q=128, b_k=128)
    for fn in (aq.flash_forward_training, aq.flash_forward_inference):
        with pytest.raises(aq.InvalidValue):
            fn(bad, Q, Q, cfg)
    with pytest.raises(aq.InvalidValue):
        aq.sage3_forward(Q, Q, np.where(Q == 0, np.inf, Q), cfg)
