"""Pin the CPU oracle (oracle/nvfp4_attn_oracle.py) against golden vectors that
tests/golden/make_golden.py produced by running the reference package itself."""

import os

import numpy as np
import pytest

from oracle import nvfp4_attn_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def codec():
    return np.load(os.path.join(GOLD, "codec.npz"))


@pytest.fixture(scope="module")
def att():
    return np.load(os.path.join(GOLD, "attention.npz"))


@pytest.mark.parametrize("name", ["randn", "wide", "adv", "f32"])
def test_quantize_bit_exact(codec, name):
    codes, scales = orc.quantize(codec[f"{name}_x"])
    np.testing.assert_array_equal(codes, codec[f"{name}_codes"])
    np.testing.assert_array_equal(scales, codec[f"{name}_scales"])
    np.testing.assert_array_equal(orc.fake_quantize(codec[f"{name}_x"]), codec[f"{name}_fq"])


def test_quantize_cols_padded(codec):
    v = codec["vcols_x"]
    codes, scales = orc.quantize_padded(np.ascontiguousarray(v.T))
    np.testing.assert_array_equal(codes, codec["vcols_codes"])
    np.testing.assert_array_equal(scales, codec["vcols_scales"])
    np.testing.assert_array_equal(orc.fake_quantize_cols(v), codec["vcols_fq"])


def test_golden_scalar_chain(codec):
    # test_codec.py:259-269: fake_quantize(2.5 in a 1x16 block) == 2.4375
    assert codec["golden_2p4375"][0, 0] == 2.4375
    assert orc.fake_quantize(np.array([[2.5] + [0.0] * 15]))[0, 0] == 2.4375


def test_negative_zero_nibbles():
    # small negative -> 0x8 nibble, exact -0.0 -> 0x0 (codec.py:84-87)
    x = np.zeros((1, 16))
    x[0, 0], x[0, 1], x[0, 2] = 6.0, -0.1, -0.0
    codes, _ = orc.quantize(x)
    assert codes[0, 0] == 0x87 and codes[0, 1] == 0x00


def test_oracle_golden_1234(att):
    tr = orc.oracle_forward(att["g1234_Q"], att["g1234_K"], att["g1234_V"], width=64)
    assert tr["O"][0, 0] == pytest.approx(0.311279296875, abs=1e-12)
    assert tr["L"][0] == pytest.approx(2.052054000774896, abs=1e-12)
    assert tr["O_prime"][3, 5] == pytest.approx(0.6328520143653195, abs=1e-12)


CASES = ["c1h0", "c1h1", "c1h0c", "d128", "d128c", "offc", "ragged"]


def _meta(att, name):
    n_q, n_k, d, causal, bq, bk = (int(v) for v in att[f"{name}_meta"])
    return n_q, n_k, d, bool(causal), bq, bk


@pytest.mark.parametrize("name", CASES)
def test_forward_training_bit_exact(att, name):
    n_q, n_k, d, causal, bq, bk = _meta(att, name)
    Q, K, V = (att[f"{name}_{t}"].astype(np.float64) for t in "QKV")
    O, L, Op = orc.forward_training(Q, K, V, causal, bq, bk, 32)
    # same fixed-order fp32 accumulation as the reference -> identical bits
    np.testing.assert_array_equal(O, att[f"{name}_O"])
    np.testing.assert_array_equal(Op, att[f"{name}_Op"])
    np.testing.assert_allclose(L, att[f"{name}_L"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", CASES)
def test_forward_inference_bit_exact(att, name):
    n_q, n_k, d, causal, bq, bk = _meta(att, name)
    Q, K, V = (att[f"{name}_{t}"].astype(np.float64) for t in "QKV")
    O, L = orc.forward_inference(Q, K, V, causal, bq, bk, 32)
    np.testing.assert_array_equal(O, att[f"{name}_Oinf"])


@pytest.mark.parametrize("name", ["c1h0", "c1h0c", "offc", "ragged"])
@pytest.mark.parametrize("variant", orc.VARIANTS)
def test_backward_bit_exact(att, name, variant):
    n_q, n_k, d, causal, bq, bk = _meta(att, name)
    Q, K, V, dO = (att[f"{name}_{t}"].astype(np.float64) for t in ("Q", "K", "V", "dO"))
    dQ, dK, dV = orc.backward(Q, K, V, dO, att[f"{name}_O"], att[f"{name}_L"],
                              att[f"{name}_Op"], causal, bq, bk, 32, variant)
    tag = variant.replace("-", "_")
    np.testing.assert_array_equal(dQ, att[f"{name}_{tag}_dQ"])
    np.testing.assert_array_equal(dK, att[f"{name}_{tag}_dK"])
    np.testing.assert_array_equal(dV, att[f"{name}_{tag}_dV"])
