"""MXFP4 codec (BlockSpec(32, E8M0), codec.py:123-203) on the GPU against golden
vectors written by the reference itself (tests/golden/make_golden_mx.py)."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def mx():
    return np.load(os.path.join(GOLD, "mxfp4.npz"))


def test_quantize_bytes_match_reference(mx):
    qt = aq.quantize(mx["x"], aq.MXFP4)
    assert qt.spec == aq.MXFP4 and qt.block_grid == (mx["x"].shape[0], 2)
    np.testing.assert_array_equal(qt.codes, mx["codes"])
    np.testing.assert_array_equal(qt.scales, mx["scales"])


def test_fake_quantize_and_dequantize_match_reference(mx):
    np.testing.assert_array_equal(aq.fake_quantize(mx["x"], aq.MXFP4), mx["fq"])
    qt = aq.QuantTensor(mx["x"].shape[0], 64, aq.MXFP4, mx["codes"], mx["scales"])
    np.testing.assert_array_equal(aq.dequantize(qt, np.float64), mx["fq"])
    np.testing.assert_array_equal(aq.fake_quantize_cols(mx["v"], aq.MXFP4), mx["fqc"])


def test_round_to_e8m0_matches_reference(mx):
    np.testing.assert_array_equal(aq.round_to_e8m0(mx["e8_x"]), mx["e8_codes"])
    assert aq.decode_e8m0(aq.round_to_e8m0(3.0)) == 4.0   # tie -> up (test_codec.py:159-162)
    assert aq.decode_e8m0(aq.round_to_e8m0(2.9)) == 2.0
    for code in range(255):
        assert int(aq.round_to_e8m0(2.0 ** (code - 127))) == code
    with pytest.raises(aq.InvalidValue):
        aq.round_to_e8m0(np.array([1.0, 0.0]))
    with pytest.raises(aq.InvalidValue):
        aq.decode_e8m0(np.uint8(0xFF))


def test_mxfp4_block_and_torch_path(mx):
    b = aq.quantize_block(mx["x"][0, :32], aq.MXFP4)
    np.testing.assert_array_equal(aq.dequantize_block(b), mx["fq"][0, :32])
    t = torch.from_numpy(mx["x"]).float().cuda()
    qt = aq.quantize(t, aq.MXFP4)
    assert torch.equal(qt.codes.cpu(), torch.from_numpy(mx["codes"]))
    with pytest.raises(aq.ShapeError):
        aq.quantize(np.zeros((2, 48)), aq.MXFP4)
