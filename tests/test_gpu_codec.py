"""GPU NVFP4 quantizers vs the reference golden vectors: bytes must be identical."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def codec():
    return np.load(os.path.join(GOLD, "codec.npz"))


@pytest.mark.parametrize("name", ["randn", "wide", "adv", "f32"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_quantize_rows_bytes(codec, name, dtype):
    x = codec[f"{name}_x"]
    t = torch.from_numpy(x.astype(np.float32)).to(dtype)
    if not torch.equal(t.float().double(), torch.from_numpy(x)):
        pytest.skip("input not representable in this dtype")
    qt = aq.quantize(t.cuda())
    np.testing.assert_array_equal(qt.codes.cpu().numpy(), codec[f"{name}_codes"])
    np.testing.assert_array_equal(qt.scales.cpu().numpy(), codec[f"{name}_scales"])
    fq = aq.fake_quantize(t.cuda().float())
    np.testing.assert_array_equal(fq.cpu().numpy().astype(np.float64), codec[f"{name}_fq"])


def test_quantize_numpy_roundtrip(codec):
    qt = aq.quantize(codec["randn_x"])
    assert isinstance(qt.codes, np.ndarray)
    np.testing.assert_array_equal(qt.codes, codec["randn_codes"])
    deq = aq.dequantize(qt)
    np.testing.assert_array_equal(deq, codec["randn_fq"].astype(np.float32))


def test_quantize_cols_padded(codec):
    v = codec["vcols_x"]
    qt = aq.quantize_cols(torch.from_numpy(v.astype(np.float32)).cuda())
    np.testing.assert_array_equal(qt.codes.cpu().numpy(), codec["vcols_codes"])
    np.testing.assert_array_equal(qt.scales.cpu().numpy(), codec["vcols_scales"])
    fq = aq.fake_quantize_cols(torch.from_numpy(v.astype(np.float32)).cuda())
    np.testing.assert_array_equal(fq.cpu().numpy().astype(np.float64), codec["vcols_fq"])


def test_random_large_vs_oracle():
    g = torch.Generator().manual_seed(11)
    x = (torch.randn(4096, 128, generator=g) * torch.exp(torch.randn(4096, 1, generator=g) * 3)).to(torch.bfloat16)
    qt = aq.quantize(x.cuda())
    c, s = orc.quantize(x.double().numpy())
    np.testing.assert_array_equal(qt.codes.cpu().numpy(), c)
    np.testing.assert_array_equal(qt.scales.cpu().numpy(), s)


def test_negative_zero_and_bump():
    x = torch.zeros(2, 16)
    x[0, 0], x[0, 1], x[0, 2] = 6.0, -0.1, -0.0
    x[1] = torch.linspace(-1e-6, 1e-6, 16)
    qt = aq.quantize(x.cuda())
    codes = qt.codes.cpu().numpy()
    assert codes[0, 0] == 0x87 and codes[0, 1] == 0x00
    assert qt.scales.cpu().numpy()[1, 0] == 1  # tiny block keeps 2^-9


def test_nonfinite_raises():
    x = torch.zeros(1, 16)
    x[0, 3] = float("nan")
    with pytest.raises(aq.InvalidValue):
        aq.quantize(x.cuda())


def test_shape_errors():
    with pytest.raises(aq.ShapeError):
        aq.quantize(torch.zeros(4, 12).cuda())
    with pytest.raises(aq.ShapeError):
        aq.quantize(torch.zeros(16).cuda())


def test_quantize_cols_c3_ragged_tail_vs_oracle():
    """C3's N = 32760 (not a multiple of 16): V^T blocked along tokens with the
    zero-padded tail (quantize_padded(V.T), codec.py:359-361, flash.py:267),
    byte-identical to the oracle for a full C3 head."""
    g = torch.Generator().manual_seed(3)
    v = torch.randn(32760, 128, generator=g).to(torch.bfloat16)
    qt = aq.quantize_cols(v.cuda())
    c, s = orc.quantize_padded(v.double().numpy().T)
    assert qt.codes.shape[-1] * 2 == 32768
    np.testing.assert_array_equal(qt.codes.cpu().numpy(), c)
    np.testing.assert_array_equal(qt.scales.cpu().numpy(), s)
