"""Element-wise code rounding (round_to_fp4 / round_to_e4m3, codec.py:63-112) and
single-block helpers (codec.py:225-258) on the GPU vs the pinned oracle,
including float64 inputs one ulp either side of every rounding midpoint (no
double rounding through float32)."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _around(points):
    pts = np.asarray(points, dtype=np.float64)
    return np.concatenate([pts, np.nextafter(pts, -np.inf), np.nextafter(pts, np.inf), pts + 1e-12, pts - 1e-12])


def test_round_to_fp4_matches_oracle():
    codec = np.load(os.path.join(GOLD, "codec.npz"))
    mids = [0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0]
    rng = np.random.default_rng(0)
    x = np.concatenate([codec["adv_x"].reshape(-1), rng.standard_normal(4096) * 3, _around(mids), -_around(mids),
                        [0.0, -0.0, -1e-30, 1e-30, 6.0, 7.0, -6.5, 1e30, -1e30]])
    got = aq.round_to_fp4(x)
    np.testing.assert_array_equal(got, orc.round_to_fp4(x))
    # float32 torch input on the device
    x32 = torch.from_numpy(x.astype(np.float32)).cuda()
    np.testing.assert_array_equal(aq.round_to_fp4(x32).cpu().numpy(), orc.round_to_fp4(x.astype(np.float32)))
    assert aq.round_to_fp4(-0.0) == 0 and aq.round_to_fp4(-0.1) == 0x8 and aq.round_to_fp4(0.25) == 0


def test_round_to_e4m3_matches_oracle():
    vals = orc.E4M3_VALUES[:127].astype(np.float64)
    mids = (vals[:-1] + vals[1:]) / 2
    rng = np.random.default_rng(1)
    x = np.concatenate([np.abs(rng.standard_normal(4096)) * 10.0 ** rng.integers(-4, 3, 4096), _around(mids),
                        _around(vals), [0.0, 448.0, 464.0, 1e6, 2.0 ** -10, 2.0 ** -11]])
    x = x[x >= 0]
    np.testing.assert_array_equal(aq.round_to_e4m3(x), orc.round_to_e4m3(x))


def test_invalid_inputs_raise():
    for bad in ([np.inf], [np.nan, 1.0]):
        with pytest.raises(aq.InvalidValue):
            aq.round_to_fp4(np.array(bad))
    with pytest.raises(aq.InvalidValue):
        aq.round_to_e4m3(np.array([1.0, -0.5]))


def test_quantize_dequantize_block():
    rng = np.random.default_rng(2)
    for _ in range(20):
        x = rng.standard_normal(16) * 10.0 ** rng.integers(-3, 3)
        blk = aq.quantize_block(x)
        codes, scales = orc.quantize(x.astype(np.float32).astype(np.float64)[None, :])
        assert blk.codes == codes.tobytes() and blk.scale == int(scales[0, 0])
        np.testing.assert_array_equal(aq.dequantize_block(blk), orc.dequantize(codes, scales, 16, np.float64)[0])
    with pytest.raises(aq.ShapeError):
        aq.quantize_block(np.zeros(8))


@pytest.mark.parametrize("n,d", [(256, 128), (384, 64), (32760, 128)])
def test_staged_tiles_identical_across_input_paths(n, d):
    # the bf16 fast paths of the tile quantizers (K1 / K2) and the general
    # kernels (taken for fp32 / fp16 inputs) write the same bytes for the same values
    import torch
    g = torch.Generator(device="cuda").manual_seed(n + d)
    q, k, v = (torch.randn(2, n, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    outs = []
    from paper_2603_00040_b200 import _lib
    nbytes = _lib.load().aq_attn_fwd_workspace_bytes(2, n, n, d, 0, 0)
    for dt in (torch.bfloat16, torch.float32, torch.float16):
        # zeroed: bytes no MMA reads (e.g. scale rows past d of a V^T image) stay equal
        ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        aq.attn_forward(q.to(dt), k.to(dt), v.to(dt), causal=True, train=False, workspace=ws)
        outs.append(ws)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
