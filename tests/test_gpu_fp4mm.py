"""fp4mm on block-scaled tcgen05 MMAs (tensors.py:54-86) vs the oracle's
block-major FP4MM, plus the reference properties (test_tensors.py:86-131)."""

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu


def _qt(x):
    codes, scales = orc.quantize(x)
    return aq.QuantTensor(x.shape[0], x.shape[1], aq.NVFP4, codes, scales), codes, scales


# N >= 256 runs the 128 x 256 kernel (staged epilogue for K <= 8192, direct beyond)
@pytest.mark.parametrize("M,N,K", [(128, 128, 128), (37, 200, 48), (256, 384, 1024), (300, 129, 272), (1, 1, 16),
                                   (129, 700, 528), (260, 512, 256), (64, 256, 8448)])
def test_fp4mm_matches_oracle(M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    a = rng.standard_normal((M, K)) * 10.0 ** rng.uniform(-2, 2, (M, 1))
    b = rng.standard_normal((N, K))
    qa, ac, asc = _qt(a)
    qb, bc, bsc = _qt(b)
    got = aq.fp4mm(qa, qb)
    ref = orc.fp4mm(ac, asc, bc, bsc, K, width=64)
    assert got.shape == (M, N) and got.dtype == np.float32
    np.testing.assert_allclose(got, ref, rtol=2e-6, atol=1e-6 * np.abs(ref).max())


def test_fp4mm_torch_operands_and_quantizer():
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(512, 256, generator=g, device="cuda")
    b = torch.randn(640, 256, generator=g, device="cuda")
    qa, qb = aq.quantize(a), aq.quantize(b)
    c = aq.fp4mm(qa, qb)
    assert c.is_cuda
    deq = aq.dequantize(qa, torch.float32).double() @ aq.dequantize(qb, torch.float32).double().T
    assert orc.rel_l2(c.double().cpu().numpy(), deq.cpu().numpy()) <= 1e-6


def test_fp4mm_errors():
    qa, _, _ = _qt(np.ones((4, 32)))
    qb, _, _ = _qt(np.ones((4, 48)))
    with pytest.raises(aq.ShapeError):
        aq.fp4mm(qa, qb)
    with pytest.raises(aq.InvalidValue):
        aq.fp4mm(qa, qa, accum_width=64)
    with pytest.raises(aq.ShapeError):
        aq.fp4mm(qa, np.ones((4, 32)))


def test_matmul():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((3, 5, 7)), rng.standard_normal((7, 4))
    np.testing.assert_allclose(aq.matmul(a, b, 64), a @ b, rtol=1e-12, atol=1e-12)
    with pytest.raises(aq.ShapeError):
        aq.matmul(a, b[:3])


@pytest.mark.parametrize("M,N,K", [(128, 128, 128), (37, 200, 96), (256, 384, 1024), (300, 129, 288), (1, 1, 32),
                                   (129, 700, 544), (64, 256, 8448)])
def test_fp4mm_mxfp4_matches_dequantized_product(M, N, K):
    # MXFP4 QuantTensors (UE8M0 per 32, codec.py:123-166) on kind::mxf4 block32:
    # exact block products, fp32 accumulation
    rng = np.random.default_rng(M + 3 * N + K)
    a = torch.from_numpy(rng.standard_normal((M, K)) * 10.0 ** rng.uniform(-3, 3, (M, 1))).float().cuda()
    b = torch.from_numpy(rng.standard_normal((N, K))).float().cuda()
    qa, qb = aq.quantize(a, aq.MXFP4), aq.quantize(b, aq.MXFP4)
    c = aq.fp4mm(qa, qb)
    ref = aq.dequantize(qa, torch.float32).double() @ aq.dequantize(qb, torch.float32).double().T
    assert c.shape == (M, N)
    np.testing.assert_allclose(c.double().cpu().numpy(), ref.cpu().numpy(), rtol=2e-6,
                               atol=1e-6 * float(ref.abs().max()))
