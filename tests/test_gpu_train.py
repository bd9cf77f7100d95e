"""GPU QAT training driver: the toy associative-recall task
trains through the NVFP4 attention operator; ablation variants run."""

import numpy as np
import pytest
import torch

from paper_2603_00040_b200 import train as T

pytestmark = pytest.mark.gpu


def test_qat_training_reduces_loss():
    cfg = T.TrainConfig(steps=60, lr=3e-3, seq_len=128, batch=8, d_model=128, n_heads=2, head_dim=64)
    _, log = T.train(cfg)
    first, last = np.mean(log.losses[:5]), np.mean(log.losses[-5:])
    assert np.all(np.isfinite(log.losses))
    assert last < 0.8 * first


@pytest.mark.parametrize("mode", ["fp4-qat/lowpreco", "fp4-qat/nofqp", "fp4-qat/naive-bf16-bwd", "mxfp4-qat"])
def test_ablation_variants_run(mode):
    cfg = T.TrainConfig(steps=3, seq_len=128, batch=4, d_model=128, n_heads=2, head_dim=64, attn_mode=mode)
    _, log = T.train(cfg)
    assert len(log.losses) == 3


def test_causal_d128_step():
    cfg = T.TrainConfig(steps=2, seq_len=256, batch=2, d_model=256, n_heads=2, head_dim=128, causal=True)
    layer, log = T.train(cfg)
    assert all(torch.isfinite(p).all() for p in layer.parameters())


def test_evaluate_modes_and_fp4_paths_agree():
    # harness.py:326-344: "fp4" (inference kernel) and "fp4-fake" (training
    # forward) agree end to end -- here bit for bit
    cfg = T.TrainConfig(steps=5, lr=3e-3, seq_len=128, batch=8, d_model=128, n_heads=2, head_dim=64)
    layer, _ = T.train(cfg)
    X, t = T.make_task(123, 128, 128, 16)
    l_bf16 = T.evaluate(layer, X, t, "bf16")
    l_fp4 = T.evaluate(layer, X, t, "fp4")
    l_fake = T.evaluate(layer, X, t, "fp4-fake")
    assert l_fp4 == l_fake
    assert abs(l_fp4 - l_bf16) <= 0.2 * l_bf16
    assert T.random_prediction_baseline(t) > 0
    with pytest.raises(Exception):
        T.evaluate(layer, X, t, "fp8")


def test_qat_matmul_straight_through():
    # harness.py:356-369 against a CPU restatement with the oracle's fake quantizer
    from oracle import nvfp4_attn_oracle as orc
    g = np.random.default_rng(5)
    A = torch.from_numpy(g.standard_normal((32, 64))).bfloat16().double().numpy()
    B = torch.from_numpy(g.standard_normal((64, 48))).bfloat16().double().numpy()
    dC = g.standard_normal((32, 48))
    C = T.qat_matmul(A, B)
    want = orc.fake_quantize(A) @ orc.fake_quantize(B)
    np.testing.assert_allclose(C, want, rtol=1e-12, atol=1e-12)
    dA, dB = T.qat_matmul_backward(A, B, dC)
    np.testing.assert_allclose(dA, dC @ orc.fake_quantize(B).T, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dB, orc.fake_quantize(A).T @ dC, rtol=1e-12, atol=1e-12)
