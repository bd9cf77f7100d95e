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


@pytest.mark.parametrize("mode", ["fp4-qat/lowpreco", "fp4-qat/nofqp", "fp4-qat/naive-bf16-bwd"])
def test_ablation_variants_run(mode):
    cfg = T.TrainConfig(steps=3, seq_len=128, batch=4, d_model=128, n_heads=2, head_dim=64, attn_mode=mode)
    _, log = T.train(cfg)
    assert len(log.losses) == 3


def test_causal_d128_step():
    cfg = T.TrainConfig(steps=2, seq_len=256, batch=2, d_model=256, n_heads=2, head_dim=128, causal=True)
    layer, log = T.train(cfg)
    assert all(torch.isfinite(p).all() for p in layer.parameters())
