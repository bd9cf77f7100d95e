"""Desk-scale QAT acceptance on the B200 (SPEC acceptance 7-9 analogues,
/root/reference/SPEC.md:564-566; harness.py:294-344).

The reference harness's toy config (harness.py:93-107: seq_len 16, d_model
32, head_dim 32, one head, batch 8, 400 steps) trained through this package's
autograd attention. The assertions are the ones the reference harness itself
satisfies at the same learning rate (profiles/r02_qat_acceptance_reference.txt;
the GPU runs are in profiles/r02_qat_acceptance_gpu.json):

* acceptance 8a at lr 3e-2: the LOW_PREC_O backward (D from O instead of O')
  drives the max gradient norm >= 10x the CORRECT run's (reference 17x,
  GPU 16-46x over seeds 0-2), or diverges;
* at lr 1e-2: LOW_PREC_O does not learn (final loss >= 5x CORRECT's; reference
  8.6x) while the other variants do;
* acceptance 8b at lr 1e-3: NO_FAKE_QUANT_P has a strictly larger grad-norm
  variance than CORRECT (reference 11.18 vs 10.69; at 1e-2 the margin is a few
  percent either way on both sides, at 3e-2 it reverses for the reference);
* acceptance 9 (second half): the FP4 training forward and the real-quant
  inference forward give the same eval loss (here bit for bit: K4 == K5).

Acceptance 7 (QAT recovery >= 50 %) is not asserted: the reference harness
does not reach it either at any learning rate tried (1e-3 ... 3e-2, up to 2000
steps: its FP4-QAT model's FP4-eval loss is 0.054 vs 0.055 for the bf16-trained
model at lr 3e-3 x 2000 steps); what is checked is that the bf16-trained model
degrades under FP4 evaluation and the QAT model stays within 2x of its own
unquantized loss.
"""

import numpy as np
import pytest
import torch

from paper_2603_00040_b200 import train as T
from paper_2603_00040_b200.errors import StabilityError

pytestmark = pytest.mark.gpu
EVAL_SEED_OFFSET = 999_983  # harness.py:287


def _run(mode, seed, lr, steps=400):
    cfg = T.TrainConfig(steps=steps, lr=lr, seed=seed, seq_len=16, batch=8, d_model=32, n_heads=1, head_dim=32,
                        attn_mode=mode, compute_dtype="fp32")
    try:
        layer, log = T.train(cfg)
    except StabilityError as e:
        return {"diverged": True, "step": e.step}
    X, Y = T.make_task(seed * 1_000_003 + EVAL_SEED_OFFSET, cfg.seq_len, cfg.d_model, 64)
    return {"diverged": False, "final": float(np.mean(log.losses[-20:])), "max_g": max(log.grad_norms),
            "var_g": float(np.var(log.grad_norms)),
            "fp4": T.evaluate(layer, X, Y, "fp4", dtype=torch.float32),
            "fp4_fake": T.evaluate(layer, X, Y, "fp4-fake", dtype=torch.float32),
            "bf16": T.evaluate(layer, X, Y, "bf16", dtype=torch.float32)}


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_low_prec_o_gradient_blowup(seed):
    good = _run("fp4-qat", seed, 3e-2)
    bad = _run("fp4-qat/lowpreco", seed, 3e-2)
    assert not good["diverged"]
    assert bad["diverged"] or bad["max_g"] >= 10.0 * good["max_g"], (good, bad)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_variants_at_lr_1e2(seed):
    good = _run("fp4-qat", seed, 1e-2)
    low = _run("fp4-qat/lowpreco", seed, 1e-2)
    bf16 = _run("bf16", seed, 1e-2)
    base = float(np.mean(T.make_task(seed * 1_000_003 + EVAL_SEED_OFFSET, 16, 32, 64)[1] ** 2))
    # CORRECT learns (well below the predict-zero baseline); LOW_PREC_O does not
    assert good["final"] < 0.1 * base and low["final"] >= 5.0 * good["final"], (good, low)
    # acceptance 9: fake-quant training forward == real-quant inference forward
    for r in (good, low, bf16):
        assert r["fp4"] == r["fp4_fake"]
    # the bf16-trained model loses accuracy under FP4 evaluation; the QAT model
    # stays within 2x of its own unquantized loss
    assert bf16["fp4"] > 1.2 * bf16["bf16"], bf16
    assert good["fp4"] <= 2.0 * good["bf16"], good


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_no_fake_quant_p_noisier_gradients(seed):
    """Acceptance 8b at lr 1e-3: not fake-quantizing P in dV raises the
    grad-norm variance over the run (GPU: 5.44 / 6.60 / 5.39 vs CORRECT 5.31 /
    6.35 / 5.22; reference seed 0: 11.18 vs 10.69)."""
    good = _run("fp4-qat", seed, 1e-3)
    nofqp = _run("fp4-qat/nofqp", seed, 1e-3)
    assert nofqp["var_g"] > good["var_g"], (good, nofqp)
