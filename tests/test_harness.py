"""The reference toy harness (attnqat/harness.py) on the B200 path
(paper_2603_00040_b200/harness.py) against golden trajectories written by the
reference itself (tests/golden/make_golden_harness.py)."""

import os

import numpy as np
import pytest

from paper_2603_00040_b200 import harness as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def hg():
    return np.load(os.path.join(GOLD, "harness.npz"))


def test_task_and_init_are_the_references(hg):
    """Same pinned PCG64 stream: data and initial weights bit for bit (harness.py:62-76, 161-182)."""
    t = H.make_task(0, 16, 32, 8)
    np.testing.assert_array_equal(t.X, hg["task0_X"])
    np.testing.assert_array_equal(t.targets, hg["task0_targets"])
    np.testing.assert_array_equal(t.match_idx, hg["task0_match"])
    m = H.ToyModel.init(32, 32, 0)
    for k, v in m.params().items():
        np.testing.assert_array_equal(v, hg[f"init_{k}"])


def test_config_validation():
    bad = H.TrainConfig(steps=0, lr=0, seq_len=2, attn_mode="x", eval_mode="y", accum_width=16, head_dim=20)
    assert len(bad.validate()) >= 6
    assert H.TrainConfig().validate() == []


def test_adamw_matches_reference_update():
    """harness.py:251-276 on one parameter, written out."""
    p = {"w": np.array([1.0, -2.0])}
    opt = H.AdamW(p, lr=0.1, weight_decay=0.01)
    g = {"w": np.array([0.5, 0.25])}
    opt.step(g)
    m = 0.1 * g["w"]
    v = 0.001 * g["w"] ** 2
    want = np.array([1.0, -2.0]) * (1 - 0.1 * 0.01) - 0.1 * (m / 0.1) / (np.sqrt(v / 0.001) + 1e-8)
    np.testing.assert_allclose(p["w"], want, rtol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(4))
def test_step0_gradients_match_reference(hg, i):
    """loss_and_grads on the reference's first batch: the loss to 1e-4 and
    every gradient within 1e-2 rel-L2 (attention in fp32 / bf16-operand MMAs
    against the reference's float64)."""
    mode = str(hg["modes"][i])
    m = H.ToyModel.init(32, 32, 0)
    loss, grads = H.loss_and_grads(m, H.make_task(0, 16, 32, 8), mode)
    assert abs(loss - float(hg[f"m{i}_loss0"])) <= 1e-4 * abs(float(hg[f"m{i}_loss0"]))
    for k, g in grads.items():
        want = hg[f"m{i}_g0_{k}"]
        assert np.linalg.norm(g - want) <= 1e-2 * np.linalg.norm(want), (mode, k)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(4))
def test_training_trajectory_tracks_reference(hg, i):
    """30 steps at lr 1e-2 against the reference harness's own trajectory.
    The step-0 batch is bit-identical, the FP4 forward loss agrees to ~1e-15
    and the gradients to ~3e-3, after which training is chaotic in the FP4
    modes (a tiny weight difference flips E2M1 codes, so trajectories fan
    out): the first steps must agree closely, the rest and the final model's
    eval losses only within the spread that chaos produces (measured: bf16
    mode <= 2 % over 30 steps; FP4 modes <= 1 % for 3 steps, <= 17 % after)."""
    mode = str(hg["modes"][i])
    cfg = H.TrainConfig(steps=30, lr=1e-2, seed=0, attn_mode=mode)
    m, log = H.train(H.ToyModel.init(cfg.d_model, cfg.head_dim, cfg.seed), cfg)
    L, G = np.array(log.losses), np.array(log.grad_norms)
    wl, wg = hg[f"m{i}_losses"], hg[f"m{i}_gnorms"]
    head = 20 if mode == "bf16" else 3
    np.testing.assert_allclose(L[:head], wl[:head], rtol=2e-2)
    np.testing.assert_allclose(G[:head], wg[:head], rtol=2e-2)
    assert np.max(np.abs(L - wl) / wl) <= 0.3, (mode, L, wl)
    ev = H.eval_batch(cfg)
    got = np.array([H.evaluate(m, ev, e) for e in ("bf16", "fp4", "fp4-fake")])
    assert got[1] == got[2]  # real-quant inference == fake-quant training forward (acceptance 9)
    np.testing.assert_allclose(got, hg[f"m{i}_eval"], rtol=0.1)
