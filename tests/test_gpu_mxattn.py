"""MXFP4 inference forward (flash_forward_inference with cfg.spec = MXFP4) on
tcgen05.mma.kind::mxf4 vs the reference's own outputs (tests/golden/make_golden_mxattn.py)."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def mx():
    return np.load(os.path.join(GOLD, "mxattn.npz"))


@pytest.mark.parametrize("name", ["m64", "m128c", "mrag"])
def test_mx_inference_matches_reference(mx, name):
    # as for NVFP4 (test_gpu_forward.py): O rel-L2 <= 1e-2 (fp32 tensor-core vs
    # fixed-order accumulation can flip a P code at a midpoint), L <= 2e-5
    n_q, n_k, d, causal, b_q, b_k = (int(x) for x in mx[f"{name}_meta"])
    cfg = aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal), spec=aq.MXFP4)
    outs = aq.flash_forward_inference(mx[f"{name}_Q"], mx[f"{name}_K"], mx[f"{name}_V"], cfg)
    assert outs.O_prime is None
    assert orc.rel_l2(outs.O, mx[f"{name}_O"]) <= 1e-2, orc.rel_l2(outs.O, mx[f"{name}_O"])
    assert np.max(np.abs(outs.L - mx[f"{name}_L"])) <= 2e-5


@pytest.mark.parametrize("name", ["m64", "m128c", "mrag"])
def test_mx_training_forward_matches_reference(mx, name):
    # O, L as the inference forward; O' = P V^F (fp16 P^ in the f16 MMA): <= 2e-3
    n_q, n_k, d, causal, b_q, b_k = (int(x) for x in mx[f"{name}_meta"])
    cfg = aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal), spec=aq.MXFP4)
    outs = aq.flash_forward_training(mx[f"{name}_Q"], mx[f"{name}_K"], mx[f"{name}_V"], cfg)
    assert orc.rel_l2(outs.O, mx[f"{name}_Otr"]) <= 1e-2
    assert orc.rel_l2(outs.O_prime, mx[f"{name}_Op"]) <= 2e-3
    assert np.max(np.abs(outs.L - mx[f"{name}_Ltr"])) <= 2e-5
    inf = aq.flash_forward_inference(mx[f"{name}_Q"], mx[f"{name}_K"], mx[f"{name}_V"], cfg)
    np.testing.assert_array_equal(outs.O, inf.O)   # same MMAs, same P codes


@pytest.mark.parametrize("name", ["m64", "m128c", "mrag"])
def test_mx_backward_matches_reference(mx, name):
    # as for NVFP4 (test_gpu_backward.py): bf16 operands in the 16-bit MMAs -> 1e-2
    n_q, n_k, d, causal, b_q, b_k = (int(x) for x in mx[f"{name}_meta"])
    cfg = aq.TileConfig(b_q=b_q, b_k=b_k, causal=bool(causal), spec=aq.MXFP4)
    Q, K, V, dO = (mx[f"{name}_{t}"] for t in ("Q", "K", "V", "dO"))
    outs = aq.flash_forward_training(Q, K, V, cfg)
    g = aq.flash_backward(Q, K, V, dO, outs, cfg)
    for t in ("dQ", "dK", "dV"):
        assert orc.rel_l2(getattr(g, t), mx[f"{name}_{t}"]) <= 1e-2, (t, orc.rel_l2(getattr(g, t), mx[f"{name}_{t}"]))


def test_mx_autograd_matches_functional():
    g = torch.Generator(device="cuda").manual_seed(21)
    q, k, v = (torch.randn(2, 2, 256, 64, generator=g, device="cuda").bfloat16().requires_grad_() for _ in range(3))
    o = aq.attn_qat(q, k, v, causal=True, spec=aq.MXFP4)
    d_o = torch.randn_like(o)
    o.backward(d_o)
    o2, lse, o_hp = aq.attn_forward_mx(q.detach(), k.detach(), v.detach(), causal=True, train=True)
    dq, dk, dv = aq.attn_backward(q.detach(), k.detach(), v.detach(), d_o, o2, o_hp, lse, causal=True, mx=True)
    assert torch.equal(o, o2)
    assert torch.equal(q.grad, dq) and torch.equal(k.grad, dk) and torch.equal(v.grad, dv)


@pytest.mark.parametrize("shape,d,causal", [((2, 5, 1100), 128, True), ((1, 3, 700), 64, True),
                                             ((2, 3, 900), 128, False)])
def test_mx_split_pass_training_forward_matches_k4(shape, d, causal, monkeypatch):
    """The MXFP4 training forward runs on the split-pass kernel K11's MX instance;
    K4's MX instance (AQ_FWD_QAT=0) has the same arithmetic: O, O' and L agree bit
    for bit (ragged tails, d = 64, the dynamic item queue from 8 causal query tiles)."""
    g = torch.Generator(device="cuda").manual_seed(33)
    q, k, v = (torch.randn(*shape, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    o11, l11, ohp11 = aq.attn_forward_mx(q, k, v, causal=causal, train=True)
    monkeypatch.setenv("AQ_FWD_QAT", "0")
    o4, l4, ohp4 = aq.attn_forward_mx(q, k, v, causal=causal, train=True)
    assert torch.equal(o11, o4) and torch.equal(l11, l4) and torch.equal(ohp11, ohp4)
