"""quantized=False (plain attention, flash.py:195-200 / 344-349): the oracle is
pinned to the reference's own outputs (tests/golden/make_golden_plain.py), and
on the GPU the package's quantized=False path matches them."""

import os

import numpy as np
import pytest

from oracle import nvfp4_attn_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["p64", "p128c", "poffc"]


@pytest.fixture(scope="module")
def pl():
    return np.load(os.path.join(GOLD, "plain.npz"))


def _case(pl, name):
    n_q, n_k, d, causal = (int(x) for x in pl[f"{name}_meta"])
    return [pl[f"{name}_{k}"] for k in ("Q", "K", "V", "dO")] + [bool(causal)]


@pytest.mark.parametrize("name", CASES)
def test_oracle_plain_matches_reference(pl, name):
    Q, K, V, dO, causal = _case(pl, name)
    O, L, Op = orc.forward_training(Q, K, V, causal, width=64, quantized=False)
    np.testing.assert_allclose(O, pl[f"{name}_O"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(Op, pl[f"{name}_Op"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(L, pl[f"{name}_L"], rtol=0, atol=1e-12)
    dQ, dK, dV = orc.backward(Q, K, V, dO, O, L, Op, causal, width=64, quantized=False)
    for k, v in (("dQ", dQ), ("dK", dK), ("dV", dV)):
        np.testing.assert_allclose(v, pl[f"{name}_{k}"], rtol=0, atol=1e-11)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_plain_matches_reference(pl, name):
    import paper_2603_00040_b200 as aq
    Q, K, V, dO, causal = _case(pl, name)
    n_q, n_k = Q.shape[0], K.shape[0]
    cfg = aq.TileConfig(b_q=n_q, b_k=n_k, causal=causal)
    outs = aq.flash_forward_training(Q, K, V, cfg, quantized=False)
    assert orc.rel_l2(outs.O, pl[f"{name}_O"]) <= 2e-3
    assert orc.rel_l2(outs.O_prime, pl[f"{name}_Op"]) <= 2e-3
    assert np.max(np.abs(outs.L - pl[f"{name}_L"])) <= 2e-5
    for variant in (aq.BwdVariant.CORRECT, aq.BwdVariant.NAIVE_BF16_BWD):
        g = aq.flash_backward(Q, K, V, dO, outs, cfg, variant=variant, quantized=False)
        for k in ("dQ", "dK", "dV"):
            assert orc.rel_l2(getattr(g, k), pl[f"{name}_{k}"]) <= 1e-2, (k, variant)


@pytest.mark.gpu
def test_gpu_plain_autograd_and_training_mode():
    import torch

    import paper_2603_00040_b200 as aq
    from paper_2603_00040_b200 import train as T
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(2, 2, 256, 64, generator=g, device="cuda").bfloat16().requires_grad_() for _ in range(3))
    o = aq.attn_qat(q, k, v, causal=True, quantized=False)
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), is_causal=True)
    assert orc.rel_l2(o.float().detach().cpu().numpy(), ref.detach().cpu().numpy()) <= 1e-2
    o.sum().backward()
    assert all(t.grad is not None and torch.isfinite(t.grad).all() for t in (q, k, v))
    cfg = T.TrainConfig(steps=3, attn_mode="bf16", seq_len=128, batch=4)
    _, log = T.train(cfg)
    assert len(log.losses) == 3 and all(np.isfinite(log.losses))


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,causal", [(1024, 128, True), (640, 64, False), (300, 128, True)])
def test_gpu_plain_forward_is_native_and_matches_oracle(n, d, causal):
    # quantized=False at d = 64 / 128 runs the hand-written kernel (aq_attn_fwd_plain);
    # bf16 operands, fp32 accumulation: O within 1e-2 of the fp64 oracle, L within 1e-4
    import torch
    import paper_2603_00040_b200 as aq
    from paper_2603_00040_b200 import plain
    g = torch.Generator(device="cuda").manual_seed(n + d)
    q, k, v = (torch.randn(2, n, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    o, lse, o_hp, _ = aq.attn_forward(q, k, v, causal=causal, train=True, quantized=False)
    o_n, l_n = plain._plain_forward_b200(q, k, v, causal, torch.bfloat16)
    assert torch.equal(o, o_n) and torch.equal(lse, l_n) and torch.equal(o_hp, o)
    Q, K, V = (t[1].double().cpu().numpy() for t in (q, k, v))
    O, L, _ = orc.forward_training(Q, K, V, causal, width=64, quantized=False, ordered=False)
    assert orc.rel_l2(o[1].float().cpu().numpy(), O) <= 1e-2
    assert np.max(np.abs(lse[1].cpu().numpy() - L)) <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("n_q,n_k,d,causal", [(300, 300, 128, True), (640, 640, 64, False), (200, 264, 24, True),
                                              (128, 128, 16, False), (1024, 1024, 128, True)])
def test_gpu_plain_backward_native_matches_oracle(n_q, n_k, d, causal):
    """quantized=False backward on aq_attn_bwd_plain (K7 with a 16-bit S recompute,
    no library attention): dQ / dK / dV within 1e-2 of the fp64 oracle
    (flash.py:317-390 with quantized=False), ragged and padded head dims included."""
    import torch
    import paper_2603_00040_b200 as aq
    g = torch.Generator(device="cuda").manual_seed(n_q + d)
    q = torch.randn(2, n_q, d, generator=g, device="cuda").bfloat16()
    k, v = (torch.randn(2, n_k, d, generator=g, device="cuda").bfloat16() for _ in range(2))
    do = torch.randn(2, n_q, d, generator=g, device="cuda").bfloat16()
    o, lse, o_hp, _ = aq.attn_forward(q, k, v, causal=causal, train=True, quantized=False)
    dq, dk, dv = aq.attn_backward(q, k, v, do, o, o_hp, lse, causal=causal, quantized=False)
    for h in range(2):
        Q, K, V, dO = (t[h].double().cpu().numpy() for t in (q, k, v, do))
        O, L, Op = orc.forward_training(Q, K, V, causal, width=64, quantized=False, ordered=False)
        assert orc.rel_l2(o[h].float().cpu().numpy(), O) <= 1e-2
        dQ, dK, dV = orc.backward(Q, K, V, dO, O, L, Op, causal, width=64, quantized=False, ordered=False)
        for got, want, name in ((dq, dQ, "dQ"), (dk, dK, "dK"), (dv, dV, "dV")):
            e = orc.rel_l2(got[h].float().cpu().numpy(), want)
            assert e <= 1e-2, (name, h, e)


def test_plain_path_has_no_library_attention():
    """The quantized=False path is the package's own kernels (no flash_attn import)."""
    src = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2603_00040_b200", "plain.py")).read()
    assert "flash_attn" not in src and "scaled_dot_product_attention" not in src
