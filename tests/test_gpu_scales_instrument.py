"""ABI-3 boundary features on the GPU: per-tensor FP32 scales (two-level NVFP4,
north_star), the non-finite flag (codec.py:313-314), head dims below 64
(flash.py:185-188 accepts any d % 16 == 0) and the instrument records
(RowState / PTileRecord, flash.py:98-124)."""

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu


def _qkv(n=512, d=128, heads=2, seed=0, n_k=None, dt=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_k = n_k or n
    return (torch.randn(heads, n, d, generator=g, device="cuda").to(dt),
            torch.randn(heads, n_k, d, generator=g, device="cuda").to(dt),
            torch.randn(heads, n_k, d, generator=g, device="cuda").to(dt))


# ------------------------------------------------------------------ tensor scales

def test_quantize_tensor_scale_one_is_bitwise_reference():
    x = torch.randn(256, 128, device="cuda")
    a, b = aq.quantize(x), aq.quantize(x, tensor_scale=1.0)
    assert torch.equal(a.codes, b.codes) and torch.equal(a.scales, b.scales) and b.tensor_scale == 1.0


@pytest.mark.parametrize("ts", [0.37, 2.0 ** -7, "auto"])
def test_quantize_tensor_scale_matches_oracle(ts):
    x = torch.randn(256, 128, device="cuda") * 3.0
    qt = aq.quantize(x, tensor_scale=ts)
    t = qt.tensor_scale
    inv = np.float32(1.0) / np.float32(t)  # the kernel quantizes x * fl(1/t) in fp32
    xs = (x.cpu().numpy() * inv).astype(np.float32)
    codes, scales = orc.quantize(xs)
    assert np.array_equal(qt.codes.cpu().numpy(), codes) and np.array_equal(qt.scales.cpu().numpy(), scales)
    deq = aq.dequantize(qt, torch.float32).cpu().numpy()
    want = orc.dequantize(codes, scales, 128, np.float64) * t
    assert np.allclose(deq, want, rtol=1e-6, atol=0)
    fq = aq.fake_quantize(x, tensor_scale=t).cpu().numpy()
    assert np.allclose(fq, want, rtol=1e-6, atol=0)
    if ts == "auto":  # the largest block scale lands on E4M3's maximum
        assert int(qt.scales.max()) == 0x7E


@pytest.mark.parametrize("causal", [False, True])
def test_unit_scales_bitwise_reference(causal):
    q, k, v = _qkv()
    o0, l0, p0, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
    o1, l1, p1, _ = aq.attn_forward(q, k, v, causal=causal, train=True, q_scale=1.0, k_scale=1.0, v_scale=1.0,
                                    p_scale=1.0, softmax_scale=1.0 / np.sqrt(128))
    assert torch.equal(o0, o1) and torch.equal(l0, l1) and torch.equal(p0, p1)


@pytest.mark.parametrize("causal", [False, True])
def test_power_of_two_scales_are_exact(causal):
    """Power-of-two tensor scales move every block scale by an exact power of two
    (no E4M3 saturation or underflow here), so O, L, O', dQ, dK, dV are unchanged bit for bit."""
    q, k, v = _qkv(seed=2)
    do = torch.randn_like(q)
    sc = dict(q_scale=2.0 ** -3, k_scale=4.0, v_scale=0.5)
    o0, l0, p0, w0 = aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True)
    o1, l1, p1, w1 = aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True, **sc)
    assert torch.equal(o0, o1) and torch.equal(l0, l1) and torch.equal(p0, p1)
    g0 = aq.attn_backward(q, k, v, do, o0, p0, l0, causal=causal, fwd_workspace=w0)
    g1 = aq.attn_backward(q, k, v, do, o1, p1, l1, causal=causal, fwd_workspace=w1, **sc)
    for a, b in zip(g0, g1):
        assert torch.equal(a, b)


def test_auto_scales_match_oracle_rows():
    """Arbitrary (non power-of-two) tensor scales against the oracle's two-level restatement."""
    q, k, v = _qkv(n=1024, seed=4)
    q, k, v = q * 7.0, k * 0.01, v * 300.0
    ts = tuple(aq.auto_tensor_scale(t) for t in (q, k, v))
    o, lse, _, _ = aq.attn_forward(q, k, v, train=False, q_scale=ts[0], k_scale=ts[1], v_scale=ts[2])
    rows = np.arange(0, 1024, 7)
    Q, K, V = (t[1].double().cpu().numpy() for t in (q, k, v))
    want = orc.forward_rows(Q, K, V, rows, False, tensor_scales=ts)
    assert orc.rel_l2(o[1].float().cpu().numpy()[rows], want["O"]) <= 1e-2
    assert np.max(np.abs(lse[1].cpu().numpy()[rows] - want["L"])) <= 5e-5


def test_p_scale_keeps_long_row_mass():
    """At long N most 16-key P blocks fall under the reference's 2^-9 scale floor
    (SURVEY E4); a P tensor scale of 1/2688 keeps them, so O moves towards the
    unquantized-P output O' (non-parity mode, documented)."""
    q, k, v = _qkv(n=8192, seed=5, heads=2)
    o1, l1, op1, _ = aq.attn_forward(q, k, v, train=True)
    o2, l2, op2, _ = aq.attn_forward(q, k, v, train=True, p_scale=1.0 / 2688)
    assert torch.equal(l1, l2) and torch.equal(op1, op2)
    e1 = orc.rel_l2(o1.float().cpu().numpy(), op1.float().cpu().numpy())
    e2 = orc.rel_l2(o2.float().cpu().numpy(), op2.float().cpu().numpy())
    print(f"rel-L2(O, O') at N=8192: p_scale=1 {e1:.3f}, p_scale=1/2688 {e2:.3f}")
    assert e2 < 0.5 * e1
    rows = np.arange(0, 8192, 97)
    Q, K, V = (t[0].double().cpu().numpy() for t in (q, k, v))
    want = orc.forward_rows(Q, K, V, rows, False, training=True, p_scale=1.0 / 2688)
    assert orc.rel_l2(o2[0].float().cpu().numpy()[rows], want["O"]) <= 1e-2


def test_p_scale_backward_consistent():
    """dV uses the same two-level P^F as the forward: with one-hot dO rows dV reads P^F
    back (exact in fp32), which must match the forward's dumped P^F times t_p."""
    n = 256
    q, k, v = _qkv(n=n, d=64, heads=1, seed=6, dt=torch.float32)
    tp = 1.0 / 2688
    pf = aq.pf_buffers(1, n, n)
    o, lse, o_hp, ws = aq.attn_forward(q, k, v, train=True, keep_for_bwd=True, p_scale=tp, pf_out=pf)
    pfb = aq.pf_buffers(1, n, n)
    do = torch.zeros_like(q)
    do[0, :, 0] = 1.0
    _, _, dv = aq.attn_backward(q, k, v, do, o, o_hp, lse, fwd_workspace=ws, p_scale=tp, pf_out=pfb,
                                grad_dtype=torch.float32)
    assert torch.equal(pf[0], pfb[0]) and torch.equal(pf[1], pfb[1])
    codes, scales = pf[0][0].cpu().numpy(), pf[1][0].cpu().numpy()
    pf_vals = orc.dequantize(codes, scales, n, np.float64) * tp
    assert np.allclose(dv[0, :, 0].cpu().numpy(), pf_vals.sum(axis=0), rtol=1e-5, atol=1e-9)


# ------------------------------------------------------------------ non-finite input

@pytest.mark.parametrize("where", ["q", "k", "v"])
def test_nonfinite_batched_path_raises(where):
    q, k, v = _qkv(n=256, seed=7)
    t = {"q": q, "k": k, "v": v}[where]
    t[1, 100, 5] = float("nan") if where != "k" else float("inf")
    aq.check_nonfinite()  # clear
    aq.attn_forward(q, k, v, train=False)
    with pytest.raises(aq.InvalidValue):
        aq.check_nonfinite()
    aq.check_nonfinite()  # reset after raising
    with pytest.raises(aq.InvalidValue):
        aq.flash_forward_inference(q[1], k[1], v[1], aq.TileConfig(b_q=128, b_k=128))
    with pytest.raises(aq.InvalidValue):
        aq.attn_qat(q, k, v, check_finite=True)


# ------------------------------------------------------------------ head dims below 64

@pytest.mark.parametrize("n_q,n_k,d,causal", [(64, 64, 32, False), (32, 64, 16, True), (48, 48, 48, False),
                                              (200, 200, 96, True), (128, 96, 112, False)])
def test_small_head_dims_vs_oracle(n_q, n_k, d, causal):
    # fp32-valued operands: the GPU quantizes fp32, so float64 inputs would be
    # rounded before quantizing (one E2M1 midpoint straddle moves O by 1e-2 at N=64)
    Q, K, V = (x.astype(np.float32).astype(np.float64) for x in orc.make_qkv(11 + d, n_q, n_k, d))
    dO = orc.randn((n_q, d), 12 + d)
    cfg = aq.TileConfig(b_q=n_q, b_k=n_k, causal=causal)
    outs = aq.flash_forward_training(Q, K, V, cfg)
    g = aq.flash_backward(Q, K, V, dO, outs, cfg)
    O, L, Op = orc.forward_training(Q, K, V, causal, n_q, n_k, 32)
    dQ, dK, dV = orc.backward(Q, K, V, dO, O, L, Op, causal, n_q, n_k, 32)
    assert orc.rel_l2(outs.O, O) <= 1e-2 and orc.rel_l2(outs.O_prime, Op) <= 2e-3
    assert np.max(np.abs(outs.L - L)) <= 2e-5
    assert orc.rel_l2(g.dQ, dQ) <= 1e-2 and orc.rel_l2(g.dK, dK) <= 1e-2 and orc.rel_l2(g.dV, dV) <= 1e-2
    inf = aq.flash_forward_inference(Q, K, V, cfg)
    Oi, Li = orc.forward_inference(Q, K, V, causal, n_q, n_k, 32)
    assert orc.rel_l2(inf.O, Oi) <= 1e-2 and np.max(np.abs(inf.L - Li)) <= 2e-5


def test_reference_quantized_false_d24_shape():
    """test_flash.py:55-61: quantized=False at d = 24 (not a multiple of 16)."""
    Q, K, V = orc.make_qkv(2, 48, 48, 24)
    cfg = aq.TileConfig(b_q=16, b_k=16)
    outs = aq.flash_forward_training(Q, K, V, cfg, quantized=False)
    O, L, Op = orc.forward_training(Q, K, V, False, 16, 16, 32, quantized=False)
    # 16-bit tensor-core operands (plain.py): O and L carry fp16 operand rounding
    assert orc.rel_l2(outs.O, O) <= 2e-3 and np.max(np.abs(outs.L - L)) <= 1e-3


# ------------------------------------------------------------------ instrument records

def test_row_state_invariant():
    """test_flash.py:101-117: after each key tile, (m, l) equal the stats over the keys seen so far."""
    Q, K, V = orc.make_qkv(8, 32, 64, 16)
    cfg = aq.TileConfig(b_q=16, b_k=16)
    inst = []
    aq.flash_forward_training(Q, K, V, cfg, instrument=inst)
    S = orc.matmul(orc.fake_quantize(Q), orc.fake_quantize(K).T, 64) / np.sqrt(16)
    states = [r for r in inst if isinstance(r, aq.RowState)]
    assert len(states) == 2 * 4
    for snap in states:
        rows = slice(snap.i_tile * 16, (snap.i_tile + 1) * 16)
        seen = S[rows, : (snap.j_tile + 1) * 16]
        m_want = seen.max(axis=1)
        l_want = np.sum(np.exp(seen - m_want[:, None]), axis=1)
        np.testing.assert_allclose(snap.m, m_want, atol=1e-5)
        np.testing.assert_allclose(snap.l, l_want, rtol=1e-5)
        assert snap.to_json_dict()["kind"] == "row_state"


@pytest.mark.parametrize("causal", [False, True])
def test_recomputation_consistency(causal):
    """test_flash.py:230-244: the backward's requantized P equals the forward's, tile for tile
    (here bit for bit: the forward's and the backward's P^F dumps are byte-identical)."""
    Q, K, V = orc.make_qkv(53, 64, 64, 16)
    cfg = aq.TileConfig(b_q=16, b_k=16, causal=causal)
    fwd_inst, bwd_inst = [], []
    outs = aq.flash_forward_training(Q, K, V, cfg, instrument=fwd_inst)
    aq.flash_backward(Q, K, V, orc.randn((64, 16), 54), outs, cfg, instrument=bwd_inst)
    fwd = {(r.i_tile, r.j_tile): r.P_fq for r in fwd_inst if isinstance(r, aq.PTileRecord)}
    bwd = {(r.i_tile, r.j_tile): r.P_fq for r in bwd_inst if isinstance(r, aq.PTileRecord)}
    assert fwd and set(fwd) == set(bwd)
    assert all(r.phase == "backward" for r in bwd_inst)
    for key, p in fwd.items():
        assert np.array_equal(p, bwd[key])


def test_p_tiles_match_oracle():
    """The dumped P^F tiles against the oracle's fake_quantize_padded(P) (flash.py:232)."""
    Q, K, V = orc.make_qkv(3, 128, 256, 64)
    cfg = aq.TileConfig(b_q=64, b_k=128, causal=True)
    inst = []
    aq.flash_forward_training(Q, K, V, cfg, instrument=inst)
    tr = orc.oracle_forward(Q, K, V, causal=True)
    tiles = [r for r in inst if isinstance(r, aq.PTileRecord)]
    assert {(r.i_tile, r.j_tile) for r in tiles} == {(0, 0), (0, 1), (1, 0), (1, 1)}
    flips = 0
    for r in tiles:
        want = tr["P_fq"][r.i_tile * 64:(r.i_tile + 1) * 64, r.j_tile * 128:(r.j_tile + 1) * 128]
        flips += int(np.sum(r.P_fq != want))
    assert flips <= 2, flips
