"""Parity at the benchmarked shapes (SURVEY §8(c) "Large configs").

The BASELINE configs run here at full size on the GPU; the CPU oracle checks
sampled heads and query rows (``forward_rows``: each query row depends only on
its own row of S, with the reference's single-key-tile semantics that C3's
N = 32760 forces, flash.py:63-71), the full backward at C4's N = 4096 and the
dQ of sampled rows at N = 64K (``backward_rows_dq``). The kernels' P^F dump
(the ``instrument`` path, flash.py:117-124) is compared code for code with the
oracle's quantize_padded(P); the flip counts are printed (run with -s) and
bounded.

Tolerances as everywhere else: O rel-L2 <= 1e-2, O' <= 2e-3, L <= 2e-5 abs,
dQ / dK / dV <= 1e-2.
"""

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
TOL_O, TOL_OP, TOL_L, TOL_G = 1e-2, 2e-3, 2e-5, 1e-2


def _inputs(B, H, N, d=128, seed=0, grad=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    ts = [torch.randn(B, H, N, d, generator=g, device="cuda").bfloat16() for _ in range(4 if grad else 3)]
    return ts


def _rows(n, seed=0):
    """First / middle / last 64 query rows (incl. the ragged tail) + 64 random ones."""
    r = np.random.default_rng(seed).choice(n, 64, replace=False)
    mid = n // 2 - 32
    return np.unique(np.r_[0:64, mid:mid + 64, n - 64:n, r])


def _head(t, h):
    return t.reshape(-1, t.shape[-2], t.shape[-1])[h].double().cpu().numpy()


def _flips(pf, want_c, want_s, rows, n_k):
    """(code flips, scale flips, codes compared) between the GPU dump rows and the oracle."""
    n16 = -(-n_k // 16) * 16
    gc = pf[0].reshape(-1, n16 // 2)[rows].cpu().numpy()
    gs = pf[1].reshape(-1, n16 // 16)[rows].cpu().numpy()
    gcn = orc.unpack(gc, n16)
    wcn = orc.unpack(want_c, n16)
    return int(np.sum(gcn != wcn)), int(np.sum(gs != want_s)), gcn.size


def _check_forward(q, k, v, causal, heads, tag, training=False, max_flip_frac=1e-4):
    B, H, N, d = q.shape
    if training:
        o, lse, o_hp, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
    else:
        o, lse, _, _ = aq.attn_forward(q, k, v, causal=causal, train=False)
    o3, l2 = o.reshape(-1, N, d), lse.reshape(-1, N)
    rows = _rows(N)
    for h in heads:
        Q, K, V = _head(q, h), _head(k, h), _head(v, h)
        want = orc.forward_rows(Q, K, V, rows, causal, training=training)
        got_o = o3[h].float().cpu().numpy()[rows]
        got_l = l2[h].cpu().numpy()[rows]
        e_o = orc.rel_l2(got_o, want["O"])
        e_l = float(np.max(np.abs(got_l - want["L"])))
        msg = f"{tag} head {h}: O {e_o:.2e} L {e_l:.2e}"
        if training:
            e_op = orc.rel_l2(o_hp.reshape(-1, N, d)[h].float().cpu().numpy()[rows], want["O_prime"])
            msg += f" O' {e_op:.2e}"
            assert e_op <= TOL_OP, msg
        # P^F of this head from the kernel's dump, from a one-head launch (bitwise the same
        # head as in the full-size run: heads are independent and the kernels deterministic)
        sl = (slice(h // H, h // H + 1), slice(h % H, h % H + 1))
        pf = aq.pf_buffers(1, N, N)
        o1, _, _, _ = aq.attn_forward(q[sl], k[sl], v[sl], causal=causal, train=training, pf_out=pf)
        assert torch.equal(o1.reshape(N, d), o3[h]), f"{tag}: one-head run differs from the full run"
        fc, fs, n_codes = _flips(pf, want["P_codes"], want["P_scales"], rows, N)
        msg += f" P^F code flips {fc}/{n_codes} scale flips {fs}"
        print(msg)
        assert e_o <= TOL_O and e_l <= TOL_L, msg
        assert fc <= max_flip_frac * n_codes and fs <= max_flip_frac * n_codes / 16, msg


def test_c2_llama_causal_inference_and_training():
    """C2: B4 H32 N8192 d128 causal (the bench headline shape)."""
    q, k, v = _inputs(4, 32, 8192)
    _check_forward(q, k, v, True, heads=(0, 77), tag="C2 infer")
    _check_forward(q, k, v, True, heads=(127,), tag="C2 train", training=True)


def test_c3_wan_noncausal_ragged():
    """C3: B1 H40 N32760 d128 non-causal; 16 does not divide N (single key tile in the reference)."""
    q, k, v = _inputs(1, 40, 32760)
    _check_forward(q, k, v, False, heads=(0, 39), tag="C3 infer")


def test_c3_early_out_is_exact():
    """The K5 pass-2 early-out (P blocks below 2^-11) skips most blocks at C3: K4, which
    never skips, must give the same O bit for bit."""
    q, k, v = (t[:, :4] for t in _inputs(1, 40, 32760, seed=3))
    o_t, l_t, _, _ = aq.attn_forward(q, k, v, train=True)
    o_i, l_i, _, _ = aq.attn_forward(q, k, v, train=False)
    assert torch.equal(o_t, o_i) and torch.equal(l_t, l_i)


@pytest.mark.parametrize("shape", [(8, 32, 4096), (1, 3, 32768)])
def test_dynamic_item_queue_covers_every_item(shape, monkeypatch):
    """Causal rows of >= 8 query tiles run the training forward (K11) on the
    dynamic item queue: every (head, query tile) must be computed exactly once, so
    O / O' / L equal the static schedule's bit for bit, and equal the inference
    kernel's (K5, static order) O and L."""
    q, k, v = _inputs(*shape, seed=5)
    o_d, l_d, ohp_d, _ = aq.attn_forward(q, k, v, causal=True, train=True)
    oi_d, li_d, _, _ = aq.attn_forward(q, k, v, causal=True, train=False)
    monkeypatch.setenv("AQ_FWD_DYN", "0")
    monkeypatch.setenv("AQ_FWDI_DYN", "0")
    o_s, l_s, ohp_s, _ = aq.attn_forward(q, k, v, causal=True, train=True)
    oi_s, li_s, _, _ = aq.attn_forward(q, k, v, causal=True, train=False)
    assert torch.equal(o_d, o_s) and torch.equal(l_d, l_s) and torch.equal(ohp_d, ohp_s)
    assert torch.equal(oi_d, oi_s) and torch.equal(li_d, li_s)
    assert torch.equal(o_d, oi_d) and torch.equal(l_d, li_d)


@pytest.mark.parametrize("shape,d,causal", [((8, 32, 4096), 128, True), ((2, 5, 1100), 128, True),
                                             ((1, 7, 3000), 64, True), ((2, 3, 2100), 128, False),
                                             ((1, 4, 1000), 64, False)])
def test_split_pass_training_forward_matches_k4(shape, d, causal, monkeypatch):
    """The training forward runs on the split-pass kernel K11 (attn_fwd_qat.cu); K4
    (AQ_FWD_QAT=0) is the single-stream kernel with the same arithmetic: O, O' and
    L must agree bit for bit (ragged tails, d = 64, both item orders)."""
    q, k, v = _inputs(*shape, d=d, seed=7)
    o10, l10, ohp10, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
    monkeypatch.setenv("AQ_FWD_QAT", "0")
    o4, l4, ohp4, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
    assert torch.equal(o10, o4) and torch.equal(l10, l4) and torch.equal(ohp10, ohp4)


@pytest.mark.parametrize("causal", [True, False])
def test_c4_training_fwd_bwd_full_heads(causal):
    """C4: B8 H32 N4096 d128, fwd + bwd through the autograd Function; two heads
    against the full tiled oracle (flash.py:176-246, 317-390)."""
    q, k, v, do = _inputs(8, 32, 4096, grad=True)
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, k, v))
    o = aq.attn_qat(qg, kg, vg, causal=causal)
    o.backward(do)
    o_f, lse, o_hp, _ = aq.attn_forward(q, k, v, causal=causal, train=True)
    assert torch.equal(o_f, o)
    for h in (0, 255):
        Q, K, V, dO = (_head(t, h) for t in (q, k, v, do))
        O, L, Op = orc.forward_training(Q, K, V, causal, 128, 128, 32, ordered=False)
        dQ, dK, dV = orc.backward(Q, K, V, dO, O, L, Op, causal, 128, 128, 32, ordered=False)
        errs = {"O": orc.rel_l2(_head(o.detach(), h), O), "O'": orc.rel_l2(_head(o_hp, h), Op),
                "L": float(np.max(np.abs(lse.reshape(-1, 4096)[h].cpu().numpy() - L))),
                "dQ": orc.rel_l2(_head(qg.grad, h), dQ), "dK": orc.rel_l2(_head(kg.grad, h), dK),
                "dV": orc.rel_l2(_head(vg.grad, h), dV)}
        print(f"C4 causal={causal} head {h}:", {k_: f"{v_:.2e}" for k_, v_ in errs.items()})
        lim = {"O": TOL_O, "O'": TOL_OP, "L": TOL_L, "dQ": TOL_G, "dK": TOL_G, "dV": TOL_G}
        assert all(errs[k_] <= lim[k_] for k_ in lim), errs


@pytest.mark.parametrize("causal", [True, False])
def test_c5_sweep_1k_full(causal):
    """C5 low end: N = 1K, B = 64, H = 32 (64K tokens x 32 heads), fwd + bwd, two heads in full."""
    q, k, v, do = _inputs(64, 32, 1024, grad=True)
    o, lse, o_hp, ws = aq.attn_forward(q, k, v, causal=causal, train=True, keep_for_bwd=True)
    dq, dk, dv = aq.attn_backward(q, k, v, do, o, o_hp, lse, causal=causal, fwd_workspace=ws)
    for h in (5, 2047):
        Q, K, V, dO = (_head(t, h) for t in (q, k, v, do))
        O, L, Op = orc.forward_training(Q, K, V, causal, 128, 128, 32, ordered=False)
        dQ, dK, dV = orc.backward(Q, K, V, dO, O, L, Op, causal, 128, 128, 32, ordered=False)
        assert orc.rel_l2(_head(o, h), O) <= TOL_O
        assert orc.rel_l2(_head(o_hp, h), Op) <= TOL_OP
        assert np.max(np.abs(lse.reshape(-1, 1024)[h].cpu().numpy() - L)) <= TOL_L
        for got, want in ((dq, dQ), (dk, dK), (dv, dV)):
            assert orc.rel_l2(_head(got, h), want) <= TOL_G


def test_c5_sweep_64k_causal_sampled():
    """C5 high end: N = 64K causal, B1 H32: forward on sampled rows (inference and the
    training O'), dQ of sampled rows through backward_rows_dq."""
    q, k, v, do = _inputs(1, 32, 65536, grad=True)
    _check_forward(q, k, v, True, heads=(31,), tag="C5 64K infer")
    o, lse, o_hp, ws = aq.attn_forward(q, k, v, causal=True, train=True, keep_for_bwd=True)
    dq, _, _ = aq.attn_backward(q, k, v, do, o, o_hp, lse, causal=True, fwd_workspace=ws)
    rows = _rows(65536, seed=1)
    h = 17
    Q, K, V, dO = (_head(t, h) for t in (q, k, v, do))
    want = orc.forward_rows(Q, K, V, rows, True, training=True)
    got_op = _head(o_hp, h)[rows]
    assert orc.rel_l2(got_op, want["O_prime"]) <= TOL_OP
    dq_want = orc.backward_rows_dq(Q, K, V, dO[rows], want["O_prime"], want["L"], rows, causal=True)
    e = orc.rel_l2(_head(dq, h)[rows], dq_want)
    print(f"C5 64K causal head {h}: dQ rows {e:.2e}")
    assert e <= TOL_G
