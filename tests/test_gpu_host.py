"""Host-buffer entry points (flash.attn_forward_host / attn_qat_host): chunked,
stream-overlapped H2D / kernels / D2H must give exactly the device-path results."""

import pytest
import torch

import paper_2603_00040_b200 as aq

pytestmark = pytest.mark.gpu


def _inputs(shape, seed=0):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(*shape, generator=g).bfloat16() for _ in range(4)]


@pytest.mark.parametrize("train", [False, True])
@pytest.mark.parametrize("chunk", [1, 3, 64])
def test_forward_host_equals_device(train, chunk):
    q, k, v, _ = _inputs((2, 5, 384, 128))
    o, lse, ohp = aq.attn_forward_host(q, k, v, causal=True, train=train, chunk_heads=chunk)
    torch.cuda.synchronize()
    o_d, lse_d, ohp_d, _ = aq.attn_forward(q.cuda(), k.cuda(), v.cuda(), causal=True, train=train)
    assert o.device.type == "cpu" and o.shape == q.shape
    assert torch.equal(o, o_d.cpu())
    assert torch.equal(lse, lse_d.cpu())
    if train:
        assert torch.equal(ohp, ohp_d.cpu())
    else:
        assert ohp is None


def test_qat_host_equals_autograd():
    q, k, v, d_o = _inputs((1, 6, 256, 64), seed=1)
    o, dq, dk, dv = aq.attn_qat_host(q, k, v, d_o, causal=False, chunk_heads=4)
    torch.cuda.synchronize()
    qg, kg, vg = (t.cuda().requires_grad_() for t in (q, k, v))
    out = aq.attn_qat(qg, kg, vg, causal=False)
    out.backward(d_o.cuda())
    assert torch.equal(o, out.detach().cpu())
    for a, b in ((dq, qg.grad), (dk, kg.grad), (dv, vg.grad)):
        assert torch.equal(a, b.cpu())


def test_numpy_reference_api_uses_host_path():
    q, k, v, _ = _inputs((1, 256, 64), seed=2)
    Q, K, V = (t[0].float().numpy() for t in (q, k, v))
    outs = aq.flash_forward_inference(Q, K, V, aq.TileConfig(128, 128))
    o_d, lse_d, _, _ = aq.attn_forward(q[0].float().cuda(), k[0].float().cuda(), v[0].float().cuda(),
                                       causal=False, train=False)
    assert (outs.O == o_d.cpu().numpy()).all()
