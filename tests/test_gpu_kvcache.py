"""FP4 KV cache (kvcache.py): attention over stored 4-bit K / V^T is bit-identical
to the inference forward on the originals, and a cache written by the
reference (golden ATQ4 files) reproduces the reference's output."""

import os

import numpy as np
import pytest
import torch

import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("n,d,causal", [(256, 128, False), (200, 64, True), (1000, 128, True), (77, 64, False)])
def test_kv4_bit_identical_to_inference(n, d, causal):
    g = torch.Generator(device="cuda").manual_seed(n + d)
    q, k, v = (torch.randn(2, 3, n, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    cache = aq.kv4_quantize(k, v)
    o, lse = aq.attn_forward_kv4(q, cache, causal=causal)
    o_ref, lse_ref, _, _ = aq.attn_forward(q, k, v, causal=causal, train=False)
    assert torch.equal(o, o_ref)
    assert torch.equal(lse, lse_ref)
    assert cache.nbytes() * 3 < 2 * k.numel() * 2   # 0.5625 B per element vs 2 B in bf16


def test_kv4_cache_matches_reference_codec():
    g = torch.Generator(device="cuda").manual_seed(3)
    k, v = (torch.randn(1, 150, 64, generator=g, device="cuda") for _ in range(2))
    cache = aq.kv4_quantize(k, v)
    kc, ks = orc.quantize(k[0].double().cpu().numpy())
    vc, vs = orc.quantize(orc.pad_cols(np.ascontiguousarray(v[0].double().cpu().numpy().T)))
    assert np.array_equal(cache.k_codes[0].cpu().numpy(), kc) and np.array_equal(cache.k_scales[0].cpu().numpy(), ks)
    assert np.array_equal(cache.vt_codes[0].cpu().numpy(), vc) and np.array_equal(cache.vt_scales[0].cpu().numpy(), vs)


def test_reference_written_cache(tmp_path):
    fx = np.load(os.path.join(GOLD, "formats.npz"))
    cache = aq.load_kv4(os.path.join(GOLD, "ref_kv"))
    assert (cache.heads, cache.n, cache.d) == (2, 200, 64)
    q = torch.from_numpy(fx["Q"]).float().cuda()
    o, lse = aq.attn_forward_kv4(q, cache)
    for h in range(2):
        assert orc.rel_l2(o[h].cpu().numpy(), fx["O"][h]) <= 1e-2
        assert np.max(np.abs(lse[h].cpu().numpy() - fx["L"][h])) <= 2e-5
    # our quantizer produces the same cache bytes, and save -> load round-trips
    mine = aq.kv4_quantize(torch.from_numpy(fx["K"]).float().cuda(), torch.from_numpy(fx["V"]).float().cuda())
    for a, b in ((mine.k_codes, cache.k_codes), (mine.k_scales, cache.k_scales), (mine.vt_codes, cache.vt_codes),
                 (mine.vt_scales, cache.vt_scales)):
        assert torch.equal(a, b)
    aq.save_kv4(mine, str(tmp_path / "kv"))
    for suf in (".k.atq4", ".vt.atq4"):
        assert (tmp_path / f"kv{suf}").read_bytes() == open(os.path.join(GOLD, f"ref_kv{suf}"), "rb").read()


def test_kv4_errors():
    g = torch.Generator(device="cuda").manual_seed(0)
    k, v = (torch.randn(2, 128, 64, generator=g, device="cuda") for _ in range(2))
    cache = aq.kv4_quantize(k, v)
    with pytest.raises(aq.ShapeError):
        aq.attn_forward_kv4(torch.randn(3, 128, 64, device="cuda"), cache)
    with pytest.raises(aq.ShapeError):
        aq.attn_forward_kv4(torch.randn(2, 256, 64, device="cuda"), cache, causal=True)
    with pytest.raises(aq.ShapeError):
        aq.kv4_quantize(k, v[:, :64])


def test_kv4_host_pipeline_equals_device():
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, v = (torch.randn(2, 5, 384, 128, generator=g, device="cuda").bfloat16() for _ in range(3))
    cache = aq.kv4_quantize(k, v)
    o_d, l_d = aq.attn_forward_kv4(q, cache, causal=True)
    o_h, l_h = aq.attn_forward_kv4_host(q.cpu().pin_memory(), cache.pin_memory(), causal=True, chunk_heads=3)
    torch.cuda.synchronize()
    assert o_h.device.type == "cpu" and torch.equal(o_h, o_d.cpu()) and torch.equal(l_h, l_d.cpu())
