"""Small ragged cases of every GPU entry point (incl. sage3, quantized=False, the ABI-3 scale / instrument
arguments), for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for n, d, causal in ((200, 64, True), (77, 128, False)):
    q, k, v, do = (torch.randn(1, 2, n, d, generator=g, device="cuda").bfloat16() for _ in range(4))
    o = aq.attn_qat(q.requires_grad_(), k.requires_grad_(), v.requires_grad_(), causal=causal)
    o.backward(do)
    aq.attn_forward(q.detach(), k.detach(), v.detach(), causal=causal, train=False)
    cache = aq.kv4_quantize(k.detach(), v.detach())
    aq.attn_forward_kv4(q.detach(), cache, causal=causal)
for n, d in ((1100, 128), (1030, 64)):  # the training forward's dynamic item queue (>= 8 causal query tiles,
    # more items than CTAs so the queue hands out claims)
    q, k, v, do = (torch.randn(1, 24, n, d, generator=g, device="cuda").bfloat16() for _ in range(4))
    aq.attn_qat(q.requires_grad_(), k.requires_grad_(), v.requires_grad_(), causal=True).backward(do)
for n, d, causal, b_q, b_k, tl in ((200, 64, True, 40, 200, True), (77, 128, False, 77, 77, True),
                                   (77, 128, True, 77, 77, False), (256, 64, True, 16, 128, True),
                                   (256, 128, False, 8, 32, True), (384, 64, True, 64, 48, True),
                                   (512, 128, False, 128, 256, True)):
    q, k, v = (torch.randn(1, 2, n, d, generator=g, device="cuda").bfloat16() + 1 for _ in range(3))
    aq.attn_forward_sage3(q, k, v, causal=causal, b_q=b_q, b_k=b_k, two_level_p=tl)
for n, d, causal in ((200, 64, True), (77, 128, False)):
    q, k, v = (torch.randn(1, 2, n, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    aq.attn_forward_mx(q, k, v, causal=causal)
    o, lse, o_hp = aq.attn_forward_mx(q, k, v, causal=causal, train=True)
    aq.attn_backward(q, k, v, torch.randn_like(q), o, o_hp, lse, causal=causal, mx=True)
    qg, kg, vg = (t.clone().requires_grad_() for t in (q, k, v))
    aq.attn_qat(qg, kg, vg, causal=causal, spec=aq.MXFP4).backward(torch.randn_like(q))
    aq.fp4mm(aq.quantize(q[0, 0].float(), aq.MXFP4), aq.quantize(k[0, 0].float(), aq.MXFP4))
for n, d, causal in ((200, 64, True), (77, 128, False), (96, 24, True)):  # quantized=False fwd + bwd (K4 / K7 PLAIN)
    q, k, v, do = (torch.randn(1, 2, n, d, generator=g, device="cuda").bfloat16() for _ in range(4))
    aq.attn_qat(q.requires_grad_(), k.requires_grad_(), v.requires_grad_(), causal=causal, quantized=False).backward(do)
for n, d in ((200, 32), (77, 128)):  # tensor scales, P tensor scale, instrument dump, non-finite flag
    q, k, v, do = (torch.randn(1, 2, n, d, generator=g, device="cuda").bfloat16() for _ in range(4))
    pf = aq.pf_buffers(2, n, n)
    o, lse, o_hp, ws = aq.attn_forward(q, k, v, causal=True, train=True, keep_for_bwd=True, q_scale="auto",
                                       k_scale=0.5, v_scale=2.0, p_scale=1 / 2688, pf_out=pf)
    aq.attn_backward(q, k, v, do, o, o_hp, lse, causal=True, fwd_workspace=ws, q_scale="auto", k_scale=0.5,
                     v_scale=2.0, p_scale=1 / 2688, pf_out=aq.pf_buffers(2, n, n))
x = torch.randn(37, 48, generator=g, device="cuda")
aq.fp4mm(aq.quantize(x), aq.quantize(torch.randn(29, 48, generator=g, device="cuda")))
aq.fake_quantize(torch.randn(5, 64, generator=g, device="cuda"), aq.MXFP4)
aq.round_to_fp4(np.linspace(-7, 7, 101))
torch.cuda.synchronize()
print("sanitize cases ok")
