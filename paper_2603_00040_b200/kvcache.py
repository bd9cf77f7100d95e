"""NVFP4 KV cache: store K and V once as 4-bit QuantTensors, attend over them.

The reference quantizes K row-wise and V as V^T with blocks along tokens inside
``flash_forward_inference`` (flash.py:265-267) on every call. Caching those
two QuantTensors turns the inference forward into "quantize Q, attend": the
paper's stated next step, a 4-bit KV cache. The cache is the
reference's own QuantTensor layout, so it round-trips through ATQ4 files
(tensors.py) and a cache quantized by the reference loads unchanged:

    K   : quantize(K)             per head (n, d)  -> codes (n, d/2),   scales (n, d/16)
    V^T : quantize_padded(V.T)    per head (d, n16) -> codes (d, n16/2), scales (d, n16/16)

Batched over heads as [heads, ...]; on disk the head axis is folded into the
rows of one 2-D QuantTensor per operand (K: heads*n rows, V^T: heads*d rows).
``attn_forward_kv4`` is bit-identical to ``attn_forward(train=False)`` on the
K / V the cache was quantized from (the repack kernel moves bytes only).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .codec import NVFP4, QuantTensor
from .errors import InvalidValue, ShapeError
from .tensors import load_quant_tensor, save_quant_tensor


@dataclass
class KV4Cache:
    heads: int
    n: int
    d: int
    k_codes: torch.Tensor     # [heads, n, d/2] u8
    k_scales: torch.Tensor    # [heads, n, d/16] u8 (E4M3)
    vt_codes: torch.Tensor    # [heads, d, n16/2] u8
    vt_scales: torch.Tensor   # [heads, d, n16/16] u8

    @property
    def n16(self):
        return -(-self.n // 16) * 16

    def to(self, device):
        return KV4Cache(self.heads, self.n, self.d, *(t.to(device) for t in
                                                      (self.k_codes, self.k_scales, self.vt_codes, self.vt_scales)))

    def pin_memory(self):
        return KV4Cache(self.heads, self.n, self.d, *(t.cpu().pin_memory() for t in
                                                      (self.k_codes, self.k_scales, self.vt_codes, self.vt_scales)))

    def nbytes(self):
        return sum(t.numel() for t in (self.k_codes, self.k_scales, self.vt_codes, self.vt_scales))

    def k_tensor(self) -> QuantTensor:
        """K as one 2-D QuantTensor (heads*n, d)."""
        return QuantTensor(self.heads * self.n, self.d, NVFP4, self.k_codes.reshape(self.heads * self.n, -1),
                           self.k_scales.reshape(self.heads * self.n, -1))

    def vt_tensor(self) -> QuantTensor:
        """V^T as one 2-D QuantTensor (heads*d, n16)."""
        return QuantTensor(self.heads * self.d, self.n16, NVFP4, self.vt_codes.reshape(self.heads * self.d, -1),
                           self.vt_scales.reshape(self.heads * self.d, -1))


def kv4_quantize(k, v) -> KV4Cache:
    """Quantize K [..., n, d] and V [..., n, d] (CUDA tensors) into a KV4Cache."""
    _lib.require_cuda()
    if k.shape != v.shape or k.dim() < 2:
        raise ShapeError(f"K {tuple(k.shape)} and V {tuple(v.shape)} must share a [..., n, d] shape")
    if k.dtype not in _lib.DT_CODE or v.dtype not in _lib.DT_CODE:
        raise InvalidValue("K and V must be float32 / bfloat16 / float16")
    n, d = k.shape[-2:]
    if d % 16:
        raise ShapeError("d must be a multiple of the block size")
    k3 = k.reshape(-1, n, d).contiguous()
    v3 = v.reshape(-1, n, d).contiguous()
    heads = k3.shape[0]
    n16 = -(-n // 16) * 16
    dev = k.device
    kc = torch.empty(heads, n, d // 2, dtype=torch.uint8, device=dev)
    ks = torch.empty(heads, n, d // 16, dtype=torch.uint8, device=dev)
    vc = torch.empty(heads, d, n16 // 2, dtype=torch.uint8, device=dev)
    vs = torch.empty(heads, d, n16 // 16, dtype=torch.uint8, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    st = _lib.stream_ptr()
    _lib.check(lib.aq_quantize_rows(_lib.ptr(k3), _lib.DT_CODE[k3.dtype], heads, n, d, d, n * d, _lib.ptr(kc),
                                    _lib.ptr(ks), None, 0, 1.0, _lib.ptr(flag), st))
    _lib.check(lib.aq_quantize_cols(_lib.ptr(v3), _lib.DT_CODE[v3.dtype], heads, n, d, d, n * d, _lib.ptr(vc),
                                    _lib.ptr(vs), None, 0, 1.0, _lib.ptr(flag), st))
    if int(flag.item()):
        raise InvalidValue("quantize requires finite input")
    return KV4Cache(heads, n, d, kc, ks, vc, vs)


def attn_forward_kv4(q, cache: KV4Cache, causal=False, out=None, lse_out=None, workspace=None, out_dtype=None):
    """Inference forward over an FP4 KV cache: q [..., n_q, d] CUDA -> (O, L).

    Same math and bits as flash_forward_inference / attn_forward(train=False)
    with the K, V the cache holds (flash.py:249-314)."""
    _lib.require_cuda()
    if q.dim() < 2:
        raise ShapeError("q must be [..., n_q, d]")
    n_q, d = q.shape[-2:]
    q3 = q.reshape(-1, n_q, d).contiguous()
    heads = q3.shape[0]
    if heads != cache.heads or d != cache.d:
        raise ShapeError(f"q {tuple(q.shape)} does not match the cache (heads {cache.heads}, d {cache.d})")
    if causal and n_q > cache.n:
        raise ShapeError("causal attention requires N_q <= N_k")
    if q.dtype not in _lib.DT_CODE:
        raise InvalidValue("q must be float32 / bfloat16 / float16")
    for t in (cache.k_codes, cache.k_scales, cache.vt_codes, cache.vt_scales):
        if t.device != q.device or t.dtype != torch.uint8 or not t.is_contiguous():
            raise InvalidValue("cache tensors must be contiguous uint8 on q's device")
    out_dtype = out_dtype or q.dtype
    lib = _lib.load()
    ws_bytes = lib.aq_attn_fwd_workspace_bytes(heads, n_q, cache.n, d, 0, 0)
    if ws_bytes <= 0:
        raise InvalidValue(f"unsupported head dim {d} (the B200 kernels take d in {{64, 128}})")
    if workspace is None:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    elif workspace.numel() < ws_bytes:
        raise ShapeError("workspace too small")
    o = out if out is not None else torch.empty((heads, n_q, d), dtype=out_dtype, device=q.device)
    lse = lse_out if lse_out is not None else torch.empty((heads, n_q), dtype=torch.float32, device=q.device)
    args = _lib.AqFwdArgs(q=q3.data_ptr(), k=None, v=None, in_dtype=_lib.DT_CODE[q.dtype], heads=heads, n_q=n_q,
                          n_k=cache.n, d=d, causal=int(causal), train=0, o=o.data_ptr(),
                          o_dtype=_lib.DT_CODE[out_dtype], o_hp=None, o_hp_dtype=0, lse=lse.data_ptr(),
                          workspace=workspace.data_ptr(), keep_for_bwd=0, operands_staged=0)
    _lib.check(lib.aq_attn_fwd_kv4(args, _lib.ptr(cache.k_codes), _lib.ptr(cache.k_scales),
                                   _lib.ptr(cache.vt_codes), _lib.ptr(cache.vt_scales), _lib.stream_ptr()))
    lead = q.shape[:-2]
    return o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q)


def save_kv4(cache: KV4Cache, prefix):
    """Write ``<prefix>.k.atq4`` and ``<prefix>.vt.atq4`` (reference ATQ4 files)."""
    save_quant_tensor(cache.k_tensor(), f"{prefix}.k.atq4")
    save_quant_tensor(cache.vt_tensor(), f"{prefix}.vt.atq4")


def load_kv4(prefix, device="cuda") -> KV4Cache:
    """Read a cache written by save_kv4 (or two reference ATQ4 files)."""
    kq = load_quant_tensor(f"{prefix}.k.atq4", device=device)
    vq = load_quant_tensor(f"{prefix}.vt.atq4", device=device)
    if kq.spec != NVFP4 or vq.spec != NVFP4:
        raise InvalidValue("the FP4 KV cache is NVFP4 (16-element blocks, E4M3 scales)")
    d = kq.cols
    if vq.rows % d:
        raise ShapeError("V^T rows are not a multiple of the head dim")
    heads = vq.rows // d
    if kq.rows % heads:
        raise ShapeError("K rows are not a multiple of the head count")
    n = kq.rows // heads
    if vq.cols != -(-n // 16) * 16:
        raise ShapeError("V^T columns do not match the padded token count")
    return KV4Cache(heads, n, d, kq.codes.reshape(heads, n, d // 2), kq.scales.reshape(heads, n, d // 16),
                    vq.codes.reshape(heads, d, vq.cols // 2), vq.scales.reshape(heads, d, vq.cols // 16))


def attn_forward_kv4_host(q, cache: KV4Cache, causal=False, out=None, lse_out=None, out_dtype=None,
                          chunk_heads=None, sync=True):
    """FP4-KV-cache inference from host memory: q [..., n_q, d] and a KV4Cache
    on the host (pinned for overlap) -> host (O, L). Only Q (16-bit) and the
    4-bit cache cross PCIe -- 0.5625 B per cached K/V element instead of 2 --
    streamed over head chunks like attn_forward_host (host.py)."""
    from .host import default_chunk, run_pipelined
    _lib.require_cuda()
    if q.device.type != "cpu" or cache.k_codes.device.type != "cpu":
        raise InvalidValue("host entry points take CPU tensors (pinned for overlapped copies)")
    n_q, d = q.shape[-2:]
    q3 = q.reshape(-1, n_q, d)
    heads = q3.shape[0]
    if heads != cache.heads or d != cache.d:
        raise ShapeError(f"q {tuple(q.shape)} does not match the cache (heads {cache.heads}, d {cache.d})")
    out_dtype = out_dtype or q.dtype
    o = out.reshape(heads, n_q, d) if out is not None else torch.empty((heads, n_q, d), dtype=out_dtype,
                                                                         pin_memory=True)
    lse = lse_out.reshape(heads, n_q) if lse_out is not None else torch.empty((heads, n_q), dtype=torch.float32,
                                                                              pin_memory=True)
    per_head = q3[0].numel() * q3.element_size() + cache.nbytes() // heads
    chunk = chunk_heads or default_chunk(heads, per_head, items_per_head=-(-n_q // 128))
    lib = _lib.load()
    ws = (lambda h: (lib.aq_attn_fwd_workspace_bytes(h, n_q, cache.n, d, 0, 0),), torch.uint8)

    def fn(dev, res, scr):
        part = KV4Cache(dev[1].shape[0], cache.n, d, *dev[1:])
        attn_forward_kv4(dev[0], part, causal=causal, out=res[0], lse_out=res[1], workspace=scr[0],
                         out_dtype=out_dtype)
    run_pipelined(fn, [q3, cache.k_codes, cache.k_scales, cache.vt_codes, cache.vt_scales], [o, lse], chunk,
                  scratch=[("kv4_ws", *ws)], sync=sync)
    lead = q.shape[:-2]
    return o.reshape(*lead, n_q, d), lse.reshape(*lead, n_q)
