"""On-disk tensor formats, byte-compatible with the reference (tensors.py:122-220).

ATNQ (dense float tensor), little endian:
    "ATNQ" | u32 version=1 | u8 width (0 = f32, 1 = f64) | u8 ndim (1..3)
    | u32 dims[ndim] | payload (row-major)
ATQ4 (QuantTensor: packed FP4 codes + block-scale grid):
    "ATQ4" | u32 version=1 | u8 scale format (0 = E4M3, 1 = E8M0) | u16 block
    | u32 rows | u32 cols | scales [rows][cols/block] u8 | codes [rows][cols/2] u8

Readers validate every field the way the reference does and raise FormatError
carrying the byte offset of the problem (truncation, bad magic / version /
width / ndim / scale format, trailing bytes). ``save_quant_tensor`` accepts a
QuantTensor whose codes / scales live on the GPU (they are copied to the host);
``load_quant_tensor(path, device=...)`` can place them straight on the GPU,
ready for ``dequantize`` or the FP4 KV cache (kvcache.py).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .codec import BlockSpec, QuantTensor, ScaleFormat
from .errors import FormatError, InvalidValue, ShapeError

TENSOR_MAGIC = b"ATNQ"
QUANT_MAGIC = b"ATQ4"
_VERSION = 1
_WIDTH = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
_WIDTH_DT = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_TENSOR_HDR = struct.Struct("<IBB")      # version, width, ndim
_QUANT_HDR = struct.Struct("<IBHII")     # version, scale format, block, rows, cols


def _host(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


class _Reader:
    """Sequential reader that reports the offset of a short read."""

    def __init__(self, fh):
        self.fh = fh
        self.pos = 0

    def take(self, n, what):
        buf = self.fh.read(n)
        if len(buf) != n:
            raise FormatError(f"truncated while reading {what}", offset=self.pos + len(buf))
        self.pos += n
        return buf

    def expect_end(self):
        if self.fh.read(1):
            raise FormatError("trailing bytes after payload", offset=self.pos)


def save_tensor(t, path):
    """Write a 1-3-D float32 / float64 tensor as ATNQ."""
    arr = np.ascontiguousarray(_host(t))
    if arr.dtype not in _WIDTH:
        raise FormatError(f"unsupported dtype {arr.dtype}")
    if arr.ndim < 1 or arr.ndim > 3:
        raise ShapeError("ATNQ stores 1-3 dimensional tensors")
    with open(path, "wb") as fh:
        fh.write(TENSOR_MAGIC + _TENSOR_HDR.pack(_VERSION, _WIDTH[arr.dtype], arr.ndim))
        fh.write(struct.pack("<" + "I" * arr.ndim, *arr.shape))
        fh.write(arr.astype(arr.dtype.newbyteorder("<"), copy=False).tobytes())


def load_tensor(path):
    """Read an ATNQ file (bit-identical round trip of save_tensor)."""
    with open(path, "rb") as fh:
        rd = _Reader(fh)
        if rd.take(4, "magic") != TENSOR_MAGIC:
            raise FormatError("bad magic", offset=0)
        version, width, ndim = _TENSOR_HDR.unpack(rd.take(_TENSOR_HDR.size, "header"))
        if version != _VERSION:
            raise FormatError(f"unsupported version {version}", offset=4)
        if width not in _WIDTH_DT:
            raise FormatError(f"unknown width code {width}", offset=8)
        if ndim < 1 or ndim > 3:
            raise FormatError(f"bad ndim {ndim}", offset=9)
        dims = struct.unpack("<" + "I" * ndim, rd.take(4 * ndim, "dims"))
        dt = _WIDTH_DT[width]
        count = 1
        for x in dims:
            count *= x
        payload = rd.take(count * dt.itemsize, "payload")
        rd.expect_end()
    return np.frombuffer(payload, dtype=dt).reshape(dims).astype(np.float32 if width == 0 else np.float64)


def save_quant_tensor(qt: QuantTensor, path):
    """Write a QuantTensor as ATQ4 (scale grid first, then packed nibbles)."""
    scales = np.ascontiguousarray(_host(qt.scales), dtype=np.uint8)
    codes = np.ascontiguousarray(_host(qt.codes), dtype=np.uint8)
    bs = qt.spec.block_size
    if scales.size != qt.rows * (qt.cols // bs) or codes.size != qt.rows * qt.cols // 2:
        raise ShapeError("QuantTensor codes / scales do not match rows x cols")
    with open(path, "wb") as fh:
        fh.write(QUANT_MAGIC + _QUANT_HDR.pack(_VERSION, qt.spec.scale_format.value, bs, qt.rows, qt.cols))
        fh.write(scales.tobytes())
        fh.write(codes.tobytes())


def load_quant_tensor(path, device=None) -> QuantTensor:
    """Read an ATQ4 file. ``device=None`` returns NumPy arrays (the reference's
    behaviour); a torch device places codes and scales there."""
    with open(path, "rb") as fh:
        rd = _Reader(fh)
        if rd.take(4, "magic") != QUANT_MAGIC:
            raise FormatError("bad magic", offset=0)
        version, fmt, bs, rows, cols = _QUANT_HDR.unpack(rd.take(_QUANT_HDR.size, "header"))
        if version != _VERSION:
            raise FormatError(f"unsupported version {version}", offset=4)
        try:
            spec = BlockSpec(bs, ScaleFormat(fmt))
        except (ValueError, InvalidValue):
            raise FormatError(f"unknown scale format {fmt} / block {bs}", offset=8) from None
        scales = np.frombuffer(rd.take(rows * (cols // bs), "scale grid"), dtype=np.uint8).reshape(rows, cols // bs)
        codes = np.frombuffer(rd.take(rows * cols // 2, "payload"), dtype=np.uint8).reshape(rows, cols // 2)
        rd.expect_end()
    if device is not None:
        return QuantTensor(rows, cols, spec, torch.from_numpy(codes.copy()).to(device),
                           torch.from_numpy(scales.copy()).to(device))
    return QuantTensor(rows, cols, spec, codes.copy(), scales.copy())


# ----------------------------------------------------------------------------
# deterministic host random streams (tensors.py:89-117): test-data generators,
# identical streams to the reference for the same seed
# ----------------------------------------------------------------------------

class Rng:
    """PCG64 stream with NumPy's standard normal; ``spawn`` derives an
    independent stream from (seed, offset) the way the reference does."""

    def __init__(self, seed):
        self.seed = int(seed)
        self._gen = np.random.Generator(np.random.PCG64(self.seed))

    def spawn(self, offset):
        return Rng(self.seed * 0x9E3779B9 + offset & 0x7FFFFFFFFFFFFFFF)

    def standard_normal(self, dims, dtype=np.float64):
        return self._gen.standard_normal(size=dims).astype(dtype)

    def integers(self, low, high=None, size=None):
        return self._gen.integers(low, high=high, size=size)

    def uniform(self, low=0.0, high=1.0, size=None):
        return self._gen.uniform(low, high, size=size)


def randn(dims, rng, scale=1.0, dtype=np.float64):
    """i.i.d. N(0, scale^2) host tensor from an Rng."""
    if scale <= 0:
        raise ShapeError("scale must be positive")
    return scale * rng.standard_normal(tuple(dims), dtype=dtype)


# ----------------------------------------------------------------------------
# matrix products (tensors.py:25-86)
# ----------------------------------------------------------------------------

def _dev_u8(a):
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8))
    return t.to("cuda").contiguous()


def fp4mm(aq, bq_t, accum_width=32):
    """C = A @ B from NVFP4 or MXFP4 QuantTensors, B supplied transposed (both
    blocked along the contraction axis; tensors.py:54-86), on block-scaled
    tcgen05 MMAs (kind::mxf4nvf4 block16 / kind::mxf4 block32). Exact block products, fp32 accumulation (accum_width=64 raises
    InvalidValue: the tensor cores accumulate in fp32). NumPy operands give a
    NumPy result, torch operands a CUDA tensor."""
    from . import _lib
    from .codec import NVFP4
    if not isinstance(aq, QuantTensor) or not isinstance(bq_t, QuantTensor):
        raise ShapeError("fp4mm operands must be QuantTensors")
    if aq.spec != bq_t.spec:
        raise ShapeError("fp4mm operands must share a BlockSpec")
    if aq.cols != bq_t.cols:
        raise ShapeError(f"contraction axes differ: {aq.cols} vs {bq_t.cols}")
    if accum_width not in (32, 64):
        raise ShapeError(f"accum_width must be 32 or 64, got {accum_width}")
    if accum_width != 32:
        raise InvalidValue("the B200 path accumulates in fp32 (tensor cores); accum_width=64 is CPU-only")
    from .codec import MXFP4
    if aq.spec not in (NVFP4, MXFP4):
        raise InvalidValue("the B200 path implements NVFP4 and MXFP4")
    _lib.require_cuda()
    as_np = not isinstance(aq.codes, torch.Tensor)
    ac, asf, bc, bsf = (_dev_u8(x) for x in (aq.codes, aq.scales, bq_t.codes, bq_t.scales))
    M, N, K = aq.rows, bq_t.rows, aq.cols
    lib = _lib.load()
    ws = torch.empty(lib.aq_fp4mm_workspace_bytes(M, N, K), dtype=torch.uint8, device="cuda")
    c = torch.empty((M, N), dtype=torch.float32, device="cuda")
    fn = lib.aq_fp4mm_mx if aq.spec == MXFP4 else lib.aq_fp4mm
    _lib.check(fn(_lib.ptr(ac), _lib.ptr(asf), M, _lib.ptr(bc), _lib.ptr(bsf), N, K, _lib.ptr(c), N,
                  _lib.ptr(ws), _lib.stream_ptr()))
    return c.cpu().numpy() if as_np else c


def matmul(a, b, accum_width=32):
    """a @ b in the accumulation width (tensors.py:32-51), on the GPU (cuBLAS
    through torch; the reference's fixed left-to-right summation order is not
    reproduced, results agree to fp32 / fp64 rounding). a may be 3-D with b
    shared across the batch."""
    from . import _lib
    if accum_width not in (32, 64):
        raise ShapeError(f"accum_width must be 32 or 64, got {accum_width}")
    dt = torch.float32 if accum_width == 32 else torch.float64
    as_np = not isinstance(a, torch.Tensor)
    _lib.require_cuda()
    ta = torch.as_tensor(np.asarray(a) if as_np else a).to("cuda", dt)
    tb = torch.as_tensor(np.asarray(b) if not isinstance(b, torch.Tensor) else b).to("cuda", dt)
    if ta.dim() not in (2, 3) or tb.dim() != 2:
        raise ShapeError("matmul expects a 2-D or 3-D left operand and 2-D right")
    if tb.shape[0] != ta.shape[-1]:
        raise ShapeError(f"inner dims mismatch: {tuple(ta.shape)} x {tuple(tb.shape)}")
    out = ta @ tb
    return out.cpu().numpy() if as_np else out
