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
