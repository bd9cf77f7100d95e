"""NVFP4 codec on the GPU, mirroring ``attnqat.codec`` (codec.py:145-381).

Same names, argument meaning and errors as the reference; the arithmetic runs
in the sm_100a quantizer kernels (csrc/quantize.cu) through the C ABI.
Inputs may be NumPy arrays (uploaded; results come back as NumPy) or torch
tensors (results stay on the GPU). float64 inputs are rounded to float32 on
upload -- the kernels quantize fp32 / bf16 / fp16 values (bit-exact versus the
reference for every value representable in those formats).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .errors import InvalidValue, ShapeError

FP4_MAX = 6.0
E4M3_MAX = 448.0


class ScaleFormat(Enum):
    E4M3 = 0
    E8M0 = 1


@dataclass(frozen=True)
class BlockSpec:
    """Block size and scale format (codec.py:150-163)."""

    block_size: int
    scale_format: ScaleFormat

    def __post_init__(self):
        if (self.block_size, self.scale_format) not in {(16, ScaleFormat.E4M3), (32, ScaleFormat.E8M0)}:
            raise InvalidValue(f"unsupported block spec ({self.block_size}, {self.scale_format})")


NVFP4 = BlockSpec(16, ScaleFormat.E4M3)
MXFP4 = BlockSpec(32, ScaleFormat.E8M0)


def _require_nvfp4(spec):
    if spec != NVFP4:
        raise InvalidValue("the B200 path implements NVFP4 (16-element blocks, E4M3 scales) only")


@dataclass
class QuantTensor:
    """Packed FP4 codes (rows, cols/2) + row-major scale grid (rows, cols/16) (codec.py:260-299)."""

    rows: int
    cols: int
    spec: BlockSpec
    codes: object
    scales: object
    # per-tensor FP32 scale of the two-level NVFP4 format (north_star): the
    # value is tensor_scale * scale * code. 1.0 is the reference's format
    # -- a QuantTensor from quantize() without the argument.
    tensor_scale: float = 1.0

    @property
    def block_grid(self):
        return (self.rows, self.cols // self.spec.block_size)

    def row_slice(self, start, stop):
        return QuantTensor(stop - start, self.cols, self.spec, self.codes[start:stop], self.scales[start:stop],
                           self.tensor_scale)

    def col_slice(self, start, stop):
        bs = self.spec.block_size
        if start % bs or stop % bs:
            raise ShapeError("column slices must align to block boundaries")
        return QuantTensor(self.rows, stop - start, self.spec, self.codes[:, start // 2:stop // 2],
                           self.scales[:, start // bs:stop // bs], self.tensor_scale)


def auto_tensor_scale(x):
    """The usual NVFP4 per-tensor scale amax(|x|) / (448 * 6): the largest block
    scale lands on E4M3's maximum (one device reduction, read back to the host)."""
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    amax = float(t.detach().abs().amax()) if t.numel() else 0.0
    return amax / (E4M3_MAX * FP4_MAX) if amax > 0 and np.isfinite(amax) else 1.0


def _ts(tensor_scale, x):
    """Resolve a tensor_scale argument: None / 1.0 (reference), 'auto', or a positive float."""
    if tensor_scale is None:
        return 1.0
    if isinstance(tensor_scale, str):
        if tensor_scale != "auto":
            raise InvalidValue(f"tensor_scale must be a positive float or 'auto', got {tensor_scale!r}")
        return auto_tensor_scale(x)
    ts = float(tensor_scale)
    if not (ts > 0 and np.isfinite(ts)):
        raise InvalidValue(f"tensor_scale must be positive and finite, got {tensor_scale}")
    return ts


def to_device(x, allow_f64=True):
    """(cuda tensor, came_from_numpy). float64 is rounded to float32."""
    _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t, was_np = x, False
    else:
        t, was_np = torch.from_numpy(np.ascontiguousarray(np.asarray(x))), True
    if not t.is_floating_point():
        t = t.to(torch.float32)
    if t.dtype == torch.float64:
        t = t.to(torch.float32)
    return t.to("cuda").contiguous(), was_np


def _out(t, as_numpy, np_dtype=None):
    if not as_numpy:
        return t
    a = t.cpu().numpy()
    return a.astype(np_dtype) if np_dtype is not None else a


def _nonfinite_check(flag):
    if int(flag.item()):
        raise InvalidValue("quantize requires finite input")


def _quantize_mx(t, codes=None, scales=None, fq=None):
    rows, cols = t.shape
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_quantize_mx(_lib.ptr(t), _lib.DT_CODE[t.dtype], rows, cols, _lib.ptr(codes),
                                          _lib.ptr(scales), _lib.ptr(fq), _lib.DT_CODE[fq.dtype] if fq is not None else 0,
                                          _lib.ptr(flag), _lib.stream_ptr()))
    _nonfinite_check(flag)


def quantize(x, spec=NVFP4, tensor_scale=None) -> QuantTensor:
    """Block-row-wise NVFP4 / MXFP4 quantization (codec.py:302-324).
    ``tensor_scale`` (NVFP4 only; None = the reference's format) selects the
    two-level format: blocks of x / tensor_scale are quantized."""
    if spec == MXFP4:
        t, was_np = to_device(x)
        if t.dim() != 2:
            raise ShapeError("quantize expects a 2-D tensor")
        rows, cols = t.shape
        if cols % 32:
            raise ShapeError(f"cols ({cols}) must be a multiple of block_size (32);"
                             " padding is the caller's responsibility")
        codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device=t.device)
        scales = torch.empty((rows, cols // 32), dtype=torch.uint8, device=t.device)
        _quantize_mx(t, codes=codes, scales=scales)
        return QuantTensor(rows, cols, spec, _out(codes, was_np), _out(scales, was_np))
    _require_nvfp4(spec)
    t, was_np = to_device(x)
    if t.dim() != 2:
        raise ShapeError("quantize expects a 2-D tensor")
    rows, cols = t.shape
    if cols % spec.block_size:
        raise ShapeError(f"cols ({cols}) must be a multiple of block_size ({spec.block_size});"
                         " padding is the caller's responsibility")
    ts = _ts(tensor_scale, t)
    codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device=t.device)
    scales = torch.empty((rows, cols // 16), dtype=torch.uint8, device=t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_quantize_rows(
        _lib.ptr(t), _lib.DT_CODE[t.dtype], 1, rows, cols, cols, rows * cols,
        _lib.ptr(codes), _lib.ptr(scales), None, 0, ts, _lib.ptr(flag), _lib.stream_ptr()))
    _nonfinite_check(flag)
    return QuantTensor(rows, cols, spec, _out(codes, was_np), _out(scales, was_np), ts)


_NP2T = {np.float32: torch.float32, np.float64: torch.float32, np.float16: torch.float16}


def dequantize(qt: QuantTensor, dtype=np.float32):
    """code x scale, exact (codec.py:327-333)."""
    was_np = not isinstance(qt.codes, torch.Tensor)
    codes = torch.as_tensor(np.ascontiguousarray(qt.codes) if was_np else qt.codes).to("cuda").contiguous()
    scales = torch.as_tensor(np.ascontiguousarray(qt.scales) if was_np else qt.scales).to("cuda").contiguous()
    tdt = dtype if isinstance(dtype, torch.dtype) else _NP2T.get(np.dtype(dtype).type, torch.float32)
    out = torch.empty((qt.rows, qt.cols), dtype=tdt, device="cuda")
    if qt.spec == MXFP4:
        _lib.check(_lib.load().aq_dequantize_mx(_lib.ptr(codes), _lib.ptr(scales), qt.rows, qt.cols, _lib.ptr(out),
                                                _lib.DT_CODE[tdt], _lib.stream_ptr()))
        return _out(out, was_np, None if isinstance(dtype, torch.dtype) else dtype)
    _lib.check(_lib.load().aq_dequantize(_lib.ptr(codes), _lib.ptr(scales), qt.rows, qt.cols,
                                         _lib.ptr(out), _lib.DT_CODE[tdt], float(qt.tensor_scale),
                                         _lib.stream_ptr()))
    return _out(out, was_np, None if isinstance(dtype, torch.dtype) else dtype)


def fake_quantize(x, spec=NVFP4, tensor_scale=None):
    """Quantize-then-dequantize, shape and dtype preserved (codec.py:336-340)."""
    if spec == MXFP4:
        t, was_np = to_device(x)
        if t.dim() != 2:
            raise ShapeError("quantize expects a 2-D tensor")
        if t.shape[1] % 32:
            raise ShapeError(f"cols ({t.shape[1]}) must be a multiple of block_size (32)")
        out = torch.empty_like(t)
        _quantize_mx(t, fq=out)
        return _out(out, was_np, np.asarray(x).dtype if was_np else None)
    _require_nvfp4(spec)
    t, was_np = to_device(x)
    if t.dim() != 2:
        raise ShapeError("quantize expects a 2-D tensor")
    rows, cols = t.shape
    if cols % spec.block_size:
        raise ShapeError(f"cols ({cols}) must be a multiple of block_size ({spec.block_size})")
    out = torch.empty_like(t)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_quantize_rows(
        _lib.ptr(t), _lib.DT_CODE[t.dtype], 1, rows, cols, cols, rows * cols,
        None, None, _lib.ptr(out), _lib.DT_CODE[out.dtype], _ts(tensor_scale, t), _lib.ptr(flag),
        _lib.stream_ptr()))
    _nonfinite_check(flag)
    np_dt = np.asarray(x).dtype if was_np else None
    return _out(out, was_np, np_dt)


def pad_cols(x, block_size):
    """Zero-pad the column axis to a block multiple (codec.py:343-356)."""
    cols = x.shape[1]
    rem = cols % block_size
    if rem == 0:
        return x
    if isinstance(x, torch.Tensor):
        return torch.nn.functional.pad(x, (0, block_size - rem))
    out = np.zeros((x.shape[0], cols + block_size - rem), dtype=np.asarray(x).dtype)
    out[:, :cols] = x
    return out


def quantize_padded(x, spec=NVFP4):
    """codec.py:359-361."""
    return quantize(pad_cols(x, spec.block_size), spec)


def fake_quantize_padded(x, spec=NVFP4):
    """codec.py:364-370."""
    n = x.shape[1]
    out = fake_quantize(pad_cols(x, spec.block_size), spec)
    return out[:, :n] if out.shape[1] != n else out


def fake_quantize_cols(x, spec=NVFP4, tensor_scale=None):
    """Blocks along the token (row) axis, ragged tail zero-padded (codec.py:373-381)."""
    if spec == MXFP4:
        t, was_np = to_device(x)
        n = t.shape[0]
        out = fake_quantize_padded(t.t().contiguous(), MXFP4)[:, :n].t().contiguous()
        return _out(out, was_np, np.asarray(x).dtype if was_np else None)
    _require_nvfp4(spec)
    t, was_np = to_device(x)
    if t.dim() != 2:
        raise ShapeError("quantize expects a 2-D tensor")
    n, cols = t.shape
    out = torch.empty_like(t)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_quantize_cols(
        _lib.ptr(t), _lib.DT_CODE[t.dtype], 1, n, cols, cols, n * cols,
        None, None, _lib.ptr(out), _lib.DT_CODE[out.dtype], _ts(tensor_scale, t), _lib.ptr(flag),
        _lib.stream_ptr()))
    _nonfinite_check(flag)
    np_dt = np.asarray(x).dtype if was_np else None
    return _out(out, was_np, np_dt)


def quantize_cols(x, spec=NVFP4, tensor_scale=None) -> QuantTensor:
    """QuantTensor of x^T with the token axis zero-padded: quantize_padded(x.T) (flash.py:267)."""
    _require_nvfp4(spec)
    t, was_np = to_device(x)
    n, cols = t.shape
    ts = _ts(tensor_scale, t)
    n16 = -(-n // 16) * 16
    codes = torch.empty((cols, n16 // 2), dtype=torch.uint8, device=t.device)
    scales = torch.empty((cols, n16 // 16), dtype=torch.uint8, device=t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_quantize_cols(
        _lib.ptr(t), _lib.DT_CODE[t.dtype], 1, n, cols, cols, n * cols,
        _lib.ptr(codes), _lib.ptr(scales), None, 0, ts, _lib.ptr(flag), _lib.stream_ptr()))
    _nonfinite_check(flag)
    return QuantTensor(cols, n16, spec, _out(codes, was_np), _out(scales, was_np), ts)


# ----------------------------------------------------------------------------
# element-wise codes and single blocks (codec.py:63-138, 225-258)
# ----------------------------------------------------------------------------

def _round_codes(x, fmt, what):
    was_np = not isinstance(x, torch.Tensor)
    if was_np:
        arr = np.asarray(x, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1)))
    else:
        arr = None
        t = x.reshape(-1)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float32)
    _lib.require_cuda()
    t = t.to("cuda").contiguous()
    codes = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_round_codes(_lib.ptr(t), 3 if t.dtype == torch.float64 else 0, t.numel(), fmt,
                                          _lib.ptr(codes), _lib.ptr(flag), _lib.stream_ptr()))
    if int(flag.item()):
        raise InvalidValue(f"{what} requires finite{' non-negative' if fmt == 1 else ''} input")
    if not was_np:
        return codes.reshape(x.shape)
    out = codes.cpu().numpy().reshape(arr.shape)
    return out if arr.ndim else out[()]


def round_to_fp4(x):
    """Nearest FP4 (E2M1) code, ties to even, saturating at +-6; -0.0 -> 0x0,
    a small negative that rounds to zero keeps the sign (codec.py:76-88).
    Exact in the input precision (float64 NumPy input is rounded in float64)."""
    return _round_codes(x, 0, "round_to_fp4")


def encode_fp4(values):
    """Alias of round_to_fp4 (codec.py:96-98)."""
    return round_to_fp4(values)


def round_to_e4m3(x):
    """Nearest finite E4M3 code of a non-negative value, ties to even, including
    subnormals; saturates at 448 -> 0x7E (codec.py:101-112)."""
    return _round_codes(x, 1, "round_to_e4m3")


_FP4_TABLE = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], dtype=np.float64)
FP4_DECODE = np.concatenate([_FP4_TABLE, -_FP4_TABLE])
FP4_DECODE[8] = 0.0   # both zeros decode to +0.0


def _e4m3_table():
    c = np.arange(256)
    e, m = (c >> 3) & 0xF, c & 7
    mag = np.where(e == 0, m * 2.0 ** -9, (1.0 + m / 8.0) * 2.0 ** (e.astype(np.float64) - 7))
    return np.where(c & 0x80, -mag, mag)


E4M3_DECODE = _e4m3_table()


def decode_fp4(codes):
    """4-bit codes -> FP4 values (codec.py:91-93)."""
    if isinstance(codes, torch.Tensor):
        return torch.as_tensor(FP4_DECODE, device=codes.device)[codes.long()]
    return FP4_DECODE[np.asarray(codes, dtype=np.uint8)]


def decode_e4m3(codes):
    """E4M3 codes -> values; NaN codes (0x7F / 0xFF) are rejected (codec.py:115-120)."""
    if isinstance(codes, torch.Tensor):
        if bool(((codes & 0x7F) == 0x7F).any()):
            raise InvalidValue("NaN E4M3 code cannot be used as a scale")
        return torch.as_tensor(E4M3_DECODE, device=codes.device)[codes.long()]
    c = np.asarray(codes, dtype=np.uint8)
    if np.any(c & 0x7F == 0x7F):
        raise InvalidValue("NaN E4M3 code cannot be used as a scale")
    return E4M3_DECODE[c]


@dataclass
class Fp4Block:
    """block_size FP4 codes packed two per byte plus one shared scale code (codec.py:225-236)."""

    codes: bytes
    scale: int
    spec: BlockSpec

    def __post_init__(self):
        if len(self.codes) != self.spec.block_size // 2:
            raise ShapeError(f"packed block must be {self.spec.block_size // 2} bytes")


def quantize_block(x, spec=NVFP4) -> Fp4Block:
    """One block of block_size finite reals -> Fp4Block (codec.py:239-248), on the GPU quantizer."""
    if spec not in (NVFP4, MXFP4):
        raise InvalidValue(f"unsupported block spec {spec}")
    arr = np.asarray(x.detach().cpu() if isinstance(x, torch.Tensor) else x, dtype=np.float64)
    if arr.shape != (spec.block_size,):
        raise ShapeError(f"block must have exactly {spec.block_size} elements")
    if not np.all(np.isfinite(arr)):
        raise InvalidValue("quantize_block requires finite input")
    qt = quantize(arr[None, :], spec)
    return Fp4Block(codes=bytes(np.asarray(qt.codes, dtype=np.uint8).reshape(-1)), scale=int(qt.scales[0, 0]),
                    spec=spec)


def dequantize_block(block: Fp4Block):
    """Fp4Block -> block_size float64 reals (scale x code, exact; codec.py:251-258)."""
    codes = np.frombuffer(block.codes, dtype=np.uint8).reshape(1, -1)
    scales = np.array([[block.scale]], dtype=np.uint8)
    qt = QuantTensor(1, block.spec.block_size, block.spec, codes, scales)
    return np.asarray(dequantize(qt, np.float64), dtype=np.float64).reshape(-1)


def round_to_e8m0(x):
    """Nearest power of two of a positive value, ties up -> E8M0 code clamped to
    0..254 (codec.py:123-136). Exact in the input precision."""
    was_np = not isinstance(x, torch.Tensor)
    arr = np.asarray(x, dtype=np.float64) if was_np else None
    t = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1))) if was_np else x.reshape(-1)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float32)
    _lib.require_cuda()
    t = t.to("cuda").contiguous()
    codes = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().aq_e8m0_codes(_lib.ptr(t), 3 if t.dtype == torch.float64 else 0, t.numel(),
                                         _lib.ptr(codes), _lib.ptr(flag), _lib.stream_ptr()))
    if int(flag.item()):
        raise InvalidValue("round_to_e8m0 requires finite positive input")
    if not was_np:
        return codes.reshape(x.shape)
    out = codes.cpu().numpy().reshape(arr.shape)
    return out if arr.ndim else out[()]


E8M0_DECODE = np.ldexp(1.0, np.arange(256) - 127)
E8M0_DECODE[255] = np.nan


def decode_e8m0(codes):
    """E8M0 codes -> 2^(code - 127); the NaN code 0xFF is rejected (codec.py:138-142)."""
    if isinstance(codes, torch.Tensor):
        if bool((codes == 0xFF).any()):
            raise InvalidValue("NaN E8M0 code cannot be used as a scale")
        return torch.as_tensor(E8M0_DECODE, device=codes.device)[codes.long()]
    c = np.asarray(codes, dtype=np.uint8)
    if np.any(c == 0xFF):
        raise InvalidValue("NaN E8M0 code cannot be used as a scale")
    return E8M0_DECODE[c]
