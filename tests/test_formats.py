"""ATNQ / ATQ4 file formats (tensors.py:122-220 of the reference): files written
by the reference load identically, our writer reproduces them byte for byte,
and malformed files raise FormatError with an offset (test_tensors.py:155-203)."""

import os

import numpy as np
import pytest

from paper_2603_00040_b200 import load_quant_tensor, load_tensor, save_quant_tensor, save_tensor
from paper_2603_00040_b200.codec import NVFP4, QuantTensor
from paper_2603_00040_b200.errors import FormatError, ShapeError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fx():
    return np.load(os.path.join(GOLD, "formats.npz"))


@pytest.mark.parametrize("name,key", [("ref_t32.atnq", "t32"), ("ref_t64.atnq", "t64")])
def test_reference_tensor_files_load_and_rewrite_identically(tmp_path, fx, name, key):
    src = os.path.join(GOLD, name)
    x = load_tensor(src)
    assert x.dtype == fx[key].dtype
    np.testing.assert_array_equal(x, fx[key])
    out = tmp_path / name
    save_tensor(x, out)
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("name", ["ref_q.atq4", "ref_kv.k.atq4", "ref_kv.vt.atq4"])
def test_reference_quant_files_rewrite_identically(tmp_path, name):
    src = os.path.join(GOLD, name)
    qt = load_quant_tensor(src)
    assert qt.spec == NVFP4
    assert qt.codes.shape == (qt.rows, qt.cols // 2) and qt.scales.shape == (qt.rows, qt.cols // 16)
    out = tmp_path / name
    save_quant_tensor(qt, out)
    assert out.read_bytes() == open(src, "rb").read()


def test_quant_matches_oracle_codec(fx):
    from oracle import nvfp4_attn_oracle as orc
    qt = load_quant_tensor(os.path.join(GOLD, "ref_q.atq4"))
    codes, scales = orc.quantize(fx["qsrc"])
    np.testing.assert_array_equal(qt.codes, codes)
    np.testing.assert_array_equal(qt.scales, scales)


def test_truncation_and_magic(tmp_path):
    data = open(os.path.join(GOLD, "ref_t32.atnq"), "rb").read()
    p = tmp_path / "t.atnq"
    for cut in (3, 8, 12, len(data) - 5):
        p.write_bytes(data[:cut])
        with pytest.raises(FormatError) as exc:
            load_tensor(p)
        assert exc.value.offset is not None
    p.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(FormatError):
        load_tensor(p)
    p.write_bytes(data + b"\0")
    with pytest.raises(FormatError) as exc:
        load_tensor(p)
    assert exc.value.offset == len(data)
    q = open(os.path.join(GOLD, "ref_q.atq4"), "rb").read()
    p.write_bytes(q[:-1])
    with pytest.raises(FormatError):
        load_quant_tensor(p)
    bad = bytearray(q)
    bad[8] = 7     # unknown scale format
    p.write_bytes(bytes(bad))
    with pytest.raises(FormatError):
        load_quant_tensor(p)


def test_write_validation(tmp_path):
    with pytest.raises(FormatError):
        save_tensor(np.zeros(3, dtype=np.int32), tmp_path / "x")
    with pytest.raises(ShapeError):
        save_tensor(np.zeros((1, 1, 1, 1), dtype=np.float32), tmp_path / "x")
    with pytest.raises(ShapeError):
        save_quant_tensor(QuantTensor(2, 32, NVFP4, np.zeros((2, 8), np.uint8), np.zeros((2, 2), np.uint8)),
                          tmp_path / "x")
