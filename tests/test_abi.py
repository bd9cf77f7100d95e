"""CPU-side checks of the C ABI: the library loads and exports every symbol the
header declares, ctypes structs match the header field order, shims validate
like the reference (no compute without a GPU)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "attnqat_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|double|const char\*)\s+(aq_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2603_00040_b200 import _lib
    lib = _lib.load()
    names = _header_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.PROTOTYPES)
    assert lib.aq_abi_version() == 3


def test_struct_fields_match_header():
    from paper_2603_00040_b200 import _lib
    src = open(os.path.join(ROOT, "include", "attnqat_b200.h")).read()
    for struct, cls in (("AqFwdArgs", _lib.AqFwdArgs), ("AqBwdArgs", _lib.AqBwdArgs),
                        ("AqSage3Args", _lib.AqSage3Args)):
        body = re.search(r"typedef struct \{([^}]*)\}\s*" + struct, src, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        fields = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            names = [x.strip().lstrip("*") for x in re.sub(r"^(const\s+)?\w+\*?\s+", "", decl).split(",")]
            fields += [re.sub(r"^\*", "", x) for x in names]
        assert [f[0] for f in cls._fields_] == fields, struct


def test_status_strings():
    from paper_2603_00040_b200 import _lib
    lib = _lib.load()
    assert lib.aq_status_string(0) == b"ok"
    assert lib.aq_status_string(4) == b"missing O_prime"


def test_workspace_queries_reject_bad_dims():
    from paper_2603_00040_b200 import _lib
    lib = _lib.load()
    assert lib.aq_attn_fwd_workspace_bytes(1, 256, 256, 96, 1, 0) == 0
    assert lib.aq_attn_fwd_workspace_bytes(2, 256, 256, 64, 1, 1) > 0
    assert lib.aq_attn_bwd_workspace_bytes(2, 256, 256, 128) > 0
    assert lib.aq_attn_fwd_sage3_workspace_bytes(2, 256, 256, 64, 96, 128) == 0   # b_q must divide n_q
    assert lib.aq_attn_fwd_sage3_workspace_bytes(2, 256, 256, 128, 64, 128) > 0
    # the pass-1 segment-maxima scratch only when segments leave the 128-key tiles
    assert (lib.aq_attn_fwd_sage3_workspace_bytes(2, 256, 384, 64, 64, 48)
            > lib.aq_attn_fwd_sage3_workspace_bytes(2, 256, 384, 64, 64, 128))


def test_tile_config_validation_matches_reference():
    import paper_2603_00040_b200 as aq
    with pytest.raises(aq.TileError):
        aq.TileConfig(b_q=10, b_k=16).validate(32, 32, True)
    with pytest.raises(aq.TileError):
        aq.TileConfig(b_q=16, b_k=8).validate(32, 32, True)
    aq.TileConfig(b_q=16, b_k=8).validate(32, 8, True)  # single key tile may be ragged
    aq.TileConfig(b_q=200, b_k=200).validate(200, 200, True)


def test_bwd_variant_semantics():
    import paper_2603_00040_b200 as aq
    V = aq.BwdVariant
    assert [v.uses_o_prime for v in V] == [True, False, True, False]
    assert [v.fake_quantizes_p for v in V] == [True, True, False, False]


def test_no_cpu_fallback():
    import torch
    import paper_2603_00040_b200 as aq
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        aq.quantize(np.zeros((4, 16)))
    with pytest.raises(RuntimeError):
        aq.flash_forward_training(np.zeros((128, 64)), np.zeros((128, 64)), np.zeros((128, 64)),
                                  aq.TileConfig(b_q=128, b_k=128))


def test_kernel_head_dim_padding_rule():
    import paper_2603_00040_b200 as aq
    assert [aq.kernel_head_dim(d) for d in (16, 32, 48, 64, 80, 96, 112, 128)] == [64] * 4 + [128] * 4
    for bad in (8, 24, 136, 256):
        with pytest.raises(aq.InvalidValue):
            aq.kernel_head_dim(bad)


def test_instrument_tile_walk_matches_reference_skips():
    """flash.py:127-132, 154: fully masked tiles are skipped (right-aligned causal)."""
    import paper_2603_00040_b200 as aq
    from paper_2603_00040_b200.flash import _visited_tiles
    cfg = aq.TileConfig(b_q=16, b_k=16, causal=True)
    assert list(_visited_tiles(32, 32, cfg)) == [(0, 0), (1, 0), (1, 1)]
    assert list(_visited_tiles(32, 64, cfg)) == [(0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (1, 2), (1, 3)]
    assert len(list(_visited_tiles(32, 64, aq.TileConfig(b_q=16, b_k=16)))) == 8


def test_header_abi3_fields_default_to_reference_semantics():
    """ABI 3: every new field's zero value is the reference's behaviour (ctypes zero-initialises)."""
    from paper_2603_00040_b200 import _lib
    a = _lib.AqFwdArgs()
    assert (a.softmax_scale, a.q_scale, a.k_scale, a.v_scale, a.p_scale) == (0.0,) * 5
    assert a.nonfinite is None and a.pf_codes is None and a.pf_scales is None
    b = _lib.AqBwdArgs()
    assert b.p_scale == 0.0 and b.pf_codes is None
