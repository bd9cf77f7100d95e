"""Time the quantizer kernels on C2-sized tensors (GPU): achieved GB/s vs HBM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from paper_2603_00040_b200 import _lib  # noqa: E402

B, H, N, d = 4, 32, 8192, 128
x = torch.randn(B * H, N, d, device="cuda").bfloat16()
lib = _lib.load()
ws = torch.empty(lib.aq_attn_fwd_workspace_bytes(B * H, N, N, d, 0, 0), dtype=torch.uint8, device="cuda")
codes = torch.empty(B * H * N * d // 2, dtype=torch.uint8, device="cuda")
scales = torch.empty(B * H * N * d // 16, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


n = x.numel()
alg = n * 2 + n // 2 + n // 16
rows = t(lambda: lib.aq_quantize_rows(x.data_ptr(), 1, B * H, N, d, d, N * d, codes.data_ptr(),
                                      scales.data_ptr(), None, 0, 1.0, None, st))
cols = t(lambda: lib.aq_quantize_cols(x.data_ptr(), 1, B * H, N, d, d, N * d, codes.data_ptr(),
                                      scales.data_ptr(), None, 0, 1.0, None, st))
print(json.dumps({"rows_ms": rows, "rows_GBs": alg / rows / 1e6, "cols_ms": cols, "cols_GBs": alg / cols / 1e6,
                  "alg_bytes": alg}))
