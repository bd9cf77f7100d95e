"""Time fp4mm (C = A B^T, NVFP4 and MXFP4 QuantTensors on tcgen05) (GPU)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from paper_2603_00040_b200 import _lib  # noqa: E402

lib = _lib.load()
for spec, M, N, K in ((aq.NVFP4, 8192, 8192, 8192), (aq.NVFP4, 16384, 16384, 4096), (aq.NVFP4, 4096, 4096, 16384),
                      (aq.MXFP4, 8192, 8192, 8192)):
    a = torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda")
    qa, qb = aq.quantize(a, spec), aq.quantize(b, spec)
    fn = lib.aq_fp4mm_mx if spec == aq.MXFP4 else lib.aq_fp4mm
    ws = torch.empty(lib.aq_fp4mm_workspace_bytes(M, N, K), dtype=torch.uint8, device="cuda")
    c = torch.empty(M, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def f():
        fn(qa.codes.data_ptr(), qa.scales.data_ptr(), M, qb.codes.data_ptr(), qb.scales.data_ptr(), N, K,
                     c.data_ptr(), N, ws.data_ptr(), st)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"fp4mm {'MX' if spec == aq.MXFP4 else 'NV'}FP4 M{M} N{N} K{K}: {ms:.3f} ms  {2.0 * M * N * K / ms / 1e9:.0f} TF/s (incl. operand repack)", flush=True)
