"""fp4mm correctness check for a tuning build (AQ_LIB_PATH): NVFP4 / MXFP4 against a torch fp64 product of the decoded operands."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402

torch.manual_seed(0)
for spec in (aq.NVFP4, aq.MXFP4):
    for M, N, K in ((256, 384, 512), (200, 130, 992), (1024, 1024, 4096), (300, 700, 1056), (128, 256, 64), (129, 257, 2048)):
        a, b = torch.randn(M, K, device="cuda"), torch.randn(N, K, device="cuda")
        qa, qb = aq.quantize(a, spec), aq.quantize(b, spec)
        c = aq.fp4mm(qa, qb)
        ref = aq.dequantize(qa).double() @ aq.dequantize(qb).double().T
        err = ((c.double() - ref).norm() / ref.norm()).item()
        print(spec.name if hasattr(spec, "name") else spec, M, N, K, f"rel {err:.2e}", "OK" if err < 1e-5 else "BAD")
