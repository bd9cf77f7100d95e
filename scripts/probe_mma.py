"""tcgen05 issue-rate / latency probes (GPU)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00040_b200 import _lib  # noqa: E402
lib = _lib.load()
st = torch.cuda.current_stream()
for kind, name, rounds in ((0, "nvf4 N256", 20000), (1, "bf16 N256", 5000), (2, "nvf4 N128", 20000),
                           (3, "nvf4 N128 + cp", 20000), (4, "nvf4 N128 round trip", 2000),
                           (5, "nvf4 N128 stream rnd", 20000), (6, "nvf4 N256 stream rnd", 20000),
                           (7, "nvf4 N128 stream 2acc+commit", 20000), (8, "nvf4 N256 same rnd", 20000),
                           (9, "bf16 N128 stream rnd", 20000), (10, "bf16 N256 stream rnd", 20000),
                           (11, "bf16 N64 stream rnd", 20000), (12, "nvf4 N64 stream rnd", 20000)):
    for ctas in (1, 148):
        lib.aq_probe_mma_peak(kind, ctas, rounds, st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.aq_probe_mma_peak(kind, ctas, rounds, st.cuda_stream)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        tf = lib.aq_probe_mma_flops(kind, ctas, rounds) / (ms * 1e-3) / 1e12
        print(f"{name:22s} ctas={ctas:3d}: {ms*1e6/rounds:8.1f} ns/instr  {tf:8.1f} TFLOP/s", flush=True)
