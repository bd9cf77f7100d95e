#!/bin/bash
# ncu captures of the inference forward kernel (K5) at C2 and C3 (GPU box).
mkdir -p gpurun_out/prof
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_infer -s 1 -c 1 -o gpurun_out/prof/k5_c3 \
    python scripts/time_fwd.py 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_infer -s 1 -c 1 -o gpurun_out/prof/k5_c2 \
    python scripts/time_fwd.py 0 > /dev/null 2>&1
ls -la gpurun_out/prof
