#!/bin/bash
# Run on the GPU box (gpurun): launch lists + one full ncu capture per hot kernel.
set -x
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c2_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c4.csv \
    python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c4_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof/attn_fwd_c2 \
    python scripts/time_fwd.py 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof/attn_fwd_train_c4 \
    python scripts/time_fwd.py 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof/attn_bwd_c4 \
    python scripts/time_bwd.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quantize -s 2 -c 3 -o gpurun_out/prof/quantize_c2 \
    python scripts/time_quant.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fp4mm_kernel -s 1 -c 1 -o gpurun_out/prof/fp4mm_8k \
    python scripts/time_fp4mm.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_sage3_c2.csv \
    python scripts/prof_sage3.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 4 -c 1 -o gpurun_out/prof/attn_fwd_sage3_c2 \
    python scripts/prof_sage3.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/prof/attn_fwd_plain_c2 \
    python scripts/prof_plain.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_infer -c 1 -o gpurun_out/prof/attn_fwd_mx_c2 \
    python scripts/prof_mx.py > /dev/null 2>&1
ls -la gpurun_out/prof
