#!/bin/bash
# K5-only refresh of the round-2 profiles (GPU box): launch lists of the C2 / C3 bench
# commands and full captures of K5 at C2 and C3. Summaries: scripts/summarize_profiles.py r02
set -x
P=gpurun_out/prof
mkdir -p $P
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $P/bench_c2_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c3.csv \
    python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $P/bench_c3_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c4.csv \
    python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $P/bench_c4_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_infer -s 1 -c 1 -o $P/attn_fwd_c2 \
    python scripts/time_fwd.py 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_infer -s 1 -c 1 -o $P/attn_fwd_c3 \
    python scripts/time_fwd.py 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o $P/attn_fwd_train_c4 \
    python scripts/time_fwd.py 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o $P/attn_bwd_c4 \
    python scripts/time_bwd.py > /dev/null 2>&1
ls -la $P
