#!/bin/bash
# K11 (split-pass training forward): the C4 bench launch list and one full capture at C4
P=gpurun_out/prof
mkdir -p $P
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c4.csv \
    python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $P/bench_c4_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_qat -s 1 -c 1 -o $P/attn_fwd_train_c4 \
    python scripts/time_fwd.py 2 > /dev/null 2>&1
ls -la $P
