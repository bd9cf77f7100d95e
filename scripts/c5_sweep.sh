#!/bin/bash
# BASELINE config 5 on one GPU: H=32 d=128, B = 65536/N, fwd+bwd (the autograd QAT step), causal and
# non-causal, N = 1K..64K, through bench.py (one JSON line per point) -> gpurun_out/c5/*.json
mkdir -p gpurun_out/c5
for n in 1024 2048 4096 8192 16384 32768 65536; do
  for sfx in "" "-nc"; do
    timeout 600 python bench.py --config c5-$n$sfx --steps 3 --warmup 3 --no-extras --no-cpu-baseline \
      > gpurun_out/c5/c5-$n$sfx.json 2> gpurun_out/c5/c5-$n$sfx.err
  done
done
ls gpurun_out/c5
