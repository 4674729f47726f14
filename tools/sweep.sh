#!/bin/bash
# Variant sweep on the GPU box: one bench line per (threads, ctas_per_sm) setting.
mkdir -p gpurun_out
OUT=gpurun_out/sweep_${1:-x}.jsonl
: > $OUT
for v in "512 1" "256 2" "512 2" "256 3" "256 4" "1024 1" "256 1"; do
  set -- $v
  timeout 300 python -u bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --threads $1 --ctas-per-sm $2 \
     2>gpurun_out/sweep_err_$1_$2.log | tail -1 >> $OUT
done
echo sweep done
