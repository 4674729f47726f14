#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/sweep_beam_${1:-x}.jsonl
: > $OUT
for beam in 10 15; do
for v in "1024 1" "512 2" "256 4"; do
  set -- $v
  timeout 300 python -u bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --threads $1 --ctas-per-sm $2 --beam $beam \
     2>/dev/null | tail -1 >> $OUT
done; done
echo done
