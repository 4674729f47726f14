#!/bin/bash
# Run on the GPU box (under gpurun): launch list + one full ncu capture of the decode launch.
# Usage: tools/profile_gpu.sh <tag> [bench args...]
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out
mkdir -p $OUT
# every launch with its device time (cold-cache, serialised: compare shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $OUT/launches_bench_$TAG.log 2>&1
# full capture of one decode launch: launches per step = [init frame_kernel, decode frame_kernel]
ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 5 -c 1 \
    -o $OUT/prof_$TAG -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $OUT/prof_bench_$TAG.log 2>&1
echo done
