#!/bin/bash
# GPU box: DRAM bytes + duration of one decode frame_kernel launch (light ncu pass).
TAG=${1:-x}; shift || true
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
WFST_NO_BUILD=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:frame_kernel -s 5 -c 1 --csv --log-file gpurun_out/dram_$TAG.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/dram_bench_$TAG.log 2>&1
echo ncu=$?
grep -E "dram__bytes|gpu__time|sector_hit" gpurun_out/dram_$TAG.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
