#!/bin/bash
# The round's record run on one GPU: bench line (value, e2e, cpu_baseline, clocks), reference
# arm, launch list and one full ncu capture of the decode launch.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -u bench.py > gpurun_out/record_bench_$TAG.log 2>&1; echo bench=$?
timeout 600 python -u bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/record_ref_$TAG.log 2>&1; echo ref=$?
timeout 900 bash tools/profile_gpu.sh $TAG > gpurun_out/record_prof_$TAG.txt 2>&1; echo prof=$?
# dram traffic of the decode launch for the bench line's roofline.traffic
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; d=dict(zip(h,rows[2]))
print(float(d['dram__bytes_read.sum'])*1e9 if False else d['dram__bytes_read.sum'], d['dram__bytes_write.sum'])
" > gpurun_out/record_traffic_$TAG.txt 2>&1
echo done
