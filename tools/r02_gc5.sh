#!/bin/bash
mkdir -p gpurun_out
STEPS=3 bash tools/exp_lib.sh tools/exp19.txt
for f in gc1 gc2 gc2b gc1o gc2o gc2bo; do python -c "import json;d=json.loads(open('gpurun_out/exp_$f.json').read().strip().splitlines()[-1]);print('$f', d['memory']['records_used_max_per_stream'])"; done
export WFST_NO_BUILD=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/p5_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --config c5 --partial > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/p5_launches.csv
