#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
export WFST_NO_BUILD=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/gc3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --config c3 --gc-frames 128 > gpurun_out/gc3_bench.log 2>&1; echo ncu=$?
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/gc3_launches.csv')))
hdr=None
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum': print(d['ID'], d['Kernel Name'][:40], d['Metric Value'], d.get('Metric Unit'))
P
