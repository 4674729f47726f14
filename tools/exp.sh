#!/bin/bash
# Run a list of bench variants on the GPU box: each line of $1 = "<tag> <bench args...>"
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
while read -r tag args; do
  [ -z "$tag" ] && continue
  timeout 600 python -u bench.py --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline $args \
     > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err
  echo "$tag rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/exp_$tag.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null)"
done < "$1"
