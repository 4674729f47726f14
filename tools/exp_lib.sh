#!/bin/bash
# Bench variants with alternative libraries: each line of $1 = "<tag> <lib|base> <bench args...>"
# (<lib> = tools/libwfst_gpu_<lib>.so built by tools/build_variant.sh).
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
cp paper_1910_10032_b200/libwfst_gpu.so /tmp/base.so
export WFST_NO_BUILD=1
while read -r tag lib args; do
  [ -z "$tag" ] && continue
  if [ "$lib" = base ]; then cp /tmp/base.so paper_1910_10032_b200/libwfst_gpu.so; else cp tools/libwfst_gpu_$lib.so paper_1910_10032_b200/libwfst_gpu.so; fi
  timeout 600 python -u bench.py --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline $args \
     > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err
  echo "$tag rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/exp_$tag.json').read().strip().splitlines()[-1]); c=d['counters_per_step']; f=c['frames']; print(d['value'], d['ms_per_step'], d['roofline']['frac'], 'cand', round(c['candidates']/f), 'ovf', round(c['overflow_inserts']/f,1))" 2>/dev/null)"
done < "$1"
cp /tmp/base.so paper_1910_10032_b200/libwfst_gpu.so
