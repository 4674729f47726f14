#!/bin/bash
# e2e A/B: host staging buffers (3 vs 6) and H2D chunk size; bench lines with e2e, no CPU baseline.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
cp paper_1910_10032_b200/libwfst_gpu.so /tmp/base.so
export WFST_NO_BUILD=1
run() { tag=$1; lib=$2; shift 2
  if [ "$lib" = base ]; then cp /tmp/base.so paper_1910_10032_b200/libwfst_gpu.so; else cp tools/libwfst_gpu_$lib.so paper_1910_10032_b200/libwfst_gpu.so; fi
  timeout 600 python -u bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/e2e_$tag.json 2> gpurun_out/e2e_$tag.err
  echo "$tag $(python -c "import json; d=json.loads(open('gpurun_out/e2e_$tag.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], round(d['e2e']['ms_per_step'],2))")"; }
run a1 base
run b1 st6
run c1 base --chunk 10
run d1 st6 --chunk 10
run a2 base
run b2 st6
run e1 st6 --chunk 50
cp /tmp/base.so paper_1910_10032_b200/libwfst_gpu.so
