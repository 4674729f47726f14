#!/bin/bash
# bench the in-tree library and each tools/libwfst_gpu_<tag>.so with extra bench arguments:
#   tools/ab_args.sh "<bench args>" tag1 tag2 ...
mkdir -p gpurun_out
ARGS=$1; shift
export WFST_NO_BUILD=1
cp paper_1910_10032_b200/libwfst_gpu.so /tmp/base.so
timeout 300 python -u bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $ARGS 2>/dev/null | tail -1 > gpurun_out/abm_base.json
for TAG in "$@"; do
  cp tools/libwfst_gpu_$TAG.so paper_1910_10032_b200/libwfst_gpu.so
  timeout 300 python -u bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $ARGS 2>/dev/null | tail -1 > gpurun_out/abm_$TAG.json
done
cp /tmp/base.so paper_1910_10032_b200/libwfst_gpu.so
echo done
