#!/bin/bash
# A/B: bench the in-tree library and an alternative build (tools/libwfst_gpu_<tag>.so)
mkdir -p gpurun_out
TAG=$1; shift
export WFST_NO_BUILD=1
timeout 300 python -u bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 > gpurun_out/ab_base_$TAG.json
cp paper_1910_10032_b200/libwfst_gpu.so /tmp/base.so
cp tools/libwfst_gpu_$TAG.so paper_1910_10032_b200/libwfst_gpu.so
timeout 300 python -u bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 > gpurun_out/ab_alt_$TAG.json
cp /tmp/base.so paper_1910_10032_b200/libwfst_gpu.so
echo ab done
