#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
export WFST_NO_BUILD=1
cp paper_1910_10032_b200/libwfst_gpu.so /tmp/new.so
cp tools/libwfst_gpu_fc.so paper_1910_10032_b200/libwfst_gpu.so
timeout 600 python tools/frame_cycles.py c3 clean > gpurun_out/fc2_clean.txt 2>&1; cat gpurun_out/fc2_clean.txt
cp /tmp/new.so paper_1910_10032_b200/libwfst_gpu.so
