#!/bin/bash
# GPU box: launch list (2 steps) + one `ncu --set full` capture of the decode frame_kernel launch.
# Usage: tools/ncu_capture.sh <tag> [bench args...]; outputs in gpurun_out/.
TAG=${1:-r02}; shift || true
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
export WFST_NO_BUILD=1
python -c "import bench; print(bench.kernel_source_sha())" > gpurun_out/prof_$TAG.sha
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/launches_bench_$TAG.log 2>&1
echo launches=$?
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 5 -c 1 \
    -o gpurun_out/prof_$TAG -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/prof_bench_$TAG.log 2>&1
echo prof=$?
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${TAG}_source.csv 2>/dev/null
ls -la gpurun_out/prof_$TAG*
