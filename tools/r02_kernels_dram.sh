#!/bin/bash
# DRAM bytes and duration of every non-frame kernel of the final build (light ncu pass, -c bounded).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/kd_build.log 2>&1; echo build=$?
export WFST_NO_BUILD=1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"best_path|settle_reset" -c 6 --csv --log-file gpurun_out/kd_bp.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/kd_bp.log 2>&1; echo bp=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"lattice" -c 6 --csv --log-file gpurun_out/kd_lat.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --lattice 8 > gpurun_out/kd_lat.log 2>&1; echo lat=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"gc_kernel" -c 6 --csv --log-file gpurun_out/kd_gc.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --gc-frames 128 > gpurun_out/kd_gc.log 2>&1; echo gc=$?
