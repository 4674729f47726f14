#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_gc.py > gpurun_out/gc1_pytest.log 2>&1; echo gc_pytest=$?; tail -15 gpurun_out/gc1_pytest.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 99 python tools/sanitize_driver.py gc > gpurun_out/gc1_memcheck.log 2>&1; echo memcheck=$?; tail -3 gpurun_out/gc1_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 99 python tools/sanitize_driver.py gc > gpurun_out/gc1_racecheck.log 2>&1; echo racecheck=$?; tail -3 gpurun_out/gc1_racecheck.log
export WFST_NO_BUILD=1
for a in "--config c3" "--config c3 --gc-frames 64" "--config c3 --preset other --gc-frames 64" "--config c5 --preset other --partial --reclaim --gc-frames 50"; do
  timeout 900 python -u bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $a > gpurun_out/gc1_bench.json 2> gpurun_out/gc1_bench.err; echo "$a rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/gc1_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['memory'])" 2>&1 | tail -2; tail -2 gpurun_out/gc1_bench.err
done
