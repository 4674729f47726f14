#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_gc.py tests/test_gpu_partial.py > gpurun_out/gc2_pytest.log 2>&1; echo gc_pytest=$?; tail -2 gpurun_out/gc2_pytest.log
export WFST_NO_BUILD=1
for a in "--config c3 --gc-frames 64" "--config c3 --gc-frames 128" "--config c3 --preset other --gc-frames 128" "--config c5 --preset other --partial --reclaim --gc-frames 50"; do
  timeout 900 python -u bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $a > gpurun_out/gc2_bench.json 2> gpurun_out/gc2_bench.err; echo "$a rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/gc2_bench.json').read().strip().splitlines()[-1]);m=d['memory'];print(d['value'],d['ms_per_step'],m['decoder_device_bytes']/1e9,m['records_used_max_per_stream'])" 2>&1 | tail -2; tail -2 gpurun_out/gc2_bench.err
done
