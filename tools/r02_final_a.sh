#!/bin/bash
# Round-2 final evidence, part A: GPU tests, smoke, headline bench, reference arm, ncu capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fa_build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/fa_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/fa_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fa_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/fa_bench.json 2> gpurun_out/fa_bench.err; echo bench=$?; tail -c 600 gpurun_out/fa_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fa_ref.json 2> gpurun_out/fa_ref.err; echo ref=$?; tail -c 300 gpurun_out/fa_ref.json
bash tools/ncu_capture.sh r02f > gpurun_out/fa_ncu.log 2>&1; echo ncu=$?; tail -3 gpurun_out/fa_ncu.log
bash tools/ncu_dram.sh r02f > gpurun_out/fa_dram.log 2>&1; echo dram=$?; tail -4 gpurun_out/fa_dram.log
