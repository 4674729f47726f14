#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_conventions.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py -k "not c4 and not c5 and not c3_full" > gpurun_out/ab4_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab4_pytest.log
bash tools/exp_lib.sh $1
