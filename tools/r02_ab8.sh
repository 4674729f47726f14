#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
timeout 1500 python -m pytest -x -q tests/test_gpu_conventions.py tests/test_gpu_fuzz.py tests/test_gpu_hist.py tests/test_gpu_lattice.py tests/test_gpu_partial.py tests/test_gpu_parity.py -k "not c4 and not c5" > gpurun_out/ab8_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ab8_pytest.log
bash tools/exp_lib.sh tools/exp16.txt
