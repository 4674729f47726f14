#!/bin/bash
# hub-after-drain: quick parity subset + A/B vs the committed build (tools/libwfst_gpu_base0.so)
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "insert_order or alpha_bound or c2_parity or tie_heavy or overflow or c3_full" tests/test_gpu_fuzz.py tests/test_gpu_layout.py tests/test_gpu_conventions.py > gpurun_out/ab1_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ab1_pytest.log
bash tools/ab_args.sh "--config c3" base0; mv gpurun_out/abm_base.json gpurun_out/ab1_new_clean.json; mv gpurun_out/abm_base0.json gpurun_out/ab1_old_clean.json
bash tools/ab_args.sh "--config c3 --preset other" base0; mv gpurun_out/abm_base.json gpurun_out/ab1_new_other.json; mv gpurun_out/abm_base0.json gpurun_out/ab1_old_other.json
for f in gpurun_out/ab1_*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read());print(d['value'],d['ms_per_step'],d['phase_share'])"); done
