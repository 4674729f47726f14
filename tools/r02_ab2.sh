#!/bin/bash
# radix digit fix A/B + per-frame cycle diagnostics
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
export WFST_NO_BUILD=1
cp paper_1910_10032_b200/libwfst_gpu.so /tmp/new.so
cp tools/libwfst_gpu_fc.so paper_1910_10032_b200/libwfst_gpu.so
timeout 600 python tools/frame_cycles.py c3 clean > gpurun_out/fc_clean.txt 2>&1
timeout 600 python tools/frame_cycles.py c3 other > gpurun_out/fc_other.txt 2>&1
cp /tmp/new.so paper_1910_10032_b200/libwfst_gpu.so
cat gpurun_out/fc_clean.txt gpurun_out/fc_other.txt
cat > /tmp/exp.txt <<'X'
new base --config c3
old base0 --config c3
newo base --config c3 --preset other
oldo base0 --config c3 --preset other
new2 base --config c3
old2 base0 --config c3
X
bash tools/exp_lib.sh /tmp/exp.txt
timeout 600 python -m pytest -x -q tests/test_gpu_layout.py tests/test_gpu_conventions.py tests/test_gpu_fuzz.py tests/test_gpu_hist.py > gpurun_out/ab2_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab2_pytest.log
