#!/bin/bash
# Round-2 GPU pass: tests + smoke + bench (C3 clean) + sanitizers + launch list + ncu capture.
mkdir -p gpurun_out
bash tools/gpu_check.sh
bash tools/sanitize.sh all
bash tools/ncu_capture.sh r02a
