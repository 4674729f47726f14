#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py, one tool at a time; logs in gpurun_out/.
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()"
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 --error-exitcode 99 \
     python tools/sanitize_driver.py ${1:-all} > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"
  tail -4 gpurun_out/sanitize_$t.log
done
