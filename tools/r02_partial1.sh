mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest -x -q tests/test_gpu_partial.py tests/test_gpu_gc.py tests/test_gpu_parity.py -k "partial or gc or c5 or reclaim" 2>&1 | tail -3
timeout 300 python tools/partial_split2.py c5 2>&1 | tail -2
timeout 300 python tools/partial_split.py c5 2>&1 | tail -2
for t in memcheck racecheck; do timeout 900 compute-sanitizer --tool $t --print-limit 20 --error-exitcode 99 python tools/sanitize_driver.py partial > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/san_$t.log; done
