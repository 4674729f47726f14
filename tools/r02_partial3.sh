mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest -x -q tests/test_gpu_partial.py tests/test_gpu_gc.py tests/test_gpu_parity.py -k "partial or gc or c5 or reclaim" 2>&1 | tail -3
timeout 300 python tools/partial_split2.py c5 2>&1 | tail -2
timeout 600 python bench.py --config c5 --partial --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 partial', d['value'], d['ms_per_step'])"
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d['ms_per_step'])"
