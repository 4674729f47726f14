mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest -x -q tests/test_gpu_fuzz.py tests/test_gpu_conventions.py 2>&1 | tail -2
bash tools/exp_lib.sh tools/exp23.txt
