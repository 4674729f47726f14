mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest -x -q tests/test_gpu_fuzz.py tests/test_gpu_conventions.py > gpurun_out/t25.log 2>&1; echo tests=$?; tail -1 gpurun_out/t25.log
bash tools/exp_lib.sh tools/exp25.txt
