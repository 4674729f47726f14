mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest -x -q -m gpu tests > gpurun_out/t29.log 2>&1; echo tests=$?; tail -1 gpurun_out/t29.log
bash tools/exp_lib.sh tools/exp29.txt
