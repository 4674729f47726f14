mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none -k regex:partial_root -s 6 -c 1 -o gpurun_out/proot python tools/partial_split2.py c5 > gpurun_out/proot.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none -k regex:partial_trace -s 6 -c 1 -o gpurun_out/ptrace python tools/partial_split2.py c5 > gpurun_out/ptrace.log 2>&1; echo ncu=$?
