mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"partial|best_path" -c 60 --csv --log-file gpurun_out/pl_launches.csv python tools/partial_split2.py c5 > gpurun_out/pl.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:partial_root -s 6 -c 1 -o gpurun_out/proot_f -f python tools/partial_split2.py c5 > gpurun_out/proot_f.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:partial_trace -s 6 -c 1 -o gpurun_out/ptrace_f -f python tools/partial_split2.py c5 > gpurun_out/ptrace_f.log 2>&1; echo ncu=$?
timeout 600 python tools/partial_split2.py c5 2>&1 | tail -2
