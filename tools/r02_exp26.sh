mkdir -p gpurun_out
bash tools/exp_lib.sh tools/exp26.txt
