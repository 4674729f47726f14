#!/bin/bash
# Multi-rank path of bench.py on a one-GPU box (gloo, both ranks on the one device): self-launch,
# per-rank decoding, max-over-ranks, result gather + rank-0 cross-check, with and without partials.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mr_build.log 2>&1; echo build=$?
export WFST_DIST_BACKEND=gloo WFST_NO_BUILD=1
timeout 900 python bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mr_c2.json 2> gpurun_out/mr_c2.err; echo c2=$?; tail -c 700 gpurun_out/mr_c2.json
timeout 900 python bench.py --gpus 2 --config c2 --partial --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mr_c2p.json 2> gpurun_out/mr_c2p.err; echo c2p=$?; tail -c 300 gpurun_out/mr_c2p.json
