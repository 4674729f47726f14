#!/bin/bash
# Round-2 bench lines for every BASELINE config (one B200): outputs gpurun_out/cfg_<tag>.json
mkdir -p gpurun_out
python -c "from paper_1910_10032_b200 import build; build.build()" || exit 1
export WFST_NO_BUILD=1
run() { tag=$1; shift; timeout ${TO:-900} python -u bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline "$@" > gpurun_out/cfg_$tag.json 2> gpurun_out/cfg_$tag.err; echo "$tag rc=$? $(tail -1 gpurun_out/cfg_$tag.json | head -c 300)"; }
run c2 --config c2
run c3other --config c3 --preset other
run c3eps --config c3eps
run c2eps --config c2eps
run c4 --config c4
run c5 --config c5
run c5partial --config c5 --partial
run c5other_reclaim --config c5 --preset other --partial --reclaim
run c3lattice --config c3 --lattice 8
