#!/bin/bash
# Round-2 final evidence (session 3 build): GPU tests, smoke, headline bench, reference arm, every config.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fc_build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fc_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/fc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/fc_smoke.log
export WFST_NO_BUILD=1
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo bench=$?; tail -c 400 gpurun_out/fc_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; echo ref=$?; tail -c 300 gpurun_out/fc_ref.json
run() { tag=$1; shift; timeout ${TO:-900} python -u bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline "$@" > gpurun_out/cfg_$tag.json 2> gpurun_out/cfg_$tag.err; echo "$tag rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/cfg_$tag.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1)"; }
run c1 --config c1
run c2 --config c2
run c2eps --config c2eps
run c3other --config c3 --preset other
run c3eps --config c3eps
run c4 --config c4
run c5 --config c5
run c5partial --config c5 --partial
run c5other_gc --config c5 --preset other --partial --reclaim --gc-frames 50
run c3gc128 --config c3 --gc-frames 128
run c3lattice --config c3 --lattice 8
run c3hist --config c3 --hist
