#!/bin/bash
# C4F build phase split (MSK_DEBUG_PATCH) + the patch parity tests
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pa_build.log 2>&1 || { tail gpurun_out/pa_build.log; exit 1; }
for rep in 1 2; do
MSK_DEBUG_PATCH=1 timeout 900 python bench.py --config C4F --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/pa_c4f.log 2> gpurun_out/pa_c4f.err; echo c4f_rc=$?
grep "patches (k_patch)" gpurun_out/pa_c4f.err | tail -3
tail -1 gpurun_out/pa_c4f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4F step', round(d['ms_per_step'],1), 'assemble', round(d['config']['phase_ms']['assemble'],1))"
done
timeout 1800 python -m pytest tests/test_gpu_threshold.py tests/test_gpu_fuzz.py tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/pa_pytest.log 2>&1; echo thresh_rc=$?; tail -2 gpurun_out/pa_pytest.log
