#!/bin/bash
# transpose index with warp-aggregated atomics (MSK_CSC_AGG=1, default) vs per-entry atomics: C4F phases, then tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for r in 1 2; do for v in 0 1; do
MSK_CSC_AGG=$v MSK_DEBUG_PATCH=1 timeout 600 python bench.py --config C4F --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/csc$v.log 2> gpurun_out/csc$v.err
echo "agg=$v $(grep 'transpose index' gpurun_out/csc$v.err | tail -1)"; tail -1 gpurun_out/csc$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  C4F', round(d['ms_per_step'],1), 'assemble', round(d['config']['phase_ms']['assemble'],1))"
done; done
timeout 1500 python -m pytest tests/test_gpu_threshold.py tests/test_gpu_diagnostics.py tests/test_gpu_fuzz.py -q -p no:cacheprovider 2>&1 | tail -1
