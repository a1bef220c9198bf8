#!/bin/bash
# A/B of the register-cached patch CG (ab/lib*.so): C4F level patch times, then the threshold tests per variant
mkdir -p gpurun_out
for r in 1 2; do for v in "$@"; do
MSK_LIB_PATH=ab/lib$v.so MSK_DEBUG_PATCH=1 timeout 600 python bench.py --config C4F --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/pr_$v.log 2> gpurun_out/pr_$v.err
echo "$v $(grep 'patches (k_patch)' gpurun_out/pr_$v.err | tail -3 | awk '{print $(NF-1)}' | tr '\n' ' ') $(tail -1 gpurun_out/pr_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('assemble', round(d['config']['phase_ms']['assemble'],1))")"
done; done
for v in "$@"; do MSK_LIB_PATH=ab/lib$v.so timeout 900 python -m pytest tests/test_gpu_threshold.py -q -p no:cacheprovider 2>&1 | tail -1; done
