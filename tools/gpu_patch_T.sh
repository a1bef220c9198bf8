#!/bin/bash
# thresholded builds at T = 3 (R = 11) and T = 6 (R = 14): per-level patch times (MSK_DEBUG_PATCH), then the threshold tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for t in 3 6; do
MSK_DEBUG_PATCH=1 timeout 600 python bench.py --config C4F --threshold $t --patch-R $((t+8)) --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/pt$t.log 2> gpurun_out/pt$t.err
echo "T=$t"; grep -E "patches \(k_patch\)" gpurun_out/pt$t.err | tail -3
tail -1 gpurun_out/pt$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('assemble', round(d['config']['phase_ms']['assemble'],1))"
done
timeout 900 python -m pytest tests/test_gpu_threshold.py -q -p no:cacheprovider 2>&1 | tail -1
