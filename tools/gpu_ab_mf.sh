#!/bin/bash
# A/B of matrix-free SpMV variants (ab/lib*.so from tools/build_variant.sh): bench C2 / C3 --matrix-free
mkdir -p gpurun_out
for r in 1 2; do
for cfg in C2 C3; do
for v in "$@"; do
  MSK_LIB_PATH=ab/lib$v.so timeout 600 python bench.py --config $cfg --matrix-free --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mf_$v.log 2>&1
  tail -1 gpurun_out/mf_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$v', round(d['ms_per_step'],2), [round(x,2) for x in d['config']['phase_ms']['solve_cg_per_level']])" 2>&1 | tail -1
done; done; done
