#!/bin/bash
# A/B of k_gather variants (ab/lib*.so): C3 bench phases (B products, evaluation kernel) and C2
mkdir -p gpurun_out
for r in 1 2; do for cfg in C3 C2; do for v in "$@"; do
  MSK_LIB_PATH=ab/lib$v.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ag_$v.log 2>&1
  tail -1 gpurun_out/ag_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phase_ms']; print('$cfg', '$v', round(d['ms_per_step'],2), 'B', round(p['solve_b_products'],3), 'eval', round(p['evaluate_kernel'],3))" 2>&1 | tail -1
done; done; done
