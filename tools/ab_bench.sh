#!/bin/bash
# ab_bench.sh V1 V2 ...: bench.py phase times with ab/libV.so, alternating, same box
for r in 1 2; do for v in "$@"; do
  MSK_LIB_PATH=ab/lib$v.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abb_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abb_$v.log').read().strip().splitlines()[-1]);p=d['config']['phase_ms'];print('$v', round(d['ms_per_step'],2), 'create', round(p['create'],2), 'assemble', round(p['assemble'],2), 'B', round(p['solve_b_products'],2), 'eval', round(p['evaluate'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"
done; done
