#!/bin/bash
# ab_variants.sh V1 V2 ...: finest-level CG timing (tools/microbench.py) with
# ab/libV.so for each variant, two alternating rounds, same box.
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for v in "$@"; do
    MSK_LIB_PATH=ab/lib$v.so python tools/microbench.py --reps 3 --config ${CFG:-C3} --level ${LEVEL:--1} > $O/abv_$v.log 2>&1
    python -c "import json,sys; d=json.loads(open('$O/abv_$v.log').read().strip().splitlines()[-1]); print('${CFG:-C3}', 'L${LEVEL:--1}', '$v', round(d['cg_ms'],3), round(d['cg_GBs'],1), d['cg_iters'])"
  done
done
