#!/bin/bash
# EXPERIMENT RECORD: the MSK_CG_MAXB hook was removed after the measurement (profiles/r02_cg_ctas_ab.txt)
# CTAs per CG level capped (MSK_CG_MAXB): per-level CG time on C3 levels 2-5 (microbench) and C2
mkdir -p gpurun_out
for cfg in C3 C2; do for lv in 2 3 4 5; do for mb in 0 74 148 296; do
  MSK_CG_MAXB=$mb timeout 300 python tools/microbench.py --reps 3 --config $cfg --level $lv > gpurun_out/mb.log 2>&1
  tail -1 gpurun_out/mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'L$lv', 'maxb=$mb', round(d['cg_ms'],3), d['cg_iters'])"
done; done; done
