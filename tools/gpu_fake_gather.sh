#!/bin/bash
# EXPERIMENT RECORD: the MSK_FAKE_GATHER timing build was removed after the measurement (profiles/r02_kcg_ab.txt); rerunning needs that variant back
mkdir -p gpurun_out
for r in 1 2; do for v in base fake; do
MSK_LIB_PATH=ab/lib$v.so MSK_CG_PHASES=1 timeout 300 python tools/microbench.py --reps 1 --level 5 > gpurun_out/fk_$v.log 2>&1
echo "$v: $(grep phases gpurun_out/fk_$v.log | tail -1)"; tail -1 gpurun_out/fk_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['cg_ms'],3), d['cg_iters'])"
done; done
