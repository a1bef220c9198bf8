#!/bin/bash
# A/B of k_cg's L2 prefetch of the next chunk's gathered r windows (MSK_RPREF=0 vs default)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rp_build.log 2>&1 || { echo build failed; tail gpurun_out/rp_build.log; exit 1; }
for rep in 1 2; do
for cfg in C3 C2; do
  for v in 0 1; do
    MSK_RPREF=$v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rp_${cfg}_$v.log 2>&1
    echo "$cfg rpref=$v rc=$?"; tail -1 gpurun_out/rp_${cfg}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],2), round(d['roofline']['frac'],4), [round(x,3) for x in d['config']['phase_ms']['solve_cg_per_level']])"
  done
done
done
for v in 0 1; do MSK_RPREF=$v MSK_CG_PHASES=1 timeout 300 python tools/microbench.py --reps 1 --level 5 2>&1 | grep -E "phases" | tail -1; done
