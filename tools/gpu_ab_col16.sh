#!/bin/bash
# A/B of k_cg's 16-bit column stream (MSK_COL16=0 vs default) on C3 and C2, then the GPU suite
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c16_build.log 2>&1 || { echo build failed; tail gpurun_out/c16_build.log; exit 1; }
for cfg in C3 C2; do
  for v in 0 1; do
    MSK_COL16=$v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c16_${cfg}_$v.log 2>&1
    echo "$cfg col16=$v rc=$?"; tail -1 gpurun_out/c16_${cfg}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],2), round(d['roofline']['frac'],4), [round(x,3) for x in d['config']['phase_ms']['solve_cg_per_level']])"
  done
done
for lv in 5 4; do MSK_CG_PHASES=1 timeout 300 python tools/microbench.py --reps 1 --level $lv 2>&1 | grep -E "phases" | tail -1; done
[ -z "${SKIP_TESTS:-}" ] && timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:-} > gpurun_out/c16_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/c16_pytest.log
