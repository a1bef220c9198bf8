#!/bin/bash
# A/B of the last-axis grid refinement (MSK_ZF = 1, 2, 4, 8) on C3 and C2 (bench
# lines) and C3 matrix-free, then the GPU suite at the default
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/zf_build.log 2>&1 || { echo build failed; tail gpurun_out/zf_build.log; exit 1; }
for cfg in C3 C2; do
  for z in 1 2 4 8; do
    MSK_ZF=$z timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/zf_${cfg}_$z.log 2>&1
    echo "$cfg zf=$z rc=$?"; tail -1 gpurun_out/zf_${cfg}_$z.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phase_ms']; print(round(d['ms_per_step'],3), round(d['value'],2), 'create', round(p['create'],3), 'asm', round(p['assemble'],3), 'B', round(p['solve_b_products'],3), 'eval', round(p['evaluate_kernel'],3), 'cg', round(p['solve_cg'],3))"
  done
done
for z in 1 4; do
  MSK_ZF=$z timeout 900 python bench.py --config C3 --matrix-free --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/zf_C3mf_$z.log 2>&1
  echo "C3mf zf=$z rc=$?"; tail -1 gpurun_out/zf_C3mf_$z.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phase_ms']; print(round(d['ms_per_step'],3), 'cg', [round(x,2) for x in p['solve_cg_per_level']])"
done
[ -z "${SKIP_TESTS:-}" ] && timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/zf_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/zf_pytest.log
