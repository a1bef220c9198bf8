#!/bin/bash
# A/B of the balanced (segmented) SpMV in k_cg (MSK_SEG=1) on C3, plus the oracle parity tests with it
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sg_build.log 2>&1 || { echo build failed; tail gpurun_out/sg_build.log; exit 1; }
for rep in 1 2; do
for v in 0 1; do
  MSK_SEG=$v timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sg_C3_$v.log 2>&1
  echo "C3 seg=$v rc=$?"; tail -1 gpurun_out/sg_C3_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],2), round(d['roofline']['frac'],4), [round(x,3) for x in d['config']['phase_ms']['solve_cg_per_level']], d['config']['cg_iters'])"
done
done
for v in 0 1; do MSK_SEG=$v MSK_CG_PHASES=1 timeout 300 python tools/microbench.py --reps 1 --level 5 2>&1 | grep -E "phases" | tail -1; done
MSK_SEG=1 timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -p no:cacheprovider -k "not matrix_free" > gpurun_out/sg_pytest.log 2>&1; echo seg_parity_rc=$?; tail -3 gpurun_out/sg_pytest.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "dist or rank or fuzz_partitioned or matrix_free" > gpurun_out/sg_dist.log 2>&1; echo dist_rc=$?; tail -3 gpurun_out/sg_dist.log
