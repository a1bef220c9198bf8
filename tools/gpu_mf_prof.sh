#!/bin/bash
# ncu capture of one finest-level k_mf_spmv launch (CFG, default C2, --matrix-free)
mkdir -p gpurun_out
CFG=${CFG:-C2}
timeout 600 python bench.py --config $CFG --matrix-free --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/mfp_bench.log 2>&1
SKIP=$(tail -1 gpurun_out/mfp_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); it=d['config']['cg_iters']; print(sum(it)-it[-1]//2)")
echo skip=$SKIP
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_mf_spmv --launch-skip $SKIP -c 1 -o gpurun_out/mf_kmf -f \
   python bench.py --config $CFG --matrix-free --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/mf_ncu.log 2>&1; echo ncu_rc=$?
