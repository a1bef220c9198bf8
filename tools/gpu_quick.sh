#!/bin/bash
# quick GPU call: build, distributed tests, emulated partition timing, CG phase split, bench line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1 || { echo build failed; tail gpurun_out/q_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_rank_threads.py -q -x -p no:cacheprovider > gpurun_out/q_dist.log 2>&1; echo dist_rc=$?; tail -2 gpurun_out/q_dist.log
timeout 600 python tools/dist_emul_bench.py --worlds 1,2,8 > gpurun_out/q_emul.log 2>&1; echo emul_rc=$?; cut -c1-200 gpurun_out/q_emul.log
for lv in 5 4; do MSK_CG_PHASES=1 timeout 300 python tools/microbench.py --reps 1 --level $lv 2>&1 | grep -E "phases|cg_ms" | tail -2; done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/q_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['config']['phase_ms'])"
