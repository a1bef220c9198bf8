python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in C3 C2; do for lv in 0 1 2 3; do for r in 1 2; do for mode in coop cluster; do
  if [ $mode = coop ]; then export MSK_NO_CLUSTER=1; else unset MSK_NO_CLUSTER; fi
  python tools/microbench.py --reps 2 --config $cfg --level $lv > gpurun_out/cl.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/cl.log').read().strip().splitlines()[-1]); print('$cfg', 'L$lv', '$mode', round(d['cg_ms'],3), d['cg_iters'])"
done; done; done; done
unset MSK_NO_CLUSTER
for cfg in C3 C2; do python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['config']['phase_ms']['solve_cg_per_level'])"; done
