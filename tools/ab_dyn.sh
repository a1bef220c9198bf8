python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for lv in 5 4 3 2; do for r in 1 2; do
  for mode in static dyn; do
    if [ $mode = static ]; then export MSK_STATIC_CHUNKS=1; else unset MSK_STATIC_CHUNKS; fi
    python tools/microbench.py --reps 2 --level $lv > gpurun_out/dyn.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/dyn.log').read().strip().splitlines()[-1]); print('L$lv', '$mode', round(d['cg_ms'],3), round(d['cg_GBs'],1))"
  done; done; done
unset MSK_STATIC_CHUNKS
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_t.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['config']['phase_ms']['solve_cg_per_level'])"
