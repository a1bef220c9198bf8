O=gpurun_out
for v in OLD NEW OLD NEW; do MSK_LIB_PATH=ab/lib$v.so python tools/microbench.py --reps 3 > $O/ab_$v.log 2>&1; echo $v $(tail -1 $O/ab_$v.log); done
python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests_exit=$?; tail -3 $O/gpu_tests.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_new.log 2>&1; echo bench_exit=$?
python -c "import json;d=json.loads(open('$O/bench_new.log').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['config']['cg_iters'],d['config']['phase_ms'])"
