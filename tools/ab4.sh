python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_t.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['phase_ms'])"
bash tools/ab_variants.sh BASE3 PF
for r in 1 2; do for v in GM4B GM5 GM6; do MSK_LIB_PATH=ab/lib$v.so python tools/microbench.py --eval --reps 3 2>&1 | tail -1 | sed "s/^/$v /"; done; done
