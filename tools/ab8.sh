python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for lv in 5 4 3 2 1; do LEVEL=$lv bash tools/ab_variants.sh BASE6 PRE; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_t.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'], d['config']['phase_ms'])"
