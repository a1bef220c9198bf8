bash tools/ab_variants.sh BASE2 LB
CFG=C5 bash tools/ab_variants.sh C4096M2 LB4096 C8192M1
python -m pytest tests/test_gpu_matrix_free.py -x -q 2>&1 | tail -2
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --matrix-free > gpurun_out/bench_c3_mf2.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_c3_mf2.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['config']['phase_ms']['solve_cg_per_level'])"
