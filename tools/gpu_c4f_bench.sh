set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c19_build.log 2>&1 || exit 1
MSK_DEBUG_PATCH=1 timeout 900 python bench.py --config C4F --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c19.log 2> gpurun_out/c19.err; echo rc=$?
tail -1 gpurun_out/c19.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4F', round(d['ms_per_step'],1), d['config']['phase_ms']['assemble'], d['config']['phase_ms']['solve'])"
grep "factor build" gpurun_out/c19.err | tail -14
