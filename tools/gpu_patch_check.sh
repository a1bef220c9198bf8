set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p16_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_threshold.py tests/test_gpu_dist.py -q -p no:cacheprovider -k "patch or thresholded" > gpurun_out/p16_thresh.log 2>&1; echo thresh_rc=$?; tail -2 gpurun_out/p16_thresh.log
timeout 900 python bench.py --config C4F --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p16_c4f.log 2>&1; echo c4f_rc=$?
tail -1 gpurun_out/p16_c4f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4F', round(d['ms_per_step'],1), d['config']['phase_ms']['assemble'])"
