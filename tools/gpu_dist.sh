set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g5_build.log 2>&1 || { echo build failed; tail gpurun_out/g5_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_rank_threads.py -q -x -p no:cacheprovider > gpurun_out/g5_dist.log 2>&1; echo dist_rc=$?; tail -5 gpurun_out/g5_dist.log
timeout 600 python tools/dist_emul_bench.py > gpurun_out/g5_emul.log 2>&1; echo emul_rc=$?; cat gpurun_out/g5_emul.log | cut -c1-300
