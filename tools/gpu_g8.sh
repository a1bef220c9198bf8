set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g8_build.log 2>&1 || { echo build failed; tail gpurun_out/g8_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_rank_threads.py -q -p no:cacheprovider > gpurun_out/g8_dist.log 2>&1; echo dist_rc=$?; tail -4 gpurun_out/g8_dist.log
timeout 1200 python tools/c4_sweep.py --Tmax 6 --norms > gpurun_out/g8_c4.log 2>&1; echo c4_rc=$?; tail -7 gpurun_out/g8_c4.log | cut -c1-600
