#!/bin/bash
# k_patch sizing check (threshold tests + C4F build time) and the GPU suite
# against the device bounds-check build
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pb_build.log 2>&1 || { echo build failed; tail gpurun_out/pb_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_threshold.py -q -p no:cacheprovider > gpurun_out/pb_thresh.log 2>&1; echo thresh_rc=$?; tail -2 gpurun_out/pb_thresh.log
MSK_DEBUG_PATCH=1 timeout 900 python bench.py --config C4F --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/pb_c4f.log 2> gpurun_out/pb_c4f.err; echo c4f_rc=$?
tail -1 gpurun_out/pb_c4f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4F', round(d['ms_per_step'],1), d['config']['phase_ms']['assemble'], d['config']['phase_ms']['solve'])"
grep "patch level" gpurun_out/pb_c4f.err | tail -2
python -m paper_2503_04914_b200.build --bounds > gpurun_out/pb_bbuild.log 2>&1; echo bounds_build=$?
MSK_LIB_PATH=$PWD/paper_2503_04914_b200/libmsk_bounds.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
   -k "not fullsize and not parity_large" > gpurun_out/pb_bounds_pytest.log 2>&1; echo bounds_pytest_rc=$?
tail -3 gpurun_out/pb_bounds_pytest.log
grep -c "MSK_DASSERT" gpurun_out/pb_bounds_pytest.log
