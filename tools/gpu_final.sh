#!/bin/bash
# Round-end style validation: build, GPU suite, smoke, bench line (20 steps, cpu baseline)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1 || { echo build failed; tail gpurun_out/f_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/f_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/f_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/f_bench.log | cut -c1-600
