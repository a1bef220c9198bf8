#!/bin/bash
# One GPU call: build, A/B of the matrix-free kernel sums (bitwise + timing),
# the GPU test suite, and a short bench line.  Logs in gpurun_out/.
set -u
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/host_cores.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1 || { echo build failed; tail gpurun_out/g_build.log; exit 1; }
if [ -z "${SKIP_AB:-}" ]; then
timeout 600 python tools/ab_gather.py --config C3 > gpurun_out/ab_C3.log 2>&1; echo ab_C3=$?; cat gpurun_out/ab_C3.log | tail -4
timeout 600 python tools/ab_gather.py --config C3 --mf --m-eval 1000000 --reps 1 > gpurun_out/ab_C3mf.log 2>&1; echo ab_C3mf=$?; tail -3 gpurun_out/ab_C3mf.log
timeout 600 python tools/ab_gather.py --config C2 --mf --reps 2 > gpurun_out/ab_C2mf.log 2>&1; echo ab_C2mf=$?; tail -3 gpurun_out/ab_C2mf.log
fi
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:-} > gpurun_out/g_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/g_pytest.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/g_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/g_bench.log | cut -c1-3000
