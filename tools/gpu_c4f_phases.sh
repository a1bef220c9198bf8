#!/bin/bash
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cf_build.log 2>&1 || exit 1
MSK_DEBUG_PATCH=1 timeout 900 python bench.py --config C4F --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cf.log 2> gpurun_out/cf.err; echo rc=$?
grep "factor build\|patch level" gpurun_out/cf.err | tail -16
