#!/bin/bash
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pp_build.log 2>&1 || exit 1
timeout 900 python bench.py --config C4F --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/pp_c4f.log 2>&1; echo c4f_rc=$?
tail -1 gpurun_out/pp_c4f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4F', round(d['ms_per_step'],1), d['config']['phase_ms']['assemble'])"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_patch --launch-skip 1 -c 1 -o gpurun_out/pp_kpatch -f \
   python bench.py --config C4F --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/pp_ncu.log 2>&1; echo ncu_rc=$?
