#!/bin/bash
# ncu capture of k_patch on level 4 of C4F (1.25M patches, the dominant launch of the build)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pp_build.log 2>&1 || exit 1


timeout 2400 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_patch --launch-skip 2 -c 1 -o gpurun_out/pp_kpatch4 -f \
   python bench.py --config C4F --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/pp_ncu4.log 2>&1; echo ncu_rc=$?
