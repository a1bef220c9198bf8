#!/bin/bash
# NVTX ranges visible to the profiler: ncu captures a k_cg launch only inside msk_solve range,
# and the finest level's CG inside "level 2/CG" of a 3-level run
mkdir -p gpurun_out
timeout 600 ncu --nvtx --nvtx-include "msk_solve/" --kernel-name-base function -k k_cg -c 1 --metrics gpu__time_duration.sum \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/nvtx1.log 2>&1; echo rc=$?
grep -E "k_cg|NVTX|msk_solve|gpu__time" gpurun_out/nvtx1.log | head -8
timeout 600 ncu --nvtx --nvtx-include "msk_solve/level 2/CG/" --kernel-name-base function -k k_cg --metrics gpu__time_duration.sum \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/nvtx2.log 2>&1; echo rc=$?
grep -cE "k_cg" gpurun_out/nvtx2.log
