#!/bin/bash
# The paper's workloads (Table 1 grids, Figure 4): L = 11..14, both schedules,
# assembled and matrix-free (the paper's mode).  One JSON line per run ->
# gpurun_out/paper_runs.jsonl
set -u
mkdir -p gpurun_out
out=gpurun_out/paper_runs.jsonl
: > $out
for L in ${LEVELS:-11 12 13 14}; do
  for mf in "" "--matrix-free"; do
    for sch in pruned literal; do
      timeout 900 python tools/paper_run.py --levels $L --schedule $sch $mf >> $out 2> gpurun_out/paper_run_err.log
      echo "L=$L $sch ${mf:-assembled} rc=$?"
    done
  done
done
