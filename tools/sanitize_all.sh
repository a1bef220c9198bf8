#!/bin/bash
# compute-sanitizer over the hot path: memcheck, racecheck,
# synccheck, initcheck on C1 (every feature) and C2 / a C2 prefix.
# Summaries -> gpurun_out/sanitize_*.log
set -u
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, log name, args...
    local tool=$1 name=$2; shift 2
    timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py "$@" \
        > $OUT/sanitize_${name}.log 2>&1
    echo "$tool $name rc=$? $(grep -E 'ERROR SUMMARY|sanitize ok' $OUT/sanitize_${name}.log | tr '\n' ' ')"
}
run memcheck  memcheck_C1      C1 --thresh --multi
run memcheck  memcheck_C1_mf   C1 --mf
run memcheck  memcheck_C2      C2 --m-eval 20000
run memcheck  memcheck_C2_mf   C2P4 --mf
run synccheck synccheck_C1     C1 --thresh --multi
run synccheck synccheck_C2P4   C2P4
run racecheck racecheck_C1     C1 --thresh --multi
run racecheck racecheck_C1_mf  C1 --mf
run racecheck racecheck_C2P4   C2P4 --m-eval 2000
run initcheck initcheck_C1     C1 --thresh
