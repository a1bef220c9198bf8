#!/bin/bash
# One GPU call: plain bench (exit 0 first), the launch list of the same command,
# and full ncu captures of the two dominant kernels.  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/prof_build.log 2>&1 || exit 1
if [ -z "${SKIP_BENCH:-}" ]; then
python bench.py --steps 5 --warmup 3 > $OUT/prof_bench.log 2>&1; echo bench_exit=$?
tail -1 $OUT/prof_bench.log
fi
for lv in 5 4 3 2; do MSK_CG_PHASES=1 python tools/microbench.py --reps 1 --level $lv 2>&1 | grep -E "phases|cg_ms" | tail -2; done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo plain_exit=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/prof_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/prof_list.log 2>&1; echo list_exit=$?
ncu --set full --clock-control none --import-source on -k k_cg -c 1 -o $OUT/prof_kcg -f \
    python tools/microbench.py --reps 1 > $OUT/prof_kcg.log 2>&1; echo kcg_exit=$?
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:^k_gather$ -c 1 -o $OUT/prof_kgather -f \
    python tools/microbench.py --reps 1 --eval > $OUT/prof_kgather.log 2>&1; echo kgather_exit=$?
