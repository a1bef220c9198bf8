#!/bin/bash
# Round profiles: the bench line (exits 0 first), the launch list of the same
# command (ncu, serialised, cold), and full captures of the finest-level k_cg
# (traffic for bench's configuration) and of the evaluation k_gather.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/p2_build.log 2>&1 || exit 1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/p2_bench.log 2>&1; echo bench_exit=$?
tail -1 $OUT/p2_bench.log | cut -c1-400
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo plain_exit=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $OUT/p2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/p2_list.log 2>&1; echo list_exit=$?
# the finest level's k_cg launch of the first bench step (pruned: levels 0..5 -> the 6th)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cg --launch-skip 5 -c 1 \
    -o $OUT/p2_kcg -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/p2_kcg.log 2>&1; echo kcg_exit=$?
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:^k_gather$ -c 1 \
    -o $OUT/p2_kgather -f python tools/microbench.py --reps 1 --eval > $OUT/p2_kgather.log 2>&1; echo kgather_exit=$?
