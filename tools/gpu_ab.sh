set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g3_build.log 2>&1 || { echo build failed; tail gpurun_out/g3_build.log; exit 1; }
timeout 600 python tools/ab_gather.py --config C3 > gpurun_out/ab3_C3.log 2>&1; echo ab_C3=$?; tail -3 gpurun_out/ab3_C3.log
timeout 600 python tools/ab_gather.py --config C2 --mf --reps 2 > gpurun_out/ab3_C2mf.log 2>&1; echo ab_C2mf=$?; tail -3 gpurun_out/ab3_C2mf.log
timeout 600 python tools/ab_gather.py --config C3 --mf --m-eval 1000000 --reps 1 > gpurun_out/ab3_C3mf.log 2>&1; echo ab_C3mf=$?; tail -3 gpurun_out/ab3_C3mf.log
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_gather_w -c 1 -o gpurun_out/prof3_kgw -f python tools/microbench.py --reps 1 --eval > gpurun_out/prof3_kgw.log 2>&1; echo ncu_w=$?
