set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g4_build.log 2>&1 || { echo build failed; tail gpurun_out/g4_build.log; exit 1; }
out=gpurun_out/br_sweep.log; : > $out
timeout 300 python tools/ab_gather.py --config C3 --reps 3 --child /tmp/x.npz >> $out 2>&1
for br in 0 1.2 1.6 2.0 2.5 4; do
  echo "BR=$br" >> $out
  MSK_GATHER_WARP=1 MSK_WS_BR=$br timeout 300 python tools/ab_gather.py --config C3 --reps 3 --child /tmp/x.npz >> $out 2>&1
done
timeout 300 python tools/ab_gather.py --config C2 --mf --reps 1 --child /tmp/x.npz >> $out 2>&1
for br in 0 1.5 2.5; do
  echo "BR=$br C2mf" >> $out
  MSK_GATHER_WARP=1 MSK_WS_BR=$br timeout 300 python tools/ab_gather.py --config C2 --mf --reps 1 --child /tmp/x.npz >> $out 2>&1
done
cat $out | cut -c1-260
