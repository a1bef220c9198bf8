#!/bin/bash
# matrix-free and C5 bench lines (one GPU call); outputs under gpurun_out/
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak | tee $O/fp64_peak.json
mkdir -p profiles && cp $O/fp64_peak.json profiles/fp64_peak.json
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --matrix-free > $O/bench_c3_mf.log 2>&1; echo c3mf_exit=$?
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo c5_exit=$?
timeout 1800 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --matrix-free > $O/bench_c5_mf.log 2>&1; echo c5mf_exit=$?
for f in bench_c3_mf bench_c5 bench_c5_mf; do tail -1 $O/$f.log | cut -c1-600; done
