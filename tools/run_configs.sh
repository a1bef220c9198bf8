#!/bin/bash
# every BASELINE config (and mode) once: one bench line each -> gpurun_out/configs.jsonl
O=gpurun_out; : > $O/configs.jsonl
for a in "C1" "C2" "C3 --schedule literal" "C4" "C4F" "C5" "C5 --matrix-free" "C3 --matrix-free"; do
  set -- $a
  timeout 1200 python bench.py --config $a --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $O/configs.jsonl
  echo "$a exit=$?"
done
