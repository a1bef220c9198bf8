#!/bin/bash
# EXPERIMENT RECORD: the symmetric fill was removed after the measurement (profiles/r02_count_sym_ab.txt); MSK_COUNT_SYM now switches the count only
# symmetric fill (default) vs the row-by-row fill (MSK_COUNT_SYM=0 turns both off): C3 / C2 create + assemble; then the suites
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for r in 1 2; do for c in C3 C2; do for v in 0 1; do
  MSK_COUNT_SYM=$v timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phase_ms']; print('$c', 'sym=$v', round(d['ms_per_step'],2), 'create', round(p['create'],3), 'assemble', round(p['assemble'],3))"
done; done; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
