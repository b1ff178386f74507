#!/bin/bash
# ruler-spacing sweep: bash tools/lr_sweep.sh "c4 c5a" "4 5 6"
for cfg in ${1:-c1 c2 c3}; do for sh in ${2:-2 3 4 5 6 7}; do
  r=$(PASGAL_BCC_LR_SHIFT=$sh python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['pipeline']['stage_ms']['listrank'])")
  echo "$cfg shift=$sh $r"
done; done
