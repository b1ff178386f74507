#!/bin/bash
# repeat bench runs to catch intermittent failures; usage: tools/stress.sh CONFIG RUNS
cfg=${1:-c4}; runs=${2:-5}
for i in $(seq 1 $runs); do
  PASGAL_BCC_DEBUG=1 timeout 600 python bench.py --config $cfg --steps 4 --warmup 2 --no-e2e --no-cpu-baseline > /tmp/s.json 2> /tmp/s.err
  rc=$?
  echo "$cfg run $i rc=$rc $(grep -h 'pasgal_bcc:' /tmp/s.err | head -2)"
done
