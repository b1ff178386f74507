#!/bin/bash
# Two-level tags: GPU parity with it forced on every graph, then A/B timings (stage ms).
tag=${1:-t2}
PASGAL_BCC_TAGS2=1 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tags2_tests_$tag.log 2>&1
echo "forced tags2 exit $?" >> gpurun_out/tags2_tests_$tag.log
for v in 0 1; do
  tools/c5a_quick.sh ${tag}_c5a_$v PASGAL_BCC_TAGS2=$v
  for c in c3 c4; do
    PASGAL_BCC_TAGS2=$v python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --no-checksum 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().splitlines()[-1]); print('$c tags2=$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['pipeline']['stage_ms'].items()})"
  done
done
