#!/bin/bash
# quick C5a device timing (stage ms) for A/B runs: tools/c5a_quick.sh TAG [ENV=VAL ...]
tag=$1; shift
env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --no-checksum > gpurun_out/c5a_$tag.json 2> gpurun_out/c5a_$tag.err
python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/c5a_{t}.json").read().splitlines()[-1])
    print(t, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["pipeline"]["stage_ms"].items()})
except Exception as e:
    print(t, "failed", e, open(f"gpurun_out/c5a_{t}.err").read()[-2000:])
PY
