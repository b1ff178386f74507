#!/bin/bash
# ncu launch lists (time + DRAM bytes per kernel) of one FAST-BCC call per config.
# usage: tools/launch_lists.sh TAG config...   (writes gpurun_out/launches_<config>_<TAG>.csv)
tag=$1; shift
for c in "$@"; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:'^k_|scan' --csv --log-file gpurun_out/launches_${c}_${tag}.csv \
      python tools/profile_run.py --config $c --calls 1 > gpurun_out/launches_${c}_${tag}.log 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_${c}_${tag}.csv > gpurun_out/launches_${c}_${tag}.txt 2>&1
done
