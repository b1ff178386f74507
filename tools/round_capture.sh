#!/bin/bash
# Round-end evidence: GPU tests, the default bench line, the ncu launch list of a short
# bench run, and one --set full capture of the dominant kernel.  TAG names the outputs.
tag=${1:-r02}
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_$tag.log
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench exit $?" >> gpurun_out/bench_$tag.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench_$tag.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
    --no-per-config --no-checksum > gpurun_out/ncu_bench_$tag.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_tags2_blk|k_tags_blk|k_labels" -c 2 -o gpurun_out/full_$tag \
    python tools/profile_run.py --config c5a --calls 1 > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i gpurun_out/full_$tag.ncu-rep --page raw --csv > gpurun_out/full_${tag}_raw.csv 2>&1
ncu -i gpurun_out/full_$tag.ncu-rep --page details --csv > gpurun_out/full_${tag}_details.csv 2>&1
rm -f gpurun_out/full_$tag.ncu-rep
