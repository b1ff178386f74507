ncu --set full --import-source on --clock-control none -k regex:"k_tags2_blk" -c 1 -o gpurun_out/full_t2 python tools/profile_run.py --config c5a --calls 1 > gpurun_out/ncu_full_t2.log 2>&1
ncu -i gpurun_out/full_t2.ncu-rep --page source --csv > gpurun_out/full_t2v1_source.csv 2>&1
ncu -i gpurun_out/full_t2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/full_t2v1_source_cuda.csv 2>&1
rm -f gpurun_out/full_t2.ncu-rep
