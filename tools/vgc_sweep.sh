python tools/config_times.py c3 c4 > gpurun_out/vgcq.json 2>&1
PASGAL_BCC_CC=afforest python tools/config_times.py c3 c4 >> gpurun_out/vgcq.json 2>&1
for q in q512 q128; do PASGAL_BCC_LIB=paper_2404_17101_b200/lib/variants/lib_$q.so python tools/config_times.py c3 c4 >> gpurun_out/vgcq.json 2>&1; done
PASGAL_BCC_VGC_TAU=4096 python tools/config_times.py c3 c4 >> gpurun_out/vgcq.json 2>&1
PASGAL_BCC_CC=vgc tools/launch_lists.sh vgc4 c3
