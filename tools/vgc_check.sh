#!/bin/bash
# VGC First-CC: GPU parity with the policy forced, then timings and launch lists
PASGAL_BCC_CC=vgc python -m pytest tests/test_gpu_parity.py -x -q -k "kats or corpus or singles or seed_inv or forest or chain or grid or c3 or repeated" > gpurun_out/vgc_tests_forced.log 2>&1
echo "forced vgc exit $?" >> gpurun_out/vgc_tests_forced.log
python tools/config_times.py c1 c3 c4 > gpurun_out/vgc_times.json 2>&1
for t in 256 4096; do PASGAL_BCC_VGC_TAU=$t python tools/config_times.py c3 c4 >> gpurun_out/vgc_times.json 2>&1; done
PASGAL_BCC_CC=vgc tools/launch_lists.sh ${1:-vgc} c3 c4
