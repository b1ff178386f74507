python tools/env_sweep.py --config c5a --check --rounds 2 --sets "A=1" > gpurun_out/sweep6.out 2>&1
PASGAL_BCC_LIB=paper_2404_17101_b200/lib/variants/lib_t3m4.so python tools/env_sweep.py --config c5a --rounds 1 --sets "A=1" >> gpurun_out/sweep6.out 2>&1
PASGAL_BCC_TAGS2=1 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tags2_tests_e.log 2>&1; echo "forced tags2 exit $?" >> gpurun_out/tags2_tests_e.log
