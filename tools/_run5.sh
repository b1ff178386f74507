python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r5.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_r5.log
PASGAL_BCC_CC=vgc python -m pytest tests/test_gpu_parity.py -x -q -k "kats or corpus or singles or seed_inv or forest or chain or grid or c3 or repeated" > gpurun_out/vgc_tests_r5.log 2>&1; echo "forced vgc exit $?" >> gpurun_out/vgc_tests_r5.log
python tools/env_sweep.py --config c5a --check --rounds 2 --sets "A=1" > gpurun_out/sweep5.out 2>&1
python tools/config_times.py c1 c2 c3 c4 >> gpurun_out/sweep5.out 2>&1
