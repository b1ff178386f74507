python -m pytest tests/test_gpu_parity.py -x -q -k "kats or corpus or singles or hub or degenerate or leaf or two_level or c2 or c3" > gpurun_out/cmp_tests.log 2>&1; echo "exit $?" >> gpurun_out/cmp_tests.log
python tools/env_sweep.py --config c5a --check --rounds 2 --sets "A=1" > gpurun_out/exp6.out 2>&1
python tools/config_times.py c2 c3 c4 >> gpurun_out/exp6.out 2>&1
