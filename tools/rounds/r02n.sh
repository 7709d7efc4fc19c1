# Device-resident ordered peel: parity subset + 1-bit probe.
mkdir -p gpurun_out
T=${TAG:-r02n}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_diag.py tests/test_gpu_acceptance.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -15 gpurun_out/${T}_gputest.log
timeout 300 python tools/onebit_probe.py > gpurun_out/${T}_onebit.log 2>&1; echo ONEBIT_RC=$?; tail -4 gpurun_out/${T}_onebit.log
