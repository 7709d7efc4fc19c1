# Flake hunt: the parity suite three times, failures captured.
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 1200 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_scale.py tests/test_gpu_world.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py tests/test_gpu_acceptance.py tests/test_gpu_integration.py -m gpu -q -p no:cacheprovider --timeout 300 -rf > gpurun_out/r02am_tests_$i.log 2>&1
echo "run $i: $(tail -1 gpurun_out/r02am_tests_$i.log)"; grep -E "^FAILED" gpurun_out/r02am_tests_$i.log | head -5
done
