# k_peel grid barrier with arrivals spread over 8 words.
mkdir -p gpurun_out
T=${TAG:-r02au}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_world.py tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/${T}_tests.log)"
timeout 200 python tools/w8_decode_probe.py 8 2>&1 | tail -1
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_peel" --log-file gpurun_out/${T}_w8.csv python tools/w8_decode_probe.py 8 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_w8.csv | grep k_peel
TAGC_DEBUG_PEEL=1 timeout 200 python tools/w8_decode_probe.py 8 2>&1 | grep "\[peel\]" | tail -3
