# k_peel: two frontier elements per lane, counter-mode round-1 frontier as local pairs.
mkdir -p gpurun_out
T=${TAG:-r02ae}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_scale.py tests/test_gpu_world.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -3 gpurun_out/${T}_gputest.log
TAGC_DEBUG_PEEL=1 timeout 200 python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8_peeldbg.log 2>&1; echo DBG_RC=$?; tail -10 gpurun_out/${T}_w8_peeldbg.log
timeout 200 python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8.log 2>&1; echo W8_RC=$?; tail -2 gpurun_out/${T}_w8.log
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_list|k_tile|k_r0|k_peel|k_final|k_emit" --log-file gpurun_out/${T}_w8_launches.csv python tools/w8_decode_probe.py 8 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_w8_launches.csv | grep k_
for i in 1 2; do timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'))"; done
