# k_peel with local (slot, entry) queues and a summing grid barrier: parity + W=8 decode probe + C4 line.
mkdir -p gpurun_out
T=${TAG:-r02p}
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_scale.py tests/test_gpu_world.py -m gpu -q -x -p no:cacheprovider --timeout 200 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -5 gpurun_out/${T}_gputest.log
TAGC_DEBUG_PEEL=1 timeout 200 python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8_peeldbg.log 2>&1; echo DBG_RC=$?; tail -12 gpurun_out/${T}_w8_peeldbg.log
timeout 200 python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8.log 2>&1; echo W8_RC=$?; tail -3 gpurun_out/${T}_w8.log
timeout 600 python -m pytest tests/test_gpu_bigworld.py tests/test_gpu_multirank.py tests/test_gpu_acceptance.py tests/test_gpu_diag.py -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/${T}_gputest2.log 2>&1; echo TEST2_RC=$?
tail -5 gpurun_out/${T}_gputest2.log
timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d.get('decode_roofline',{}).get('span_ms'), d['peel'])"
