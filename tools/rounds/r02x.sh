# Deferred scatter on a side stream overlapping the decode list build (W=1).
mkdir -p gpurun_out
T=${TAG:-r02x}
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_world.py tests/test_gpu_scale.py tests/test_gpu_bigworld.py tests/test_gpu_overlap.py tests/test_gpu_optimizer.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -3 gpurun_out/${T}_gputest.log
for i in 1 2; do timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d['peel'])"; done
