# Deferred scatter in groups of <= 2^27 floats: parity + Llama threshold sweep + C4 line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py tests/test_gpu_exchange.py -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -2
for v in "X=1" "TAGC_DEFER_SCATTER_BYTES=16000000" "TAGC_DEFER_SCATTER_BYTES=8000000"; do
env $v timeout 600 python bench.py --workload llama3-8b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['kernel_ms'])"
done
for v in "X=1" "TAGC_DEFER_SCATTER_BYTES=8000000"; do
env $v timeout 300 python bench.py --workload gpt2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step --no-extras 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpt2 $v', d['value'], d['ms_per_step'], d['stages_ms'])"
done
timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'], d.get('stages_ms'))"
