# Experiment: output zero fill on a side stream + value scatter, instead of k_emit.
for v in 0 1 0 1; do
TAGC_EMIT_SCATTER=$v timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $v', d['value'], d['ms_per_step'], d.get('stages_ms'))"
done
for v in 0 1; do
TAGC_EMIT_SCATTER=$v timeout 200 python bench.py --workload gpt2 --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpt2 $v', d['value'], d['ms_per_step'], d.get('stages_ms'))"
done
TAGC_EMIT_SCATTER=1 timeout 600 python -m pytest tests/test_gpu_world.py tests/test_gpu_exchange.py tests/test_gpu_scale.py -q -x -p no:cacheprovider 2>&1 | tail -1
