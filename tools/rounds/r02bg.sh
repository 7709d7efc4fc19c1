# Round 0 split into probes (before the sketch is final) and gather.
mkdir -p gpurun_out
T=${TAG:-r02bg}
timeout 1200 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_world.py tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py tests/test_gpu_optimizer.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/${T}_tests.log)"
for v in 1 0 1 0; do
TAGC_SPLIT_R0=$v timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 split=$v', d['value'], d['ms_per_step'], d['stages_ms']['decode'])"
done
for v in "1 33554432" "0 33554432" "1 0" "0 0" "1 33554432" "1 0"; do set -- $v
TAGC_SPLIT_R0=$1 TAGC_DEFER_SCATTER_BYTES=$2 timeout 200 python bench.py --workload gpt2 --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpt2 split=$1 defer=$2', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['stages_ms']['decode'])"
done
