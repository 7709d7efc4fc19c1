# Llama-3-8B layout: deferral threshold sweep.
for v in "X=1" "TAGC_DEFER_SCATTER_BYTES=0" "TAGC_DEFER_SCATTER_BYTES=16000000"; do
env $v timeout 600 python bench.py --workload llama3-8b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['kernel_ms'])"
done
