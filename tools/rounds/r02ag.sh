# Llama-3-8B layout: decode group size sweep (bytes per bucket = counter + residual).
for mb in 48 96 160 320; do
TAGC_DECODE_GROUP_MB=$mb timeout 600 python bench.py --workload llama3-8b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($mb, d['value'], d['ms_per_step'], d['stages_ms'], d['launches_per_step'] if 'launches_per_step' in d else d['gpu_launches'])"
done
