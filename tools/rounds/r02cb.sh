mkdir -p gpurun_out
T=r02cb
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "codec or golden or exchange or scale or multirank" 2>&1 | tail -1
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv 2>&1 | grep -E "list_write|list_count"
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms']['decode'], d['extras']['gpt2']['ms_per_step'])"; done
