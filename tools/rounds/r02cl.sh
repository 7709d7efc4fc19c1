mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_emit -c 20 --csv --log-file gpurun_out/r02cl_emit.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02cl_emit.csv 2>&1 | grep k_emit
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['extras']['gpt2']; print(d['value'], d['ms_per_step'], d['stages_ms']['decode'], g['ms_per_step'], g['owner_step']['fused_ms'])"; done
