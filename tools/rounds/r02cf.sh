mkdir -p gpurun_out
TAGC_DEBUG_PEEL=1 timeout 300 python tools/w8_decode_probe.py 8 2>&1 | grep "\[peel\]" | tail -3
timeout 300 python tools/w8_decode_probe.py 8 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms']['decode'], d['extras']['gpt2']['ms_per_step'], d['extras']['gpt2-paper']['ms_per_step'])"; done
