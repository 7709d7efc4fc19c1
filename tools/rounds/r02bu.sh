B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step"
P='import json,sys; d=json.loads(sys.stdin.read()); g=d["extras"]["gpt2"]; print(d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], g["ms_per_step"], g["k_fused_tma_ms"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for r in 1 2; do timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"; done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/density_sweep.py --steps 5 2>&1 | tail -6
