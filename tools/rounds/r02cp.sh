B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step --no-extras"
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"])'
for r in 1 2 3 4; do for k in 8 10; do echo -n "K=$k: "; TAGC_FUSED_TILES_PER_CTA=$k timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"; done; done
