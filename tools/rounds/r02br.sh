# Fused pass: claim prefetch (default) vs static ranges at C4.
B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step --no-extras"
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"])'
for r in 1 2 3; do
for v in 48 4096; do
  echo -n "above=$v: "; TAGC_FUSED_CHUNK_ABOVE_MB=$v timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"
done
done
