# A/B: list passes' CTA count; round-0 grid (one pass vs persistent).
B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step"
P='import json,sys; d=json.loads(sys.stdin.read()); g=d["extras"]["gpt2"]; print(d["value"], d["ms_per_step"], d["stages_ms"]["decode"], g["ms_per_step"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for r in 1 2; do
for v in "0 8" "1024 8" "0 0" "0 16" "1024 0"; do
  set -- $v
  echo -n "list_ctas=$1 r0=$2: "; TAGC_LIST_CTAS=$1 TAGC_R0_GRID=$2 timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"
done
done
