# L2 persisting-window experiment on the direct sketch scatter (C4).
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3"
for v in "X=1" "TAGC_DEFER_SCATTER_BYTES=1000000000000" "TAGC_DEFER_SCATTER_BYTES=1000000000000 TAGC_L2_PERSIST_MB=64" "TAGC_DEFER_SCATTER_BYTES=1000000000000 TAGC_L2_PERSIST_MB=96" "TAGC_DEFER_SCATTER_BYTES=1000000000000 TAGC_L2_PERSIST_MB=120" "TAGC_DEFER_SCATTER_BYTES=1000000000000 TAGC_L2_PERSIST_MB=120 TAGC_GRAPHS=0"; do echo "== $v"; env $v timeout 200 $B 2>&1 | grep -E "^\[l2\]|^\{" | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('[l2]'): print(l.strip()); continue
    d=json.loads(l); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d['roofline']['kernel_ms'])"; done
