# Round-0 entries per thread / list-write grid variants (C4).
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3"
for v in "X=1" "TAGC_R0_PER=4" "TAGC_R0_PER=1" "TAGC_LW_GRID=2" "TAGC_LW_GRID=8"; do echo "== $v"; env $v timeout 200 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'))"; done
