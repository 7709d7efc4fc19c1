B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step"
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stages_ms"]["decode"], d["extras"]["gpt2"]["ms_per_step"])'
for r in 1 2; do for k in 3 2 1; do echo -n "emit/SM=$k: "; TAGC_EMIT_PER_SM=$k timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"; done; done
