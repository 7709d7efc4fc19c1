# A/B: defer every sketch (pure-stream fused pass, non-persistent) at GPT-2 and the Llama layout.
P='import json,sys; d=json.loads(sys.stdin.read()); g=d["extras"]["gpt2"]; print(d["ms_per_step"], g["ms_per_step"], g["k_fused_tma_ms"], g["stages_ms"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for v in 33554432 0 4194304; do
  echo -n "defer>$v gpt2: "; TAGC_DEFER_SCATTER_BYTES=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "$P"
done
PL='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["stages_ms"])'
for v in 33554432 0 16777216; do
  echo -n "defer>$v llama: "; TAGC_DEFER_SCATTER_BYTES=$v timeout 900 python bench.py --workload llama3-8b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "$PL"
done
