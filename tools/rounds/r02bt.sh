# Fused pass K (tiles per CTA) at the Llama-3-8B layout and GPT-2 with larger K.
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["stages_ms"])'
for k in 0 8 16; do
  echo -n "llama K=$k: "; TAGC_FUSED_TILES_PER_CTA=$k timeout 900 python bench.py --workload llama3-8b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "$P"
done
P2='import json,sys; d=json.loads(sys.stdin.read()); g=d["extras"]["gpt2"]; print(g["ms_per_step"], g["k_fused_tma_ms"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for k in 0 32 64; do
  echo -n "gpt2 K=$k: "; TAGC_FUSED_TILES_PER_CTA=$k timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "$P2"
done
