# A/B: fused-pass chunk claiming for small sketches (GPT-2) and chunk size at C4.
B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step"
P='import json,sys; d=json.loads(sys.stdin.read()); g=d["extras"]["gpt2"]; print(d["ms_per_step"], d["roofline"]["kernel_ms"], g["ms_per_step"], g["k_fused_tma_ms"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for r in 1 2; do
for v in "48 2" "0 2" "0 1" "0 4" "48 4"; do
  set -- $v
  echo -n "above=$1 chunk=$2: "; TAGC_FUSED_CHUNK_ABOVE_MB=$1 TAGC_FUSED_CHUNK=$2 timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"
done
done
