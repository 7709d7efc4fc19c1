# Fused pass: persistent (0) vs non-persistent K tiles per CTA.
B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step"
P='import json,sys; d=json.loads(sys.stdin.read()); g=d["extras"]["gpt2"]; print(d["ms_per_step"], d["roofline"]["kernel_ms"], g["ms_per_step"], g["k_fused_tma_ms"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for r in 1 2; do
for k in 0 4 8 16; do
  echo -n "K=$k: "; TAGC_FUSED_TILES_PER_CTA=$k timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"
done
done
TAGC_FUSED_TILES_PER_CTA=8 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "codec or golden or exchange" 2>&1 | tail -1
