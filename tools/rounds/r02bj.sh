# High-load decode A/B: warp-aggregated peel overflow pushes, full state clear (auto vs off).
mkdir -p gpurun_out
for t in 90 95 98; do
  for z in 0 1; do
    echo "theta=$t zero_state=$z"; TAGC_DECODE_ZERO_STATE=$z TAGC_DEBUG_PEEL=1 timeout 300 python tools/density_sweep.py --steps 1 --theta $t 2>&1 | tail -2 | cut -c1-600
  done
done
timeout 900 python tools/density_sweep.py --steps 5 > gpurun_out/r02bj_density_sweep.jsonl 2>&1; cat gpurun_out/r02bj_density_sweep.jsonl
