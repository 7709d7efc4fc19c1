# racecheck of the fused pass: persistent vs non-persistent grids (is the TMA-stage hazard a cross-CTA shared-memory reuse artefact?)
mkdir -p gpurun_out
for k in 0 8 1000000; do
  TAGC_FUSED_TILES_PER_CTA=$k timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize_workload.py > gpurun_out/r02bx_race_k$k.log 2>&1
  echo "K=$k: $(tail -1 gpurun_out/r02bx_race_k$k.log)"
done
