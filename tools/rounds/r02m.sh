# Round-2: sanitizer logs, W=8 / 1-bit decode baselines, C4 variants.
mkdir -p gpurun_out
T=${TAG:-r02m}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_workload.py > gpurun_out/${T}_sanitize_${tool}.log 2>&1; echo SAN_${tool}_RC=$?; tail -3 gpurun_out/${T}_sanitize_${tool}.log
done
timeout 300 python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8.log 2>&1; echo W8_RC=$?; tail -12 gpurun_out/${T}_w8.log
timeout 300 python tools/onebit_probe.py > gpurun_out/${T}_onebit.log 2>&1; echo ONEBIT_RC=$?; tail -12 gpurun_out/${T}_onebit.log
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3"
for v in "X=1" "TAGC_DEFER_SCATTER_BYTES=1000000000000" "TAGC_FUSED_EMIT=1"; do echo "== $v"; env $v timeout 150 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d.get('decode_roofline',{}).get('span_ms'), d['roofline']['kernel_ms'], d['peel'])"; done
