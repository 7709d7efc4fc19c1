# k_peel CTA-local rounds (acq_rel decrements) vs grid rounds.
mkdir -p gpurun_out
T=${TAG:-r02as}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_world.py tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/${T}_tests.log)"
for v in 1 0; do
echo "== TAGC_PEEL_LOCAL=$v"
TAGC_PEEL_LOCAL=$v timeout 200 python tools/w8_decode_probe.py 8 2>&1 | tail -1
TAGC_PEEL_LOCAL=$v TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_peel" --log-file gpurun_out/${T}_w8_$v.csv python tools/w8_decode_probe.py 8 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_w8_$v.csv | grep k_peel
TAGC_PEEL_LOCAL=$v timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d['peel'])"
done
TAGC_DEBUG_PEEL=1 timeout 200 python tools/w8_decode_probe.py 8 2>&1 | grep "\[peel\]" | tail -4
