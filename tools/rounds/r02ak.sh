# Nibble bucket counters in the decode's counter mode.
mkdir -p gpurun_out
T=${TAG:-r02ak}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_scale.py tests/test_gpu_world.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -2 | head -c 300
for v in "X=1" "X=1"; do
env $v timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d.get('stages_ms'))"
done
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_list|k_r0|k_peel" --csv --log-file gpurun_out/${T}_dec.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_dec.csv | grep k_
