T=${TAG:-r02v}
for x in 0 1 2; do
TAGC_DS_BIN_SHIFT=$x timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($x, d['value'], d['ms_per_step'], d.get('stages_ms'))"
TAGC_DS_BIN_SHIFT=$x TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ds" --csv --log-file gpurun_out/${T}_ds$x.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_ds$x.csv | grep k_ds
done
timeout 300 python -m pytest tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py -q -x -p no:cacheprovider 2>&1 | tail -2
