# ds_place at 2 CTAs/SM (256 threads, 4096-record batches).
mkdir -p gpurun_out
T=${TAG:-r02ab}
timeout 600 python -m pytest tests/test_gpu_scale.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -2
for i in 1 2; do timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'))"; done
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ds" --csv --log-file gpurun_out/${T}_ds.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_ds.csv | grep k_ds
