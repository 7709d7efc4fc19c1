mkdir -p gpurun_out
T=${TAG:-r02k}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_scale.py tests/test_gpu_bigworld.py tests/test_gpu_diag.py tests/test_gpu_world.py -m gpu -q -x -p no:cacheprovider --timeout 240 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -5 gpurun_out/${T}_gputest.log
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3"
for v in "X=1" "TAGC_DEFER_SCATTER_BYTES=1000000000000"; do echo "== $v"; env $v timeout 150 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d.get('decode_roofline',{}).get('span_ms'), d['roofline']['kernel_ms'], d['peel'])"; done
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches_summary.txt 2>&1; grep tagc gpurun_out/${T}_launches_summary.txt
