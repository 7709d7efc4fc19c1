# Round-2: remaining GPU tests, C4 launch list (cold, serialised), variant timings.
mkdir -p gpurun_out
T=${TAG:-r02h}
timeout 1500 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_multirank.py tests/test_gpu_optimizer.py tests/test_gpu_overlap.py tests/test_gpu_scale.py tests/test_gpu_world.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -8 gpurun_out/${T}_gputest.log
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches_summary.txt 2>&1; cat gpurun_out/${T}_launches_summary.txt
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3"
for v in "X=1" "TAGC_FUSED_EMIT=1" "TAGC_DEFER_SCATTER_BYTES=1000000000000" "TAGC_DECODE_FULL_STATE=1"; do echo "== $v"; env $v timeout 300 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stages_ms'), d.get('decode_roofline',{}).get('span_ms'), d['roofline']['kernel_ms'])"; done
