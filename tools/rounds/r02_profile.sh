# Round-2 capture: GPU suite, C4 launch list (cold, serialised), one ncu --set full of the decode + select chain.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo TEST_RC=$?
tail -5 gpurun_out/${TAG}_gputest.log
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1; cat gpurun_out/${TAG}_launches_summary.txt
