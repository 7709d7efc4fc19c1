# Round-2 checkpoint: full GPU suite, smoke, default bench line, reference arm, launch list.
mkdir -p gpurun_out
T=${TAG:-r02ac}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -4 gpurun_out/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo SMOKE_RC=$?; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo BENCH_RC=$?; tail -1 gpurun_out/${T}_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo REF_RC=$?; tail -1 gpurun_out/${T}_bench_ref.log | cut -c1-300
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches_summary.txt 2>&1; grep tagc gpurun_out/${T}_launches_summary.txt
