# Density sweep on the current build (C4 bucket, theta 99.9 .. 90) and a theta=90 launch list.
mkdir -p gpurun_out
T=${TAG:-r02bi}
timeout 900 python tools/density_sweep.py --steps 5 > gpurun_out/${T}_density_sweep.jsonl 2> gpurun_out/${T}_density.err; echo SWEEP_RC=$?
cat gpurun_out/${T}_density_sweep.jsonl
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${T}_t90_launches.csv python tools/density_sweep.py --steps 1 --theta 90 > gpurun_out/${T}_t90_ncu.log 2>&1; echo NCU_RC=$?
python tools/launch_summary.py gpurun_out/${T}_t90_launches.csv > gpurun_out/${T}_t90_launches_summary.txt 2>&1
tail -30 gpurun_out/${T}_t90_launches_summary.txt
