# High-load decode after staged overflow appends (round 0 lists, k_peel global queue): sweep + decode tests.
mkdir -p gpurun_out
for t in 90 95; do
  for z in 0 1; do
    echo "theta=$t zero_state=$z"; TAGC_DECODE_ZERO_STATE=$z TAGC_DEBUG_PEEL=1 timeout 300 python tools/density_sweep.py --steps 1 --theta $t 2>&1 | tail -2 | cut -c1-600
  done
done
timeout 900 python tools/density_sweep.py --steps 5 > gpurun_out/r02bk_density_sweep.jsonl 2>&1; cat gpurun_out/r02bk_density_sweep.jsonl
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/r02bk_t90_launches.csv python tools/density_sweep.py --steps 1 --theta 90 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02bk_t90_launches.csv 2>&1 | grep tagc_b200 > gpurun_out/r02bk_t90_launches_summary.txt; cat gpurun_out/r02bk_t90_launches_summary.txt
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "codec or golden or scale or exchange or multirank or bigworld" 2>&1 | tail -3
