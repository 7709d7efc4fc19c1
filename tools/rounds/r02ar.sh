# k_peel small-peel shortcut: parity + C4 / GPT-2 peel times.
mkdir -p gpurun_out
T=${TAG:-r02ar}
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_golden.py tests/test_gpu_exchange.py tests/test_gpu_world.py tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_bigworld.py -q -x -p no:cacheprovider 2>&1 | tail -1
for wl in c4 gpt2; do
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_peel|k_r0_sub" --csv --log-file gpurun_out/${T}_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
echo "$wl: $(python tools/launch_summary.py gpurun_out/${T}_$wl.csv | grep k_ | tr -s ' ' | tr '\n' ' ')"
done
timeout 200 python tools/w8_decode_probe.py 8 2>&1 | tail -1
