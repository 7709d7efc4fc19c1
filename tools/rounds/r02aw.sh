# Grid-barrier poll backoff sweep (prebuilt library variants in tmp_libs/).
for ns in 0 30 100 300; do
cp tmp_libs/lib_$ns.so paper_2504_05638_b200/libtagc_b200.so
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_peel" --log-file gpurun_out/bw_$ns.csv python tools/w8_decode_probe.py 8 > /dev/null 2>&1
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_peel" --csv --log-file gpurun_out/bc_$ns.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
echo "ns=$ns w8 $(python tools/launch_summary.py gpurun_out/bw_$ns.csv | grep k_peel | tr -s ' ') | c4 $(python tools/launch_summary.py gpurun_out/bc_$ns.csv | grep k_peel | tr -s ' ')"
done
