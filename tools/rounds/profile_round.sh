# Round profile capture: launch list of a bench step (cold, serialised) and one
# ncu --set full capture of the dominant kernels; outputs in gpurun_out/.
mkdir -p gpurun_out
TAGC_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
TAGC_GRAPHS=0 ncu --set full --clock-control none --import-source on \
    -k regex:"k_fused_tma|k_sample|k_window|k_finish_select|k_fixup|k_list|k_r0_phase1|k_emit|k_peel" -s 20 -c 10 -o gpurun_out/full \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
