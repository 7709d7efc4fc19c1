# ncu --set full of the C4 step's decode + deferred-scatter kernels (one launch each, warm step).
mkdir -p gpurun_out
T=${TAG:-r02q}
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 1 --warmup 3"
TAGC_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_list_count|k_list_write|k_r0_phase1|k_r0_subtract_cnt|k_peel|k_emit|k_ds_place|k_ds_apply|k_ds_count|k_fused_tma|k_finish_select" -s 33 -c 11 -o gpurun_out/${T}_full $B > gpurun_out/${T}_ncu.log 2>&1; echo NCU_RC=$?
python tools/ncu_summary.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1; grep -E "^==|duration|dram__bytes|stalls|hit_rate|lts__throughput" gpurun_out/${T}_ncu_summary.txt
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null; ls -la gpurun_out/${T}_raw.csv
