# ncu --set full with source of the C4 decode list/round-0 kernels.
mkdir -p gpurun_out
T=${TAG:-r02y}
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 1 --warmup 3"
TAGC_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_list_count|k_list_write|k_r0_phase1|k_emit" -s 12 -c 4 -o gpurun_out/${T}_full $B > gpurun_out/${T}_ncu.log 2>&1; echo NCU_RC=$?
python tools/ncu_summary.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1; cat gpurun_out/${T}_ncu_summary.txt
ncu -i gpurun_out/${T}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_source.csv 2>/dev/null; ls -la gpurun_out/${T}_source.csv
ncu -i gpurun_out/${T}_full.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>/dev/null
