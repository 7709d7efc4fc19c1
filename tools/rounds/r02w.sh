# ncu --set full of the new deferred-scatter kernels (C4).
mkdir -p gpurun_out
T=${TAG:-r02w}
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 1 --warmup 3"
TAGC_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_ds_place|k_ds_apply_smem" -s 6 -c 2 -o gpurun_out/${T}_full $B > gpurun_out/${T}_ncu.log 2>&1; echo NCU_RC=$?
python tools/ncu_summary.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1; cat gpurun_out/${T}_ncu_summary.txt
ncu -i gpurun_out/${T}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_source.csv 2>/dev/null; ls -la gpurun_out/${T}_source.csv
