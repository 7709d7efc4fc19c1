# ncu --set full of k_fused_tma (and the high-load decode kernels) at C4 theta = 90.
mkdir -p gpurun_out
TAGC_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_fused_tma|k_r0_subtract_cnt|k_peel|k_ds_place" -s 4 -c 4 -o gpurun_out/r02bl_t90 \
  python tools/density_sweep.py --steps 1 --theta 90 > gpurun_out/r02bl_ncu.log 2>&1; echo NCU_RC=$?
python tools/ncu_summary.py gpurun_out/r02bl_t90.ncu-rep > gpurun_out/r02bl_t90_ncu_summary.txt 2>&1
python tools/ncu_hot.py gpurun_out/r02bl_t90.ncu-rep cuda 25 k_fused_tma > gpurun_out/r02bl_fused_hot.txt 2>&1
head -120 gpurun_out/r02bl_t90_ncu_summary.txt
