# one ncu --set full capture of the fused select/encode pass of the bench step
mkdir -p gpurun_out
ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/fused_tma python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
echo done
