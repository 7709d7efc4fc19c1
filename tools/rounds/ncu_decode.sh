# one ncu --set full capture of the decode kernels of the bench step
mkdir -p gpurun_out
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_r0|k_accumulate|k_peel|k_build" -s 15 -c 5 -o gpurun_out/decode python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dec.log 2>&1
echo done
