# GPU tests, the bench (TMA and register fused pass), and one ncu --set full capture of each
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
TAGC_FUSED_TMA=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench0.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/fused_tma python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
echo done
