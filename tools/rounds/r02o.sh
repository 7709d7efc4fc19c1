# W=8 owner decode: per-kernel launch list of the decode chain; paper-setting W=2 line with both ranks on one GPU.
mkdir -p gpurun_out
T=${TAG:-r02o}
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_list|k_tile|k_r0|k_peel|k_final|k_emit|k_zero|k_stage" --log-file gpurun_out/${T}_w8_launches.csv python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8_ncu.log 2>&1; echo NCU_RC=$?
python tools/launch_summary.py gpurun_out/${T}_w8_launches.csv > gpurun_out/${T}_w8_summary.txt; cat gpurun_out/${T}_w8_summary.txt
TAGC_DEBUG_PEEL=1 timeout 300 python tools/w8_decode_probe.py 8 > gpurun_out/${T}_w8_peeldbg.log 2>&1; echo DBG_RC=$?; tail -30 gpurun_out/${T}_w8_peeldbg.log
TAGC_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --exchange peer --workload gpt2-paper --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_paper_w2.log 2>&1; echo W2_RC=$?; tail -1 gpurun_out/${T}_paper_w2.log
