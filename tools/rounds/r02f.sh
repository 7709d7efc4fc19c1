mkdir -p gpurun_out
TAGC_DEBUG_PEER=1 TAGC_PEER_TIMEOUT_MS=4000 timeout 300 python -m pytest "tests/test_gpu_multirank.py::test_peer_exchange_matches_oracle" -q -p no:cacheprovider -s > gpurun_out/r02f_peerdbg.log 2>&1; echo PEER_RC=$?; tail -3 gpurun_out/r02f_peerdbg.log
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 1 --warmup 3"
TAGC_GRAPHS=0 TAGC_FUSED_EMIT=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_list|k_r0_phase1|k_r0_subtract_cnt|k_peel|k_emit|k_ds_apply|k_ds_place|k_sample" -s 40 -c 9 -o gpurun_out/r02f_full $B > gpurun_out/r02f_ncu.log 2>&1; echo NCU_RC=$?
TAGC_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"k_r0_emit|k_final_fix" -s 10 -c 2 -o gpurun_out/r02f_fused $B > gpurun_out/r02f_ncu2.log 2>&1; echo NCU2_RC=$?
ls -la gpurun_out
