mkdir -p gpurun_out
for k in "2-4-5" "4-4-2" "2-1-2"; do
TAGC_DEBUG_PEER=1 TAGC_PEER_TIMEOUT_MS=5000 timeout 300 python -m pytest "tests/test_gpu_multirank.py::test_peer_exchange_matches_oracle[$k]" -q -p no:cacheprovider -s > gpurun_out/r02j_peer_$k.log 2>&1; echo PEER_RC=$?; tail -1 gpurun_out/r02j_peer_$k.log
done
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 1 --warmup 3"
TAGC_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_list|k_r0_phase1|k_ds_count|k_ds_place|k_ds_apply|k_sample|k_emit|k_finish_select|k_fixup" -s 30 -c 10 -o gpurun_out/r02j_full $B > gpurun_out/r02j_ncu.log 2>&1; echo NCU_RC=$?
python tools/ncu_summary.py gpurun_out/r02j_full.ncu-rep > gpurun_out/r02j_ncu_summary.txt 2>&1; cat gpurun_out/r02j_ncu_summary.txt | grep -E "^==|duration|dram__bytes|stalls|hit_rate"
