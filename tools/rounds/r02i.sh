mkdir -p gpurun_out
for k in "2-4-5" "4-4-2"; do
TAGC_DEBUG_PEER=1 TAGC_PEER_TIMEOUT_MS=5000 timeout 300 python -m pytest "tests/test_gpu_multirank.py::test_peer_exchange_matches_oracle[$k]" -q -p no:cacheprovider -s > gpurun_out/r02i_peer_$k.log 2>&1; echo PEER_RC=$?; tail -3 gpurun_out/r02i_peer_$k.log
done
