# Round-2 checkpoint r02cq (template r02ap): full GPU suite, smoke, bench, reference arm, Llama line,
# C4 launch list, ncu --set full of the top kernels, sanitizer over the workload.
mkdir -p gpurun_out
T=${TAG:-r02cq}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -3 gpurun_out/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo SMOKE_RC=$?; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo BENCH_RC=$?; tail -1 gpurun_out/${T}_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo REF_RC=$?
timeout 900 python bench.py --workload llama3-8b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-owner-step > gpurun_out/${T}_bench_llama.log 2>&1; echo LLAMA_RC=$?
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches_summary.txt 2>&1
B="python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 1 --warmup 3"
TAGC_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_fused_tma|k_ds_place|k_ds_apply_smem|k_list_write|k_r0_phase1|k_peel|k_emit" -s 10 -c 7 -o gpurun_out/${T}_full $B > gpurun_out/${T}_ncu.log 2>&1; echo NCU_RC=$?
python tools/ncu_summary.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_ncu_full_summary.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_workload.py > gpurun_out/${T}_sanitize_${tool}.log 2>&1; echo SAN_${tool}_RC=$?; tail -1 gpurun_out/${T}_sanitize_${tool}.log
done
timeout 900 python tools/density_sweep.py --steps 5 > gpurun_out/${T}_density_sweep.jsonl 2>&1; echo SWEEP_RC=$?
