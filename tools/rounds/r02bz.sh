# Llama-3-8B layout: launch list of one exchange step (where do the 15.7 ms of grouped decode go?)
mkdir -p gpurun_out
TAGC_GRAPHS=0 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r02bz_llama_launches.csv python bench.py --workload llama3-8b --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-owner-step > gpurun_out/r02bz_ncu.log 2>&1; echo NCU_RC=$?
python tools/launch_summary.py gpurun_out/r02bz_llama_launches.csv > gpurun_out/r02bz_llama_launches_summary.txt 2>&1
grep tagc gpurun_out/r02bz_llama_launches_summary.txt; tail -2 gpurun_out/r02bz_llama_launches_summary.txt
