# GPT-2 (theta 99, w 4) launch list of the exchange step.
mkdir -p gpurun_out
TAGC_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02cc_gpt2_launches.csv python bench.py --workload gpt2 --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02cc_gpt2_launches.csv 2>&1 | grep tagc
timeout 600 python bench.py --workload gpt2 --no-cpu-baseline --no-extras --no-e2e --no-owner-step 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['kernel_ms'], d['decode_roofline']['span_ms'])"
