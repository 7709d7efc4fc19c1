# k_emit: per-thread vector stores vs TMA bulk stores.
mkdir -p gpurun_out
T=${TAG:-r02ao}
for v in "X=1" "TAGC_EMIT_STG=1"; do
env $v timeout 200 python bench.py --no-extras --no-e2e --no-owner-step --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d.get('stages_ms'))"
done
TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_emit" --csv --log-file gpurun_out/${T}_emit.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --no-owner-step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_emit.csv | grep k_
