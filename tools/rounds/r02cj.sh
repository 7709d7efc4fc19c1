B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step --no-extras"
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stages_ms"]["decode"])'
for r in 1 2; do for k in 2 4 8 16; do echo -n "place/SM=$k: "; TAGC_DS_PLACE_PER_SM=$k timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"; done; done
for k in 2 8; do TAGC_DS_PLACE_PER_SM=$k TAGC_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ds -c 20 --csv --log-file gpurun_out/r02cj_ds$k.csv $B > /dev/null 2>&1; echo "k=$k"; python tools/launch_summary.py gpurun_out/r02cj_ds$k.csv 2>&1 | grep k_ds; done
