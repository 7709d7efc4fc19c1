# Programmatic dependent launch A/B + full GPU suite.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
B="python bench.py --no-cpu-baseline --no-e2e --no-owner-step"
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["extras"]["gpt2"]["ms_per_step"], d["extras"]["gpt2-paper"]["ms_per_step"])'
for r in 1 2 3; do for v in 1 0; do echo -n "pdl=$v: "; TAGC_PDL=$v timeout 600 $B 2>/dev/null | tail -1 | python -c "$P"; done; done
