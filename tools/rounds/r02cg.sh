mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python tools/onebit_probe.py 2>&1 | tail -2 | head -1; done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ordered or onebit or w1 or multirank or ipc or peer or world or bigworld" 2>&1 | tail -1
