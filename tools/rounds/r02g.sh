# Round-2 checkpoint: full GPU suite, smoke, default bench line, C4 launch list.
mkdir -p gpurun_out
T=${TAG:-r02g}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 600 > gpurun_out/${T}_gputest.log 2>&1; echo TEST_RC=$?
tail -15 gpurun_out/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo SMOKE_RC=$?; tail -3 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo BENCH_RC=$?; tail -1 gpurun_out/${T}_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo REF_RC=$?; tail -1 gpurun_out/${T}_bench_ref.log
