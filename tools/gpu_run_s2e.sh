# children-index Evaluate: parity + cold-solve timing + bench
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2e_tests.log 2>&1; tail -4 gpurun_out/s2e_tests.log
export GRAPH_CACHE=/tmp/g1m.npz
PIRRT_KIDS_MIN=0 timeout 600 python tools/wide_probe.py 2>&1 | tail -1
timeout 600 python tools/wide_probe.py 2>&1 | tail -1
python bench.py --no-cpu-baseline > gpurun_out/s2e_bench.json 2> gpurun_out/s2e_bench.err; cut -c1-200 gpurun_out/s2e_bench.json; tail -2 gpurun_out/s2e_bench.err
