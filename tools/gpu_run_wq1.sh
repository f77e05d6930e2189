# work-queue Evaluate: GPU parity suite, then bench in both Evaluate modes
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/wq1_tests.log 2>&1; tail -15 gpurun_out/wq1_tests.log
for mode in wq level; do
  PIRRT_BFS=$mode timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/wq1_bench_$mode.json 2> gpurun_out/wq1_bench_$mode.err
  python -c "import json;d=json.load(open('gpurun_out/wq1_bench_$mode.json'));print('$mode', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
