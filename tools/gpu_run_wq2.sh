# work-queue Evaluate v2: GPU parity suite, then bench in both Evaluate modes + keep sweep
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/wq2_tests.log 2>&1; tail -15 gpurun_out/wq2_tests.log
for mode in wq:32 level:0 wq:16 wq:64 wq:8; do
  m=${mode%%:*}; k=${mode##*:}
  PIRRT_BFS=$m PIRRT_WQ_KEEP=$k timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/wq2_bench_$m$k.json 2> gpurun_out/wq2_bench_$m$k.err
  python -c "import json;d=json.load(open('gpurun_out/wq2_bench_$m$k.json'));print('$mode', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
