# level mode default: parity suite, halves sweep, wq (greedy claims + edge-parallel local levels)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lv1_tests.log 2>&1; tail -4 gpurun_out/lv1_tests.log
for mode in level:4 level:1 level:2 level:8 wq:32; do
  m=${mode%%:*}; k=${mode##*:}
  PIRRT_BFS=$m PIRRT_HALVES=$k timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv1_bench_$m$k.json 2> gpurun_out/lv1_bench_$m$k.err
  python -c "import json;d=json.load(open('gpurun_out/lv1_bench_$m$k.json'));print('$mode', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
