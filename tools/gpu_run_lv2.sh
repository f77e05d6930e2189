# level queue records (g + out-rows travel with the pushed child)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lv2_tests.log 2>&1; tail -4 gpurun_out/lv2_tests.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv2_bench_$i.json 2> gpurun_out/lv2_bench_$i.err
  python -c "import json;d=json.load(open('gpurun_out/lv2_bench_$i.json'));print('$i', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
