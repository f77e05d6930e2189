# level mode + work-queue tail
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lv4_tests.log 2>&1; tail -3 gpurun_out/lv4_tests.log
for t in -1 0 2000 600; do
  PIRRT_WQ_TAIL=$t timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv4_bench_$t.json 2> gpurun_out/lv4_bench_$t.err
  python -c "import json;d=json.load(open('gpurun_out/lv4_bench_$t.json'));print('tail=$t', d['value'], d['exploit_ms_mean'], d['append_plus_readout_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
GRAPH_CACHE=/tmp/g_probe.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py > gpurun_out/lv4_trace.log 2>&1; grep -v "^$" gpurun_out/lv4_trace.log | tail -14
