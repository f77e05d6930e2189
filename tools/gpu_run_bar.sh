# software grid barrier vs cooperative_groups grid.sync
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/bar_tests.log 2>&1; tail -3 gpurun_out/bar_tests.log
for v in sw cgbar sw; do
  lib=paper_2003_04920_b200/lib/libpirrt.so; [ $v = cgbar ] && lib=paper_2003_04920_b200/lib/libpirrt_cgbar.so
  PIRRT_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/bar_bench_$v.json 2> gpurun_out/bar_bench_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bar_bench_$v.json'));print('$v', d['value'], d['exploit_ms_mean'], d['append_plus_readout_ms_mean'], d['phase_ms'], d['roofline']['frac'])"
done
GRAPH_CACHE=/tmp/g_probe.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py > gpurun_out/bar_trace.log 2>&1; grep -v "^$" gpurun_out/bar_trace.log | tail -16
