# block-chunked edge-parallel level expansion vs warp-per-item
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lv3_tests.log 2>&1; tail -3 gpurun_out/lv3_tests.log
for h in 0 4 0; do
  PIRRT_HALVES=$h timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv3_bench_$h.json 2> gpurun_out/lv3_bench_$h.err
  python -c "import json;d=json.load(open('gpurun_out/lv3_bench_$h.json'));print('halves=$h', d['value'], d['exploit_ms_mean'], d['append_plus_readout_ms_mean'], d['phase_ms'], d['roofline']['frac'])"
done
GRAPH_CACHE=/tmp/g_probe.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py > gpurun_out/lv3_trace.log 2>&1; grep -v "^$" gpurun_out/lv3_trace.log | tail -16
