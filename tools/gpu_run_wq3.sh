# batched visits + unified rows: GPU parity suite, bench both Evaluate modes + keep sweep, wq trace
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/wq3_tests.log 2>&1; tail -4 gpurun_out/wq3_tests.log
for mode in level:0 wq:32 wq:16 wq:64; do
  m=${mode%%:*}; k=${mode##*:}
  PIRRT_BFS=$m PIRRT_WQ_KEEP=$k timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/wq3_bench_$m$k.json 2> gpurun_out/wq3_bench_$m$k.err
  python -c "import json;d=json.load(open('gpurun_out/wq3_bench_$m$k.json'));print('$mode', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
PIRRT_WQ_KEEP=32 GRAPH_CACHE=/tmp/g_probe.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py > gpurun_out/wq3_trace_32.log 2>&1; grep "^wq\|==" gpurun_out/wq3_trace_32.log | tail -6
PIRRT_BFS=level GRAPH_CACHE=/tmp/g_probe.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py > gpurun_out/wq3_trace_level.log 2>&1; grep -v "^$" gpurun_out/wq3_trace_level.log | tail -18
