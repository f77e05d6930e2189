# work queue: out-rows travel with the items, rows prefetched into L2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lv7_tests.log 2>&1; tail -3 gpurun_out/lv7_tests.log
for wk in -1:32 2000:32 -1:16 0:32; do
  w=${wk%%:*}; k=${wk##*:}
  PIRRT_WQ_WIDE=$w PIRRT_WQ_KEEP=$k timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv7_$w_$k.json 2> gpurun_out/lv7_$w_$k.err
  python -c "import json;d=json.load(open('gpurun_out/lv7_$w_$k.json'));print('wide=$w keep=$k', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'])"
done
GRAPH_CACHE=/tmp/g_probe.npz PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_trace.so python tools/level_probe.py > gpurun_out/lv7_trace.log 2>&1; grep "^wq" gpurun_out/lv7_trace.log | tail -3
