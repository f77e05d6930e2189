# hand over to the work queue once the frontier is wide (PIRRT_WQ_WIDE)
for wk in 0:32 1000:32 2000:32 3000:32 1000:16 2000:64 500:32; do
  w=${wk%%:*}; k=${wk##*:}
  PIRRT_WQ_WIDE=$w PIRRT_WQ_KEEP=$k timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv6_$w_$k.json 2> gpurun_out/lv6_$w_$k.err
  python -c "import json;d=json.load(open('gpurun_out/lv6_$w_$k.json'));print('wide=$w keep=$k', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'])"
done
