# work-queue tail threshold / keep sweep
for tk in 2000:32 3000:32 4500:32 7000:32 3000:64 4500:64 3000:16; do
  t=${tk%%:*}; k=${tk##*:}
  PIRRT_WQ_TAIL=$t PIRRT_WQ_KEEP=$k timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/lv5_bench_$t_$k.json 2> gpurun_out/lv5_bench_$t_$k.err
  python -c "import json;d=json.load(open('gpurun_out/lv5_bench_$t_$k.json'));print('tail=$t keep=$k', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'], d['roofline']['frac'])"
done
