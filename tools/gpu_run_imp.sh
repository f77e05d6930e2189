# Improve unroll / lanes-per-vertex variants (Evaluate unchanged)
for v in base u8l16 u8l32 u6l16 u4l32 base; do
  lib=paper_2003_04920_b200/lib/libpirrt.so; [ $v != base ] && lib=paper_2003_04920_b200/lib/libpirrt_$v.so
  PIRRT_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz > gpurun_out/imp_$v.json 2> gpurun_out/imp_$v.err
  python -c "import json;d=json.load(open('gpurun_out/imp_$v.json'));print('$v', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['roofline']['improve_phase_GBps'])"
done
