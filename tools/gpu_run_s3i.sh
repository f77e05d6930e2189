for i in 1 2 3; do
for lib in libpirrt.so libpirrt_ui3.so libpirrt_ui6.so; do
  PIRRT_LIB=paper_2003_04920_b200/lib/$lib python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench8.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
done
done
