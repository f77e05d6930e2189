for i in 1 2 3; do
  (cd old_ref && python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('old', d['value'], d['exploit_ms_mean'], d['phase_ms'])")
  python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A  ', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
  PIRRT_LIB=paper_2003_04920_b200/lib/libpirrt_C.so python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C  ', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
  PIRRT_KIDS_MIN=0 PIRRT_WIDE_TASKS=0 python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A00', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
done
