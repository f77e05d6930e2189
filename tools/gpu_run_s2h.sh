# headline A/B: session-start build (old_ref) vs HEAD, interleaved
for i in 1 2 3; do
  (cd old_ref && python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('old', d['value'], d['exploit_ms_mean'], d['phase_ms'])")
  python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('new', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
done
