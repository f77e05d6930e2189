timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2j_tests.log 2>&1; tail -3 gpurun_out/s2j_tests.log
export GRAPH_CACHE=/tmp/g1m.npz
timeout 600 python tools/wide_probe.py 2>&1 | tail -1
for i in 1 2; do
  (cd old_ref && python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('old', d['value'], d['exploit_ms_mean'], d['phase_ms'])")
  python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('new', d['value'], d['exploit_ms_mean'], d['phase_ms'])"
done
