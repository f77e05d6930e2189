timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2x_tests.log 2>&1; tail -4 gpurun_out/s2x_tests.log
for i in 1 2; do
for f in 0 1; do
  PIRRT_FUSE_ROOT=$f python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench6.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fuse=$f', d['value'], d['exploit_ms_mean'], d['phase_ms'], d['grid_barriers_per_exploit'])"
done
done
