timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2n_tests.log 2>&1; tail -3 gpurun_out/s2n_tests.log
for i in 1 2; do
 for f in 0 1; do
  PIRRT_WQ_FILL=$f python bench.py --no-cpu-baseline --graph-cache /tmp/g_bench2.npz 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fill=$f', d['value'], d['exploit_ms_mean'], d['phase_ms'], 'e2e', d['e2e']['value'], 'sync', d['e2e']['sync_value'])"
 done
done
PIRRT_DEBUG_HOST=1 GRAPH_CACHE=/tmp/g1m.npz timeout 600 python tools/wide_probe.py 2>&1 | tail -8
ls -la /tmp/*.npz
PIRRT_DEBUG_HOST=1 timeout 1500 python tools/gstar_probe.py --n 1000000 --cache /tmp/g1m_star.npz --skip-batches --out gpurun_out/gstar_1m_c.json 2>&1 | tail -8
